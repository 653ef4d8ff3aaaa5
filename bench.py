#!/usr/bin/env python
"""Benchmark of the B200 forward-convolution engine (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5] [--batch B] [--engine fused|twostage]
                    [--report PATH]        # per-layer sweep of all BASELINE configs

A *step* is one pass of the hot path over one batch of synthetic input: every
layer of the workload convolved once with its filter bank.  The default is
the configuration BASELINE.json's metric is quoted on ("at 1/2/4/8 B200"):
configs[4], the 53 convolutions of ResNet-50 v1.5 at a global batch of 256,
batch-sharded over the GPUs (strong scaling; it fits one GPU).  ``value`` is
whole-job GFLOP/s (algorithmic flops 2*N*M*Ho*Wo*C*hf*wf of all ranks /
max-over-ranks device time of K steps, each step replayed as one CUDA graph
with inputs resident in HBM).

Also reported: ``e2e`` (same metric through the host-buffer C-ABI drop-in,
H2D of inputs+filters and D2H of outputs inside the timed region),
``roofline`` (the dominant kernel family's algorithmic TFLOP/s (or GB/s for
HBM-bound layers) from CUDA events recorded between the layers of one
sequential pass of the same step, over the FFMA2 peak measured live by
``b2c_probe_fp32_peak`` or MEASURED_PEAKS.json's HBM bandwidth),
``cpu_baseline`` (the oracle's C port of the reference's conv_twostage on the
host's cores, plus the real convkit functions when baseline/_ref holds the
reference), ``clocks`` (NVML during the timed region) and ``gpu_launches``.
Under torchrun, ``gather`` times the NCCL gather of one layer's output to
rank 0 separately (never folded into ``value``).

``tensor_core_variant``: the north star's optional tcgen05 implicit-GEMM
engine (3xTF32 by default, ``--tc-engine``) on the same workload and operands,
with its own stated tolerance and a tensor-bound roofline.

``--impl reference`` times the reference algorithm on the CPU (the oracle
port of convkit.conv_twostage, all host threads) for the same metric and
workload: each step is one pass over every layer of the workload at a bounded
sample batch (stated in ``cpu_baseline.sample``); under torchrun only rank 0
runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.45: 148 SMs x 128 FP32 lanes x 2 x 1965 MHz
DEFAULT_BATCH = {"c1": 1, "c2": 32, "c3": 128, "c4": 128, "c5": 256}
STRONG = {"c5"}  # ResNet-50 N=256 is split across GPUs (strong scaling)


def parse():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=("c1", "c2", "c3", "c4", "c5"), default="c5")
    ap.add_argument("--batch", type=int, default=0, help="images per layer (per GPU, or global for c5)")
    ap.add_argument("--engine", choices=("fused", "twostage", "tf32x3", "tf32"), default="fused")
    ap.add_argument("--tc-engine", choices=("tf32x3", "tf32", "none"), default="tf32x3",
                    help="tensor-core variant reported separately in the same line (north star: optional, own tolerance)")
    ap.add_argument("--report", default="", help="write a per-layer sweep of every BASELINE config to PATH")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--schedule", choices=("dataflow", "sequential"), default="dataflow",
                    help="dataflow: data-independent layers of the source network (inception branches, ResNet "
                         "projection shortcuts) run concurrently inside the step graph; sequential: one stream")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--layer-passes", type=int, default=3,
                    help="sequential passes of the step with CUDA events between layers (roofline attribution)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are best-effort metadata
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


# --------------------------------------------------------------------------- CPU legs
def host_info():
    """The host the CPU legs ran on: usable cores, CPU model, BLAS threads."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"affinity_cpus": len(os.sched_getaffinity(0)), "cpu_model": model,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


def port_pass(work, threads):
    """One pass of the oracle's C port of convkit.conv_twostage over `work`
    (stage 1 + stage 2, the reference's rounding); strided layers, which the
    reference's conv_twostage refuses (twostage.py:74-75), through the port of
    conv_naive (its strided path, reference.py:58-83).  Returns (s, flops)."""
    import oracle

    secs = flops = 0.0
    for c, x, w in work:
        t0 = time.perf_counter()
        if c.stride == 1:
            oracle.conv_twostage(c, x, w, threads=threads)
        else:
            oracle.conv_naive(c, x, w, threads=threads)
        secs += time.perf_counter() - t0
        flops += c.flops
    return secs, flops


def sample_work(cfgs, sample_batch, rng_seed=0):
    import oracle
    from paper_2103_16234_b200.configs import filter_dims, input_dims

    work = []
    for i, cfg in enumerate(cfgs):
        c = cfg.with_batch(sample_batch)
        work.append((c, oracle.make_uniform(input_dims(c), seed=rng_seed + 2 * i),
                     oracle.make_uniform(filter_dims(c), seed=rng_seed + 2 * i + 1)))
    return work


def cpu_run(cfgs, sample_batch, min_seconds):
    """The port on every host thread, whole passes over the workload's layers
    at `sample_batch`, for at least `min_seconds`."""
    import oracle

    threads = oracle.max_threads()
    work = sample_work(cfgs, sample_batch)
    secs = flops = 0.0
    passes = 0
    while passes == 0 or secs < min_seconds:
        ds, df = port_pass(work, threads)
        secs += ds
        flops += df
        passes += 1
    return flops / secs / 1e9, threads, passes


def convkit_legs(cfgs, budget_s=6.0):
    """The real reference functions (convkit from baseline/_ref or
    $CONVKIT_REF, when present): conv_twostage(workers=1) and conv_naive on
    one core, conv_naive_f64 on OpenBLAS's threads, each over the workload's
    layers at N=1 in network order until `budget_s` is spent (bounded sample).
    Layers the reference refuses are recorded with the reference harness's
    skip strings (bench.py:63-78)."""
    import importlib

    for p in (os.environ.get("CONVKIT_REF"), os.path.join(ROOT, "baseline", "_ref")):
        if p and os.path.isdir(os.path.join(p, "convkit")) and p not in sys.path:
            sys.path.insert(0, p)
    try:
        ck = importlib.import_module("convkit")
        from convkit.bench import skip_reason
    except Exception as exc:  # noqa: BLE001 - the reference is optional on the GPU box
        return {"available": False, "why": f"convkit not importable: {exc.__class__.__name__}"}
    out = {"available": True, "source": os.path.dirname(ck.__file__), "legs": {}}
    for algo, fn in (("twostage", lambda x, w, c: ck.conv_twostage(x, w, c, workers=1)),
                     ("naive", lambda x, w, c: ck.conv_naive(x, w, c)),
                     ("naive_f64", lambda x, w, c: ck.conv_naive_f64(x, w, c))):
        secs = flops = 0.0
        done, skips = [], []
        for i, cfg in enumerate(cfgs):
            c = cfg.with_batch(1)
            kc = ck.ConvConfig(c.name, n=1, c=c.c, h=c.h, w=c.w, m=c.m, hf=c.hf, wf=c.wf, stride=c.stride,
                               pad_h=c.pad_h, pad_w=c.pad_w)
            why = skip_reason("twostage", kc, ck.DEFAULT_WORKSPACE_LIMIT) if algo == "twostage" else None
            if why:
                skips.append({"layer": c.name, "skip": why})
                continue
            x = ck.make_tensor(ck.input_dims(kc), "uniform", seed=2 * i)
            w = ck.make_tensor(ck.filter_dims(kc), "uniform", seed=2 * i + 1)
            t0 = time.perf_counter()
            fn(x, w, kc)
            secs += time.perf_counter() - t0
            flops += c.flops
            done.append(c.name)
            if secs >= budget_s:
                break
        out["legs"][algo] = {"gflops": round(flops / secs / 1e9, 4) if secs else None,
                             "cores": 1 if algo != "naive_f64" else "openblas",
                             "layers_timed": len(done), "seconds": round(secs, 2), "skips": skips,
                             "sample": f"first {len(done)} layers in network order at N=1 "
                                       f"(bounded to ~{budget_s:.0f} s)"}
    return out


def reference_arm(args, cfgs, metric, config):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    sample_batch = 1
    threads = oracle.max_threads()
    work = sample_work(cfgs, sample_batch)
    for _ in range(args.warmup):
        port_pass(work, threads)
    tot_t = tot_f = 0.0
    for _ in range(args.steps):
        t, f = port_pass(work, threads)
        tot_t += t
        tot_f += f
    value = tot_f / tot_t / 1e9
    sample = (f"each step = one pass over all {len(cfgs)} layers of {args.workload} at N={sample_batch} "
              f"(the bench's batch is {config['global_batch']}; images are independent, so GFLOP/s is "
              f"batch-size independent up to cache effects); oracle C port of convkit.conv_twostage "
              f"(stage1+stage2, reference rounding) on {threads} threads; strided layers, which "
              f"conv_twostage refuses, via the conv_naive port")
    cfg = dict(config, reference_sample_batch=sample_batch)
    line = {"metric": metric, "value": round(value, 3), "unit": "GFLOP/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * tot_t / args.steps, 3), "higher_is_better": True,
            "scaling": "strong" if args.workload in STRONG else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
                             "sample": sample, "host": host_info()},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU leg
def make_operands(cfgs, device, seed):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    xs, ws, ys = [], [], []
    for cfg in cfgs:
        xs.append(torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device=device) * 2 - 1)
        ws.append(torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device=device) * 2 - 1)
        ho = (cfg.h + 2 * cfg.pad_h - cfg.hf) // cfg.stride + 1
        wo = (cfg.w + 2 * cfg.pad_w - cfg.wf) // cfg.stride + 1
        ys.append(torch.empty((cfg.n, cfg.m, ho, wo), device=device))
    return xs, ws, ys


def graph_time(fn, reps):
    """Device time (ms) of one call of ``fn``: ``reps`` calls captured in a CUDA
    graph, the graph replayed 3 times (median) -- host launch overhead (Python,
    ctypes, planning) stays out, so small layers show their kernel time."""
    import torch

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    return sorted(ts)[1]


def time_layers(layers, xs, ws, ys, reps=20):
    """Per-layer kernel time (ms), each layer replayed back to back in a CUDA
    graph (L2-warm, isolated) -- used only by the --report sweep."""
    return [graph_time(lambda L=L, x=x, w=w, y=y: L(x, w, out=y), reps) for L, x, w, y in zip(layers, xs, ws, ys)]


def time_layers_in_step(layers, xs, ws, ys, passes=3):
    """Per-layer device time (ms) inside the step: the step's layers run once
    in network order on one stream with a CUDA event recorded between
    consecutive layers (on the launching stream), so every layer meets the
    cache state the step leaves it (the previous layers' operands, not its
    own) and the per-layer times add up to one sequential step.  A device
    spin (torch.cuda._sleep) at the head lets the host enqueue the whole pass
    first, so no launch gaps fall inside the intervals.  Mean of `passes`."""
    import torch

    stream = torch.cuda.current_stream()
    n = len(layers)
    acc = [0.0] * n
    for L, x, w, y in zip(layers, xs, ws, ys):  # plans resolved, workspaces allocated
        L(x, w, out=y)
    torch.cuda.synchronize()
    for _ in range(passes):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        torch.cuda._sleep(200_000_000)  # ~0.1 s of device time: the host gets ahead
        ev[0].record(stream)
        for i, (L, x, w, y) in enumerate(zip(layers, xs, ws, ys)):
            L(x, w, out=y)
            ev[i + 1].record(stream)
        ev[-1].synchronize()
        for i in range(n):
            acc[i] += ev[i].elapsed_time(ev[i + 1])
    return [a / passes for a in acc]


TRAFFIC_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r2_traffic.json")


def dominant_kernel(cfgs, layers, layer_ms, workload, peak_tflops, hbm_gbs):
    """The kernel family with the largest share of the step's device time
    (per-layer times from time_layers_in_step, split-C sums included): its
    algorithmic flop and bytes per launch, its binding roofline (FP32 when its
    layers' flop/byte is above the ridge peak_fp32/HBM, else HBM), achieved =
    algorithmic work / its summed time, and -- when a committed ncu capture of
    the same layers and plans exists (profiles/r2_traffic.json, written by
    tools/traffic.py) -- the measured DRAM bytes per launch."""
    fam = {}
    for c, L, t in zip(cfgs, layers, layer_ms):
        k = L.family.replace("_dsm", "")
        e = fam.setdefault(k, {"ms": 0.0, "flops": 0, "bytes": 0, "layers": []})
        e["ms"] += t
        e["flops"] += c.flops
        e["bytes"] += c.compulsory_bytes
        e["layers"].append(c.name)
    name, e = max(fam.items(), key=lambda kv: kv[1]["ms"])
    n = len(e["layers"])
    ridge = peak_tflops * 1e12 / (hbm_gbs * 1e9)
    bound = "fp32" if e["flops"] / e["bytes"] >= ridge else "hbm"
    traffic, src = None, None
    try:
        with open(TRAFFIC_PATH) as fh:
            rec = json.load(fh).get(workload, {})
        got = [rec[l]["dram_bytes"] for l in e["layers"] if l in rec and rec[l].get("family", "").replace(
            "_dsm", "") == name]
        if len(got) == n:
            traffic = round(sum(got) / n)
            src = ("ncu dram__bytes_read.sum + dram__bytes_write.sum of the same layers and plans "
                   "(cold cache, conv kernel + its split-C sum), mean per launch: " + os.path.basename(TRAFFIC_PATH))
    except (OSError, ValueError, KeyError):
        pass
    sec = e["ms"] * 1e-3
    return {"kernel": name, "bound": bound, "achieved_tflops": e["flops"] / sec / 1e12,
            "achieved_gbs": e["bytes"] / sec / 1e9, "ms_per_step": e["ms"],
            "share": round(e["ms"] / sum(layer_ms), 4), "launches": n, "flop_per_launch": round(e["flops"] / n),
            "bytes_per_launch": round(e["bytes"] / n), "traffic": traffic, "traffic_source": src,
            "layers": e["layers"]}


def layer_rooflines(cfgs, layers, layer_ms, peak_tflops, hbm_gbs):
    """Per layer: µs, GFLOP/s, its binding roofline and the fraction of it."""
    ridge = peak_tflops * 1e12 / (hbm_gbs * 1e9)
    rows = []
    for c, L, t in zip(cfgs, layers, layer_ms):
        sec = t * 1e-3
        if c.flops / c.compulsory_bytes >= ridge:
            bound, frac = "fp32", c.flops / sec / (peak_tflops * 1e12)
        else:
            bound, frac = "hbm", c.compulsory_bytes / sec / (hbm_gbs * 1e9)
        rows.append({"layer": c.name, "us": round(t * 1e3, 2), "gflops": round(c.flops / sec / 1e9, 1),
                     "bound": bound, "roofline_frac": round(frac, 4), "family": L.family})
    return rows


def time_cudnn(cfgs, xs, ws, reps=10):
    """cuDNN fp32 (TF32 disabled) through torch, per layer, best algorithm
    (benchmark mode) -- an external library baseline for the report only (the
    paper compares cuConv against the best cuDNN algorithm)."""
    import torch
    import torch.nn.functional as F

    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    out = []
    for c, x, w in zip(cfgs, xs, ws):
        def run(c=c, x=x, w=w):
            return F.conv2d(x, w, stride=c.stride, padding=(c.pad_h, c.pad_w))
        for _ in range(3):  # benchmark-mode algorithm selection before capture
            run()
        torch.cuda.synchronize()
        out.append(graph_time(run, reps))
    torch.backends.cudnn.benchmark = False
    return out


def sweep_report(path, device, peak_tflops):
    """Per-layer µs / GFLOP/s / roofline for every BASELINE config and batch."""
    import torch
    from paper_2103_16234_b200 import ConvLayer
    from paper_2103_16234_b200 import workloads as W

    hbm = peaks().get("hbm_gbs", 6540.8)
    rows = []
    for wl, (_, batches) in W.WORKLOADS.items():
        for n in batches:
            cfgs = W.layers(wl, n)
            layers = [ConvLayer(c, "fused") for c in cfgs]
            xs, ws, ys = make_operands(cfgs, device, 1)
            ms = time_layers(layers, xs, ws, ys, reps=10)
            tcl = [ConvLayer(c, "tf32x3") for c in cfgs]
            tms = time_layers(tcl, xs, ws, ys, reps=10)
            cud = time_cudnn(cfgs, xs, ws, reps=10)
            for c, L, t, T, tt, cu in zip(cfgs, layers, ms, tcl, tms, cud):
                flop_per_byte = c.flops / c.compulsory_bytes
                ridge = peak_tflops * 1e12 / (hbm * 1e9)
                if flop_per_byte >= ridge:
                    bound, frac = "fp32", c.flops / (t * 1e-3) / (peak_tflops * 1e12)
                else:
                    bound, frac = "hbm", c.compulsory_bytes / (t * 1e-3) / (hbm * 1e9)
                rows.append({"workload": wl, "batch": n, "layer": c.name, "c": c.c, "hw": c.h, "m": c.m,
                             "f": c.hf, "stride": c.stride, "us": round(t * 1e3, 2),
                             "gflops": round(c.flops / (t * 1e-3) / 1e9, 1), "bound": bound,
                             "roofline_frac": round(frac, 4), "family": L.family, "grid": L.grid,
                             "tf32x3_us": round(tt * 1e3, 2), "tf32x3_gflops": round(c.flops / (tt * 1e-3) / 1e9, 1),
                             "tf32x3_plan": T.family,
                             "cudnn_fp32_us": round(cu * 1e3, 2),
                             "cudnn_fp32_gflops": round(c.flops / (cu * 1e-3) / 1e9, 1)})
            del xs, ws, ys
            torch.cuda.empty_cache()
    with open(path, "w") as fh:
        json.dump({"peak_fp32_tflops": peak_tflops, "hbm_gbs": hbm, "rows": rows}, fh, indent=1)
    return rows


def time_graph(lib, layers, xs, ws, ys, args, world, device, local_rank, groups=None):
    """Warm up, capture one step (every layer once) as a CUDA graph, then time
    exactly `steps` replays between barriers + synchronize (CUDA events on
    the replay stream, max over ranks).  `groups` (workloads.schedule) runs
    data-independent layers of a group on parallel streams inside the graph
    (fork/join by events); groups in order.  Returns (ms, launches/step, clocks)."""
    import torch
    import torch.distributed as dist

    groups = groups or [[i] for i in range(len(layers))]
    side = [torch.cuda.Stream() for _ in range(max(len(g) for g in groups))]

    def step():
        main = torch.cuda.current_stream()
        for grp in groups:
            if len(grp) == 1:
                i = grp[0]
                layers[i](xs[i], ws[i], out=ys[i])
                continue
            fork = torch.cuda.Event()
            fork.record(main)
            joins = []
            for k, i in enumerate(grp):
                s = side[k]
                s.wait_event(fork)
                with torch.cuda.stream(s):
                    layers[i](xs[i], ws[i], out=ys[i])
                ev = torch.cuda.Event()
                ev.record(s)
                joins.append(ev)
            for ev in joins:
                main.wait_event(ev)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    cap_stream = torch.cuda.Stream()
    with torch.cuda.stream(cap_stream):
        step()  # warm on the capture stream (allocates per-layer workspaces)
        torch.cuda.synchronize()
        lib.b2c_reset_launch_count()
        with torch.cuda.graph(graph, stream=cap_stream):
            step()
    launches_per_step = int(lib.b2c_launch_count())
    for _ in range(max(args.warmup, 3)):
        graph.replay()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        start.record()
        for _ in range(args.steps):
            graph.replay()
        end.record()
        torch.cuda.synchronize()
    ms_local = start.elapsed_time(end)
    if world > 1:
        t = torch.tensor([ms_local], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        return float(t.item()), launches_per_step, clk
    return ms_local, launches_per_step, clk


def gpu_local_cpus(index: int):
    """CPUs on the GPU's NUMA node (NVML affinity mask), within this process's
    allowed set; None if unknown."""
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = ((os.cpu_count() or 64) + 63) // 64
        masks = pynvml.nvmlDeviceGetCpuAffinity(h, words)
        cpus = {64 * i + b for i, m in enumerate(masks) for b in range(64) if (int(m) >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:  # noqa: BLE001 - binding is an optimisation, never a requirement
        return None


def e2e_run(lib, nat, cfgs, xs, ws, ys, engine_id, steps, world, device, local_rank):
    """See _e2e_run; the host side (pinned buffers and the calling thread) is
    bound to the GPU's NUMA node while it runs (first-touch placement of the
    pinned pages next to the GPU's PCIe root), then the affinity is restored."""
    saved = os.sched_getaffinity(0)
    cpus = None if os.environ.get("B2C_NO_NUMA_BIND") else gpu_local_cpus(local_rank)
    if cpus and cpus != saved:
        os.sched_setaffinity(0, cpus)
    try:
        out = _e2e_run(lib, nat, cfgs, xs, ws, ys, engine_id, steps, world, device, local_rank)
    finally:
        os.sched_setaffinity(0, saved)
    out["host_binding"] = (f"{len(cpus)} of {len(saved)} CPUs (GPU-local NUMA node)" if cpus and cpus != saved
                           else "none")
    return out


def _e2e_run(lib, nat, cfgs, xs, ws, ys, engine_id, steps, world, device, local_rank):
    """Same metric through the host-buffer C-ABI: every step copies each
    layer's input and filters from pinned host memory, convolves, and copies
    the output back, all layers of the step in one b2c_conv_host_layers call
    (copies and compute of consecutive layers overlap on three streams).
    Wall time, max over ranks."""
    import ctypes

    import torch
    import torch.distributed as dist

    n = len(cfgs)
    descs = (nat.ConvDesc * n)()
    xp, wp, yp = ((ctypes.c_void_p * n)() for _ in range(3))
    keep = []
    h2d = d2h = 0
    for i, (c, x, w, y) in enumerate(zip(cfgs, xs, ws, ys)):
        hx = torch.empty(x.shape, dtype=torch.float32, pin_memory=True).copy_(x)
        hw = torch.empty(w.shape, dtype=torch.float32, pin_memory=True).copy_(w)
        hy = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
        keep += [hx, hw, hy]
        descs[i] = nat.desc(c)
        xp[i], wp[i], yp[i] = hx.data_ptr(), hw.data_ptr(), hy.data_ptr()
        h2d += hx.numel() * 4 + hw.numel() * 4
        d2h += hy.numel() * 4

    def e2e_step():
        nat.check(lib.b2c_conv_host_layers(n, descs, xp, wp, yp, engine_id, local_rank))

    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        e2e_step()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    flops = sum(c.flops for c in cfgs)
    return {"value": round(flops * world * steps / dt / 1e9, 3), "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
            "ms_per_step": round(1e3 * dt / steps, 3),
            "path": "b2c_conv_host_layers (C ABI, pinned host buffers; H2D/compute/D2H of consecutive layers "
                    "overlapped on 3 streams, 6 device slots)"}


TC_TOLERANCE = {"tf32x3": "relative_error vs conv_naive_f64 <= 1e-5*max(1, K/4096) (the fp32 gate)",
                "tf32": "relative_error vs conv_naive_f64 <= 5e-3"}


def tensor_core_variant(args, lib, nat, cfgs, gcfgs, xs, ws, ys, world, device, local_rank):
    """The north star's optional tcgen05 implicit-GEMM variant on the same
    workload and operands, reported separately with its stated tolerance.
    Roofline: tensor-bound against the tf32 dense rate, taken as half the
    measured cuBLAS bf16 burst rate (MEASURED_PEAKS.json; B200 dense
    tf32:bf16 = 1:2), divided by the MMA work per product: 3 for 3xTF32 with
    tf32 corrections, 2 when the two correction products run as bf16 MMAs
    (each at twice the tf32 rate: 1 + 1/2 + 1/2), 1 for plain tf32 —
    flop-weighted over the layers' plans."""
    from paper_2103_16234_b200 import workloads as W
    from paper_2103_16234_b200.sharding import shard_layer

    eng = args.tc_engine
    layers = [shard_layer(g, c, eng) for g, c in zip(gcfgs, cfgs)]

    groups = W.schedule(args.workload, cfgs) if args.schedule == "dataflow" else None
    ms_total, launches, clk = time_graph(lib, layers, xs, ws, ys, args, world, device, local_rank, groups)
    flops = sum(c.flops for c in cfgs)
    layer_ms = time_layers_in_step(layers, xs, ws, ys, passes=args.layer_passes)
    kern_ms = sum(layer_ms)
    pk = peaks()
    tf32_peak = pk.get("bf16_tflops", 1590.0) / 2.0
    passes = 3 if eng == "tf32x3" else 1
    units = [(1.0 if eng == "tf32" else (2.0 if L._tc.bf16_corrections else 3.0)) for L in layers]
    unit_eq = sum(c.flops * u for c, u in zip(cfgs, units)) / flops  # tf32 MMA passes per product
    achieved = flops / (kern_ms * 1e-3) / 1e12
    e2e = None
    if args.e2e_steps > 0:
        e2e = e2e_run(lib, nat, cfgs, xs, ws, ys, nat.ENGINES[eng], args.e2e_steps, world, device, local_rank)
    return {"engine": eng, "value": round(flops * world * args.steps / (ms_total * 1e-3) / 1e9, 3),
            "unit": "GFLOP/s", "ms_per_step": round(ms_total / args.steps, 4), "tolerance": TC_TOLERANCE[eng],
            "dtype": "tf32x3 (fp32 operands split hi+lo, fp32 accumulate in TMEM)" if passes == 3 else "tf32",
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3),
                         "peak": round(tf32_peak / unit_eq, 3), "unit": "TFLOP/s",
                         "frac": round(achieved * unit_eq / tf32_peak, 4), "traffic": None,
                         "peak_source": ("MEASURED_PEAKS.json bf16_tflops / 2 (dense tf32 rate)"
                                         + (f" / {unit_eq:.2f} (3xTF32: tf32 hi*hi + bf16 or tf32 correction "
                                            "MMAs, flop-weighted over the plans)" if passes == 3 else "")),
                         "kernel_ms_per_step": round(kern_ms, 4)},
            "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches * args.steps,
            "per_layer": [{"layer": c.name, "us": round(t * 1e3, 2), "gflops": round(c.flops / (t * 1e-3) / 1e9, 1),
                           "plan": L.family} for c, L, t in zip(cfgs, layers, layer_ms)]}


def time_gather(lib, cfgs, ys, world, rank, device):
    """NCCL gather of the largest layer output of the step to rank 0 (only
    when a single-device result is requested; never inside ``value``):
    device time, max over ranks, and the bytes moved."""
    import torch
    import torch.distributed as dist

    i = max(range(len(ys)), key=lambda k: ys[k].numel())
    y = ys[i]
    parts = [torch.empty_like(y) for _ in range(world)] if rank == 0 else None
    dist.gather(y, parts, dst=0)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dist.gather(y, parts, dst=0)
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b)], device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    nbytes = y.numel() * 4 * world
    return {"layer": cfgs[i].name, "bytes": nbytes, "ms": round(float(t.item()), 4),
            "gbs": round(nbytes / (float(t.item()) * 1e-3) / 1e9, 1), "collective": "dist.gather (NCCL) to rank 0"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2103_16234_b200 import workloads as W

    batch = args.batch or DEFAULT_BATCH[args.workload]
    strong = args.workload in STRONG
    per_rank = batch // world if strong else batch
    if strong and batch % world:
        raise SystemExit(f"--batch {batch} does not split over {world} GPUs")
    gcfgs = W.layers(args.workload, batch)          # the global layer (plans pinned to it)
    cfgs = W.layers(args.workload, per_rank)        # this rank's slab
    global_batch = per_rank * world
    metric = "fp32 conv GFLOP/s & us/layer (% of FP32/HBM roofline) at 1/2/4/8 B200 vs CPU ref"
    config = {"workload": f"{args.workload}: {W.DESCRIPTIONS[args.workload]}", "layers": len(cfgs),
              "global_batch": global_batch, "batch_per_gpu": per_rank, "engine": args.engine,
              "parallelism": f"batch-sharded dp{world} (filters replicated, no collective on the hot path)",
              "schedule": args.schedule + (" (inception branches / projection shortcuts concurrent, "
                                           "modules and blocks in order)" if args.schedule == "dataflow" else ""),
              "l2": "per-step working set > 126 MB L2 (each layer's operands evicted by the others between steps)"}

    if args.impl == "reference":
        reference_arm(args, cfgs, metric, config)
        return

    import torch
    import torch.distributed as dist
    from paper_2103_16234_b200 import _native as nat
    from paper_2103_16234_b200.sharding import shard_layer

    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    lib = nat.lib()

    # live FP32 roofline denominator (NVML sampled during the probe as a cross-check of its clock)
    tf, fpc, mhz = (nat.ctypes.c_double() for _ in range(3))
    with ClockSampler(local_rank) as probe_clk:
        nat.check(lib.b2c_probe_fp32_peak(4000, nat.ctypes.byref(tf), nat.ctypes.byref(fpc), nat.ctypes.byref(mhz)))
    peak_tflops = tf.value
    hbm = peaks().get("hbm_gbs", 6540.8)

    # every rank runs its slab with the order-relevant plan fields of the global
    # layer, so the outputs are bitwise those of the unsharded batch
    layers = [shard_layer(g, c, args.engine) for g, c in zip(gcfgs, cfgs)]
    xs, ws, ys = make_operands(cfgs, device, 1234 + rank)
    groups = W.schedule(args.workload, cfgs) if args.schedule == "dataflow" else None
    ms_total, launches_per_step, clk = time_graph(lib, layers, xs, ws, ys, args, world, device, local_rank, groups)
    flops_step_rank = sum(c.flops for c in cfgs)
    value = flops_step_rank * world * args.steps / (ms_total * 1e-3) / 1e9
    ms_per_step = ms_total / args.steps
    # per-layer device times inside a sequential pass of the same step -> roofline attribution
    layer_ms = time_layers_in_step(layers, xs, ws, ys, passes=args.layer_passes)
    kern_ms = sum(layer_ms)
    achieved_tflops = flops_step_rank / (kern_ms * 1e-3) / 1e12
    bytes_step = sum(c.compulsory_bytes for c in cfgs)
    per_layer = layer_rooflines(cfgs, layers, layer_ms, peak_tflops, hbm)
    dom = dominant_kernel(cfgs, layers, layer_ms, args.workload, peak_tflops, hbm)
    hbm_layers = [r for r in per_layer if r["bound"] == "hbm"]

    gather = time_gather(lib, cfgs, ys, world, rank, device) if world > 1 else None

    # e2e: host buffers through the C-ABI drop-in (H2D x,w + kernel + D2H y per layer)
    e2e = None
    if args.e2e_steps > 0:
        e2e_engine = args.engine if args.engine != "twostage" else "fused"
        e2e = e2e_run(lib, nat, cfgs, xs, ws, ys, nat.ENGINES[e2e_engine], args.e2e_steps, world, device,
                      local_rank)

    # the optional tensor-core variant (tcgen05 implicit GEMM), reported separately
    tc = None
    if args.tc_engine != "none" and args.engine not in ("tf32x3", "tf32"):
        tc = tensor_core_variant(args, lib, nat, cfgs, gcfgs, xs, ws, ys, world, device, local_rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample_batch = 1
        gflops, threads, passes = cpu_run(cfgs, sample_batch, 10.0)
        cpu = {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
               "sample": f"{passes} pass(es) over all {len(cfgs)} {args.workload} layers at N={sample_batch} "
                         f"(>= 10 s), oracle C port of convkit.conv_twostage (stage1+stage2, reference "
                         f"rounding; strided layers via the conv_naive port), {threads} threads",
               "host": host_info(), "convkit": convkit_legs(cfgs)}

    if args.report and rank == 0:
        sweep_report(args.report, device, peak_tflops)

    if rank == 0:
        dom_peak = peak_tflops if dom["bound"] == "fp32" else hbm
        dom_ach = dom["achieved_tflops"] if dom["bound"] == "fp32" else dom["achieved_gbs"]
        line = {"metric": metric, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
                "us_per_layer": round(1e3 * ms_per_step / len(cfgs), 3),
                "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic (uniform [-1,1) inputs and filters, torch RNG on device)",
                "config": config,
                "roofline": {"bound": dom["bound"], "achieved": round(dom_ach, 3), "peak": round(dom_peak, 3),
                             "unit": "TFLOP/s" if dom["bound"] == "fp32" else "GB/s",
                             "frac": round(dom_ach / dom_peak, 4), "traffic": dom["traffic"],
                             "kernel": dom["kernel"], "kernel_share_of_step": dom["share"],
                             "kernel_ms_per_step": round(dom["ms_per_step"], 4),
                             "launches_per_step": dom["launches"],
                             "algorithmic_flop_per_launch": dom["flop_per_launch"],
                             "algorithmic_bytes_per_launch": dom["bytes_per_launch"],
                             "traffic_source": dom["traffic_source"],
                             "timing": (f"CUDA events between the layers of {args.layer_passes} sequential "
                                        "passes of the step on the launching stream (time_layers_in_step)"),
                             "peak_source": ("b2c_probe_fp32_peak: FFMA2 register-blocked loop on all SMs, measured "
                                             f"live ({fpc.value:.1f} FMA/clk/SM at {mhz.value:.0f} MHz in-kernel; "
                                             f"NVML median {probe_clk.summary()['sm_mhz']} MHz)"
                                             if dom["bound"] == "fp32" else "MEASURED_PEAKS.json hbm_gbs"),
                             "frac_of_nominal_fp32_74.45": round(dom["achieved_tflops"] / NOMINAL_FP32_TFLOPS, 4),
                             "step": {"achieved": round(achieved_tflops, 3),
                                      "frac": round(achieved_tflops / peak_tflops, 4),
                                      "frac_of_nominal_74.45": round(achieved_tflops / NOMINAL_FP32_TFLOPS, 4),
                                      "graph_step_achieved": round(flops_step_rank / (ms_per_step * 1e-3) / 1e12, 3),
                                      "bytes_per_step": bytes_step,
                                      "hbm_frac": round(bytes_step / (kern_ms * 1e-3) / (hbm * 1e9), 4),
                                      "sequential_step_ms": round(kern_ms, 4)},
                             "hbm_bound_layers": hbm_layers},
                "e2e": e2e, "cpu_baseline": cpu, "clocks": clk.summary(),
                "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
                "gather": gather, "per_layer": per_layer, "tensor_core_variant": tc}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
