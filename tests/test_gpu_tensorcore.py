"""Parity of the tensor-core engines (tcgen05 implicit GEMM) with the oracle.

Stated tolerances (BASELINE.json north star: "an optional
TF32/BF16 tcgen05 implicit-GEMM variant ... reported separately, with its own
stated tolerance"):

* engine="tf32x3" (3xTF32 operand splitting, main and correction terms in
  separate TMEM accumulators): the fp32 gate itself,
      relative_error vs conv_naive_f64 <= tol(K) = 1e-5 * max(1, K/4096)
* engine="tf32" (operands truncated to tf32 by the tensor core):
      relative_error vs conv_naive_f64 <= 5e-3
  and, tighter, within 2e-6 of the exact product of the tf32-truncated
  operands (the hardware truncates, it does not round).

Both engines are for finite data: a +/-inf operand makes the 3xTF32 correction
terms 0*inf = NaN (documented in DESIGN.md); NaN and the reference's
0*inf-over-padding rule are not asserted here (the fused / two-stage engines
keep them exactly, see test_gpu_parity.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import cfg_from

import paper_2103_16234_b200 as pk

pytestmark = pytest.mark.gpu

TF32_TOL = 5e-3
ENGINES = ("tf32x3", "tf32")


def tol(cfg, engine) -> float:
    import oracle

    return oracle.fp32_tolerance(cfg.c, cfg.hf, cfg.wf) if engine == "tf32x3" else TF32_TOL


def operands(rec):
    import oracle

    c = rec["cfg"]
    x = oracle.make_uniform((c["n"], c["c"], c["h"], c["w"]), rec["seed_in"])
    w = oracle.make_uniform((c["m"], c["c"], c["hf"], c["wf"]), rec["seed_f"])
    return cfg_from(c), pk.Tensor4(x), pk.Tensor4(w)


def trunc_tf32(a):
    return (np.asarray(a, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("corpus", ["corpus_2024", "corpus_general"])
def test_tensor_core_corpora_within_stated_tolerance(golden, corpus, engine):
    """The reference acceptance corpus (seed 2024, 200 configs incl. 1x1/3x3/5x5,
    C up to 64) and the stride / asymmetric-pad / even-filter corpus, through
    the host-buffer drop-in (conv_twostage's operand contract)."""
    import oracle

    worst = 0.0
    for rec in golden[corpus]:
        cfg, x, w = operands(rec)
        got = pk.conv_forward(x, w, cfg, engine=engine).data
        ref = oracle.conv_f64(cfg, x.data, w.data)
        err = oracle.relative_error(got, ref)
        worst = max(worst, err)
        assert err <= tol(cfg, engine), (cfg, err)
    print(f"{engine} {corpus}: worst relative error {worst:.3g}")


@pytest.mark.parametrize("engine", ENGINES)
def test_tensor_core_baseline_layers(golden, engine):
    import oracle

    for rec in golden["baseline_layers"]:
        cfg, x, w = operands(rec)
        got = pk.conv_forward(x, w, cfg, engine=engine).data
        ref = oracle.conv_f64(cfg, x.data, w.data)
        assert oracle.relative_error(got, ref) <= tol(cfg, engine), (cfg.name, cfg.n)


def test_tf32_is_exact_product_of_truncated_operands(golden):
    """engine='tf32' computes the truncated-operand convolution (up to fp32
    accumulation), i.e. the tensor core truncates fp32 -> tf32."""
    import oracle

    for rec in golden["corpus_general"][:40]:
        cfg, x, w = operands(rec)
        got = pk.conv_forward(x, w, cfg, engine="tf32").data
        ref = oracle.conv_f64(cfg, trunc_tf32(x.data), trunc_tf32(w.data))
        assert oracle.relative_error(got, ref) <= 2e-6, cfg


TC_CASES = [
    pk.ConvConfig("deepK", n=2, c=520, h=9, w=9, m=72, hf=3, wf=3, pad_h=1, pad_w=1),  # K = 4680
    pk.ConvConfig("wideM", n=1, c=48, h=10, w=12, m=300, hf=1, wf=1),                  # 2 filter tiles
    pk.ConvConfig("w7", n=5, c=64, h=7, w=7, m=80, hf=3, wf=3, pad_h=1, pad_w=1),        # 4x8 chunks
    pk.ConvConfig("w14", n=3, c=40, h=14, w=14, m=48, hf=5, wf=5, pad_h=2, pad_w=2),     # 2x16 chunks
    pk.ConvConfig("w27", n=2, c=24, h=27, w=27, m=40, hf=5, wf=5, pad_h=2, pad_w=2),
    pk.ConvConfig("s2", n=2, c=32, h=15, w=15, m=48, hf=3, wf=3, stride=2, pad_h=1, pad_w=1),
    pk.ConvConfig("c7s2", n=1, c=3, h=40, w=38, m=64, hf=7, wf=7, stride=2, pad_h=3, pad_w=3),
    pk.ConvConfig("1x1s2", n=2, c=64, h=14, w=14, m=96, hf=1, wf=1, stride=2),
    pk.ConvConfig("even", n=2, c=9, h=9, w=10, m=17, hf=2, wf=4, pad_h=1, pad_w=2),
    pk.ConvConfig("flatodd", n=8, c=33, h=7, w=7, m=50, hf=1, wf=1),                     # H*W = 49
    pk.ConvConfig("one", n=1, c=1, h=1, w=1, m=1, hf=1, wf=1),
    pk.ConvConfig("bigpad", n=1, c=2, h=3, w=4, m=3, hf=3, wf=3, pad_h=4, pad_w=5),
    pk.ConvConfig("manyimg", n=300, c=4, h=3, w=3, m=17, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("stride3", n=2, c=6, h=17, w=13, m=9, hf=3, wf=3, stride=3),
]


def _torch_ops(cfg, seed=0):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
    return x, w


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("cfg", TC_CASES, ids=lambda c: c.name)
def test_tensor_core_shapes_deterministic(cfg, engine):
    import oracle

    x, w = _torch_ops(cfg, 3)
    layer = pk.ConvLayer(cfg, engine)
    a = layer(x, w).cpu().numpy()
    b = layer(x, w).cpu().numpy()
    assert a.tobytes() == b.tobytes(), "not deterministic run to run"
    ref = oracle.conv_f64(cfg, x.cpu().numpy(), w.cpu().numpy())
    assert oracle.relative_error(a, ref) <= tol(cfg, engine), (layer.family, oracle.relative_error(a, ref))


@pytest.mark.parametrize("engine", ENGINES)
def test_tensor_core_forced_filter_tiles_agree(engine):
    """Every filters-per-tile choice gives the same bits: each output's
    accumulation order depends only on (c, hf, wf), never on the tile plan."""
    cfg = pk.ConvConfig("tiles", n=2, c=40, h=12, w=12, m=96, hf=3, wf=3, pad_h=1, pad_w=1)
    x, w = _torch_ops(cfg, 5)
    outs = {nf: pk.ConvLayer(cfg, engine, filters_per_tile=nf, splits=1)(x, w).cpu().numpy() for nf in (16, 32, 48, 96)}
    first = outs[16]
    assert all(v.tobytes() == first.tobytes() for v in outs.values())


@pytest.mark.parametrize("engine", ENGINES)
def test_tensor_core_split_k_within_tolerance_and_deterministic(engine):
    import oracle

    cfg = pk.ConvConfig("splitk", n=2, c=96, h=10, w=10, m=40, hf=3, wf=3, pad_h=1, pad_w=1)
    x, w = _torch_ops(cfg, 6)
    ref = oracle.conv_f64(cfg, x.cpu().numpy(), w.cpu().numpy())
    for sp in (1, 2, 3, 5, 54):
        layer = pk.ConvLayer(cfg, engine, splits=sp)
        a = layer(x, w).cpu().numpy()
        assert a.tobytes() == layer(x, w).cpu().numpy().tobytes()
        assert oracle.relative_error(a, ref) <= tol(cfg, engine), (sp, layer.family)


@pytest.mark.parametrize("wl,name", [("c4", "vgg4_2"), ("c5", "layer3.1.conv2"), ("c3", "alexnet-conv2"), ("c5", "layer1.0.conv2"),
                                     ("c2", "4e-1x1"), ("c5", "conv1")])
def test_tensor_core_full_size_layers_sampled_images(wl, name):
    """BASELINE full sizes, checked on a seeded sample of images (images are
    independent: the per-image oracle pins the batch)."""
    import oracle
    import torch
    from paper_2103_16234_b200 import workloads as W

    n = {"c5": 256, "c4": 8, "c3": 128, "c2": 32}[wl]
    cfg = next(c for c in W.layers(wl, n) if c.name == name)
    x, w = _torch_ops(cfg, 11)
    y = pk.conv2d(x, w, stride=cfg.stride, padding=(cfg.pad_h, cfg.pad_w), engine="tf32x3")
    one = cfg.with_batch(1)
    wn = w.cpu().numpy()
    for img in (0, n // 2, n - 1):
        ref = oracle.conv_f64(one, x[img:img + 1].cpu().numpy(), wn)
        assert oracle.relative_error(y[img:img + 1].cpu().numpy(), ref) <= tol(cfg, "tf32x3"), img
    torch.cuda.synchronize()


def test_tensor_core_graph_capture_and_c_abi_plan():
    import torch

    cfg = pk.ConvConfig("g", n=8, c=64, h=14, w=14, m=96, hf=3, wf=3, pad_h=1, pad_w=1)
    x, w = _torch_ops(cfg, 9)
    layer = pk.ConvLayer(cfg, "tf32x3")
    assert layer.grid > 0 and layer.workspace_bytes > 0 and "tf32x3" in layer.family
    y = layer(x, w)
    want = y.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        layer(x, w, out=y)  # allocate the workspace outside capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            layer(x, w, out=y)
    y.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)


@pytest.mark.parametrize("engine", ("fused", "tf32x3"))
def test_pipelined_host_layers_match_single_calls(engine):
    """b2c_conv_host_layers (H2D / compute / D2H of consecutive layers
    overlapped) returns exactly what one conv_forward call per layer does."""
    cfgs = [pk.ConvConfig(f"l{i}", n=2, c=c, h=h, w=h, m=m, hf=f, wf=f, pad_h=f // 2, pad_w=f // 2, stride=s)
            for i, (c, h, m, f, s) in enumerate([(16, 14, 24, 3, 1), (24, 7, 40, 1, 1), (40, 9, 8, 5, 1),
                                                 (8, 15, 16, 3, 2), (16, 28, 32, 1, 1)])]
    layers = [(pk.make_tensor(pk.input_dims(c), "uniform", seed=10 + i),
               pk.make_tensor(pk.filter_dims(c), "uniform", seed=20 + i), c) for i, c in enumerate(cfgs)]
    outs = pk.conv_forward_layers(layers, engine=engine)
    for (x, w, c), o in zip(layers, outs):
        assert o.data.tobytes() == pk.conv_forward(x, w, c, engine=engine).data.tobytes(), c.name


def test_harness_run_bench_validates_every_engine(tmp_path):
    from paper_2103_16234_b200 import harness as H

    cfgs = pk.preset_configs()[:3] + pk.preset_configs()[-2:]
    recs = H.run_bench(cfgs, ("fused", "twostage", "tf32x3", "tf32"), (1, 2), repeats=3)
    assert len(recs) == len(cfgs) * 2 * 4
    assert all(r.validated for r in recs if not r.skipped), [(r.config, r.algorithm, r.max_rel_error) for r in recs]
    assert all(r.max_rel_error == 0.0 for r in recs if r.algorithm == "twostage")  # it is the reference
    H.emit_report(recs, tmp_path / "r.csv")
    H.emit_report(recs, tmp_path / "r.md", "md")
    assert (tmp_path / "r.csv").read_text().count("\n") == len(recs) + 1


def test_harness_cli_validate_and_run(tmp_path, capsys):
    """``validate`` / ``run`` subcommands (reference cli.py:123-145): exit 0, one ok line per run."""
    from paper_2103_16234_b200 import harness as H

    assert H.main(["validate", "--algos", "fused,twostage,tf32x3", "--batches", "1"]) == 0
    out = capsys.readouterr().out
    assert out.count("ok   ") == len(pk.preset_configs()) * 3 and "FAIL" not in out
    rep = tmp_path / "r.csv"
    assert H.main(["run", "--algos", "fused,tf32", "--batches", "2", "--repeats", "2", "--baseline", "fused",
                   "--out", str(rep)]) == 0
    assert rep.read_text().count("\n") == len(pk.preset_configs()) * 2 + 1


def test_bench_line_contract_on_gpu():
    """bench.py (our arm) prints one JSON line with every contract key: device
    value, e2e through the C ABI with host buffers, the dominant-kernel
    roofline, clocks sampled during the timed region, our kernel launches."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "bench.py", "--workload", "c1", "--steps", "3", "--warmup", "3",
                        "--e2e-steps", "1", "--no-cpu-baseline"], cwd=root, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    rf = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= rf.keys()
    assert 0 < rf["frac"] < 1.5 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["gpu_launches"] >= d["steps"]
