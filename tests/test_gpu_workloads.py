"""Parity of exactly what the benchmark executes: every layer of every
BASELINE workload at its bench batch, through the plans that ship.

For C1 (N=1), C2 (N=32), C3 (N=128), C4 (N=8 and N=128) and C5 (N=256):
* the ConvLayer the bench builds resolves to the shipped tuned_plans.json
  entry (the registry's resolution: the last entry per shape and engine);
* engine="fused" on the whole batch, checked on three seeded images (first,
  middle, last) against the per-image f64 oracle (conv_naive_f64,
  reference.py:86-103) under tol(K) = 1e-5*max(1, K/4096) — images are
  independent and the per-image oracle equals the batch slice bitwise
  (SURVEY §8(c)); a second run must be bitwise identical;
* engine="tf32x3" on the same operands and images under the same gate;
* at N=1, engine="twostage" on every stride-1 layer is bitwise equal to the
  oracle's conv_naive (reference.py:58-83; the reference's criterion 1,
  test_acceptance.py:90-110).

Anchors: /root/reference/pkg/tests/test_acceptance.py:90-110 (bitwise +
f64 criteria), /root/reference/pkg/src/convkit/bench.py:142-148 (per-config
validation of every benchmarked layer).
"""

from __future__ import annotations

import json

import numpy as np
import pytest

import paper_2103_16234_b200 as pk
from paper_2103_16234_b200 import workloads as W

pytestmark = pytest.mark.gpu

CASES = [("c1", 1), ("c2", 32), ("c3", 128), ("c4", 8), ("c4", 128), ("c5", 256)]


def _shipped():
    """(desc tuple, engine) -> the entry the registry resolves to (last wins)."""
    from paper_2103_16234_b200._native import TUNED_PATH

    out = {}
    for e in json.loads(TUNED_PATH.read_text())["plans"]:
        out[(tuple(e["desc"]), e["engine"])] = e
    return out


def _operands(cfg, seed):
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
    return x, w


def _check_plan(layer, cfg, engine, shipped, bad):
    e = shipped.get((cfg.as_tuple(), engine))
    if e is None:
        return
    if engine == "fused":
        got = (layer.family.replace("_dsm", ""), layer.splits, layer.reduce if layer.splits > 1 else 0)
        want = (e["family"], int(e.get("splits", 1)), int(e.get("reduce", 0)) if int(e.get("splits", 1)) > 1 else 0)
        if want[2] == 0 and want[1] > 1:
            want = (want[0], want[1], 1)  # planner default reduction for split plans
    else:
        t = layer._tc
        got = (t.mode, t.filters_per_tile, t.splits) + ((t.m_halves,) if e.get("mh") else ())
        want = (int(e["mode"]), int(e["nf"]), int(e["splits"])) + ((int(e["mh"]),) if e.get("mh") else ())
    if got != want:
        bad.append(f"{cfg.name} {engine}: plan {got} != shipped {want}")


@pytest.mark.parametrize("wl,n", CASES, ids=[f"{w}-N{n}" for w, n in CASES])
def test_every_bench_layer_fused_and_tf32x3_vs_f64_oracle(wl, n):
    import oracle
    import torch

    shipped = _shipped()
    threads = oracle.max_threads()
    bad, worst = [], {"fused": 0.0, "tf32x3": 0.0}
    for i, cfg in enumerate(W.layers(wl, n)):
        x, w = _operands(cfg, 1000 + i)
        one = cfg.with_batch(1)
        imgs = sorted({0, n // 2, n - 1})
        xs = {k: x[k:k + 1].cpu().numpy() for k in imgs}
        wn = w.cpu().numpy()
        refs = {k: oracle.conv_f64(one, xs[k], wn, threads=threads) for k in imgs}
        tol = oracle.fp32_tolerance(cfg.c, cfg.hf, cfg.wf)
        for engine in ("fused", "tf32x3"):
            layer = pk.ConvLayer(cfg, engine)
            _check_plan(layer, cfg, engine, shipped, bad)
            y = layer(x, w)
            y2 = layer(x, w)
            torch.cuda.synchronize()
            if not torch.equal(y, y2):
                bad.append(f"{cfg.name} {engine} ({layer.family}): not deterministic run to run")
            for k in imgs:
                err = oracle.relative_error(y[k:k + 1].cpu().numpy(), refs[k])
                worst[engine] = max(worst[engine], err)
                if not err <= tol:
                    bad.append(f"{cfg.name} {engine} ({layer.family}) image {k}: rel err {err:.3g} > {tol:.3g}")
            del y, y2
        del x, w
        torch.cuda.empty_cache()
    print(f"{wl} N={n}: worst relative error fused {worst['fused']:.3g}, tf32x3 {worst['tf32x3']:.3g}")
    assert not bad, "\n".join(bad)


@pytest.mark.parametrize("wl", ["c1", "c2", "c3", "c4", "c5"])
def test_every_stride1_layer_twostage_bitwise_at_batch1(wl):
    """The drop-in's default engine reproduces the reference's pinned fp32
    order exactly on every stride-1 layer of every workload."""
    import oracle

    threads = oracle.max_threads()
    bad = []
    for i, cfg in enumerate(W.layers(wl, 1)):
        if cfg.stride != 1:
            continue
        x = oracle.make_uniform(pk.input_dims(cfg), 2000 + 2 * i)
        w = oracle.make_uniform(pk.filter_dims(cfg), 2001 + 2 * i)
        out, stats = pk.conv_twostage(pk.Tensor4(x), pk.Tensor4(w), cfg)
        want = oracle.conv_naive(cfg, x, w, threads=threads)
        if out.data.tobytes() != want.tobytes():
            bad.append(f"{cfg.name}: max ulp {oracle.max_ulp_diff(out.data, want)}")
        assert stats.stage2_invoked == (cfg.hf * cfg.wf > 1)
    assert not bad, "\n".join(bad)


# --- planes beyond 2^16 pixels (exact magic division) -------------

BIG_PLANES = [
    pk.ConvConfig("big320-3x3", n=2, c=8, h=320, w=320, m=20, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("big512-3x3", n=2, c=8, h=512, w=512, m=16, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("big512-1x1s2", n=2, c=16, h=512, w=512, m=24, hf=1, wf=1, stride=2),
    pk.ConvConfig("big513-1x1", n=2, c=16, h=513, w=511, m=24, hf=1, wf=1),
]


@pytest.mark.parametrize("cfg", BIG_PLANES, ids=lambda c: c.name)
def test_large_planes_every_family(cfg):
    """Output planes of 102,400-262,144 pixels: every fused family and a
    split-C plan in both reduction modes against the f64 oracle, and the
    two-stage engine bitwise against conv_naive (stride 1)."""
    import oracle
    import torch

    xn = oracle.make_uniform(pk.input_dims(cfg), 31)
    wn = oracle.make_uniform(pk.filter_dims(cfg), 32)
    ref = oracle.conv_f64(cfg, xn, wn, threads=oracle.max_threads())
    tol = oracle.fp32_tolerance(cfg.c, cfg.hf, cfg.wf)
    x, w = torch.from_numpy(xn).cuda(), torch.from_numpy(wn).cuda()
    ran = 0
    for fam in pk.matching_families(cfg):
        for splits, reduce in ((1, 0), (2, 1), (2, 2)):
            try:
                layer = pk.ConvLayer(cfg, family=fam, splits=splits, reduce=reduce)
            except pk.InvalidPlan:
                continue
            y = layer(x, w).cpu().numpy()
            err = oracle.relative_error(y, ref)
            assert err <= tol, (layer.family, splits, reduce, err)
            ran += 1
    assert ran > 0
    if cfg.stride == 1:
        out, _ = pk.conv_twostage(pk.Tensor4(xn), pk.Tensor4(wn), cfg)
        assert out.data.tobytes() == oracle.conv_naive(cfg, xn, wn, threads=oracle.max_threads()).tobytes()


def test_misaligned_output_view_takes_the_scalar_stage2():
    """conv2d(..., out=buf[1:]) — a valid contiguous view at an odd float
    offset — must not reach the float4 stage-2 path."""
    import oracle
    import torch

    cfg = pk.ConvConfig("mis", n=2, c=64, h=14, w=14, m=32, hf=3, wf=3, pad_h=1, pad_w=1)
    xn = oracle.make_uniform(pk.input_dims(cfg), 5)
    wn = oracle.make_uniform(pk.filter_dims(cfg), 6)
    x, w = torch.from_numpy(xn).cuda(), torch.from_numpy(wn).cuda()
    numel = cfg.n * cfg.m * 14 * 14
    buf = torch.empty(numel + 1, device="cuda")
    out = buf[1:].view(cfg.n, cfg.m, 14, 14)
    assert out.data_ptr() % 16 != 0
    pk.ConvLayer(cfg, splits=4, reduce=1)(x, w, out=out)
    torch.cuda.synchronize()
    ref = oracle.conv_f64(cfg, xn, wn)
    assert oracle.relative_error(out.cpu().numpy(), ref) <= oracle.fp32_tolerance(cfg.c, 3, 3)
    # the paper-faithful engine's stage 2 on the same misaligned view: bitwise
    y2 = pk.conv2d(x, w, stride=1, padding=1, engine="twostage", out=out)
    torch.cuda.synchronize()
    assert y2.cpu().numpy().tobytes() == oracle.conv_naive(cfg, xn, wn).tobytes()
