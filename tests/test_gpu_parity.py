"""Parity of the CUDA engine with the reference, through the C ABI.

* engine="twostage" (paper-faithful stage 1 + stage 2) must be BITWISE equal
  to the reference's own conv_twostage/conv_naive outputs (sha256 fixtures
  made by importing the reference, tests/golden/make_golden.py), NaN-aware on
  the special-value cases.
* engine="fused" (FFMA2, split-C) must be within
      tol(K) = 1e-5 * max(1, K/4096),  K = c*hf*wf
  of conv_naive_f64 (relative_error, reference.py:254-271) and within the
  reference harness's own 1e-4 (bench.py:30-35), for every kernel family and
  reduction split that can run the layer, deterministic run to run.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import cfg_from

import paper_2103_16234_b200 as pk


pytestmark = pytest.mark.gpu


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def operands(rec):
    import oracle

    c = rec["cfg"]
    x = oracle.make_uniform((c["n"], c["c"], c["h"], c["w"]), rec["seed_in"])
    w = oracle.make_uniform((c["m"], c["c"], c["hf"], c["wf"]), rec["seed_f"])
    return cfg_from(c), pk.Tensor4(x), pk.Tensor4(w)


def tol(cfg) -> float:
    import oracle

    return oracle.fp32_tolerance(cfg.c, cfg.hf, cfg.wf)


# --- paper-faithful two-stage engine: bitwise ---------------------------------

def test_twostage_bitwise_vs_reference_corpus(golden):
    bad = []
    for rec in golden["corpus_2024"]:
        cfg, x, w = operands(rec)
        out, stats = pk.conv_twostage(x, w, cfg)
        if sha(out.data) != rec["twostage"]:
            bad.append(cfg.name)
        assert stats.workspace_bytes == rec["stats"]["workspace_bytes"]
        assert stats.stage1_tasks_run == rec["stats"]["stage1_tasks_run"]
        assert stats.stage2_invoked == rec["stats"]["stage2_invoked"]
    assert not bad, f"{len(bad)} configs differ from the reference: {bad[:10]}"


def test_twostage_bitwise_vs_reference_presets_and_layers(golden):
    for rec in golden["presets"] + [r for r in golden["baseline_layers"] if "twostage" in r]:
        cfg, x, w = operands(rec)
        out, stats = pk.conv_twostage(x, w, cfg, workspace_limit=1 << 40)
        assert sha(out.data) == rec["twostage"], cfg.name
        assert stats.filter_row_global_loads == rec["stats"]["filter_row_global_loads"]


def test_twostage_special_values(golden, special_arrays):
    for i, c in enumerate(golden["special_values"]):
        cfg = cfg_from(c)
        x, w = special_arrays[f"sv{i}_x"], special_arrays[f"sv{i}_w"]
        want = special_arrays[f"sv{i}_twostage"]
        got, _ = pk.conv_twostage(pk.Tensor4(x), pk.Tensor4(w), cfg)
        assert np.array_equal(np.isnan(got.data), np.isnan(want)), cfg.name
        m = ~np.isnan(want)
        assert got.data[m].tobytes() == want[m].tobytes(), cfg.name


def test_stage1_and_stage2_bitwise_vs_oracle(golden):
    import oracle

    for rec in golden["corpus_2024"][:60]:
        cfg, x, w = operands(rec)
        parts, st1 = pk.stage1_scalar_prods(x, w, cfg)
        want = oracle.stage1(cfg, x.data, w.data)
        assert parts.data.tobytes() == want.tobytes(), cfg.name
        assert st1.stage1_tasks_run == pk.plan_launch(cfg).blocks and not st1.stage2_invoked
        out, st2 = pk.stage2_sum(parts, cfg)
        assert sha(out.data) == rec["twostage"] and st2.stage2_invoked


def test_reference_known_answers_on_gpu():
    # test_twostage.py:95-104, 128-139, 169-175
    cfg = pk.ConvConfig("t", n=1, c=2, h=1, w=1, m=1, hf=1, wf=1)
    parts, stats = pk.stage1_scalar_prods(pk.Tensor4(np.array([3, 4], np.float32).reshape(1, 2, 1, 1)),
                                          pk.Tensor4(np.array([0.5, 0.25], np.float32).reshape(1, 2, 1, 1)), cfg)
    assert parts.data[0, 0, 0, 0, 0] == 2.5 and stats.stage1_tasks_run == 1
    cfg3 = pk.ConvConfig("t", n=1, c=1, h=3, w=3, m=1, hf=3, wf=3, pad_h=1, pad_w=1)
    one = pk.make_tensor((1, 1, 3, 3), "constant", value=1.0)
    parts, _ = pk.stage1_scalar_prods(one, one, cfg3)
    assert parts.data[0, 0, 0].tolist() == [[0, 0, 0], [0, 1, 1], [0, 1, 1]]
    assert parts.data[4, 0, 0].tolist() == [[1, 1, 1]] * 3
    cfg2 = pk.ConvConfig("t", n=1, c=1, h=2, w=2, m=1, hf=2, wf=2)
    p = np.zeros((4, 1, 1, 1, 1), np.float32)
    p[:, 0, 0, 0, 0] = [1, 2, 4, 8]
    out, _ = pk.stage2_sum(pk.PartialSums(p), cfg2)
    assert out.data[0, 0, 0, 0] == 15.0


# --- fused engine: tolerance ----------------------------------------------------

@pytest.mark.parametrize("corpus", ["corpus_2024", "corpus_general"])
def test_fused_within_tolerance(golden, corpus):
    import oracle

    worst = 0.0
    for rec in golden[corpus]:
        cfg, x, w = operands(rec)
        got = pk.conv_forward(x, w, cfg).data
        ref = oracle.conv_f64(cfg, x.data, w.data)
        assert sha(ref) == rec["f64"]  # the checker itself is the reference's oracle
        err = oracle.relative_error(got, ref)
        worst = max(worst, err)
        assert err <= tol(cfg) and err <= 1e-4, (cfg.name, err)
    print(f"{corpus}: worst relative error {worst:.3g}")


def test_fused_baseline_layers(golden):
    import oracle

    for rec in golden["baseline_layers"]:
        cfg, x, w = operands(rec)
        got = pk.conv_forward(x, w, cfg).data
        ref = oracle.conv_f64(cfg, x.data, w.data)
        assert oracle.relative_error(got, ref) <= tol(cfg), (cfg.name, cfg.n)


def test_fused_special_values_nan_positions():
    """Non-finite propagation (0*inf over padding, inf-inf, nan) lands on the
    same outputs as the reference order.  Finite values are kept far from
    overflow: near FLT_MAX, whether a partial sum overflows depends on the
    summation order, which the fused engine does not share (the two-stage
    engine, which does, is checked bitwise on such cases above)."""
    import oracle

    rng = np.random.default_rng(77)
    specials = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, 1e-40], np.float32)
    for i in range(12):
        f = int(rng.choice((1, 3, 5)))
        p = int(rng.integers(0, f))
        cfg = pk.ConvConfig(f"fs{i}", n=int(rng.integers(1, 3)), c=int(rng.integers(1, 20)),
                            h=int(rng.integers(f, 12)), w=int(rng.integers(f, 12)), m=int(rng.integers(1, 40)),
                            hf=f, wf=f, pad_h=p, pad_w=p)
        x = rng.uniform(-2, 2, pk.input_dims(cfg)).astype(np.float32)
        w = rng.uniform(-2, 2, pk.filter_dims(cfg)).astype(np.float32)
        kx, kw = rng.random(x.shape) < 0.03, rng.random(w.shape) < 0.03
        x[kx] = rng.choice(specials, int(kx.sum()))
        w[kw] = rng.choice(specials, int(kw.sum()))
        want = oracle.conv_naive(cfg, x, w)
        got = pk.conv_forward(pk.Tensor4(x), pk.Tensor4(w), cfg).data
        assert np.array_equal(np.isnan(got), np.isnan(want)), cfg
        inf = np.isinf(want)
        assert np.array_equal(np.isinf(got), inf) and np.array_equal(np.sign(got[inf]), np.sign(want[inf]))


def _torch_ops(cfg, seed=0):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
    return x, w


PLAN_CASES = [
    pk.ConvConfig("p3", n=3, c=37, h=14, w=14, m=40, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("p1", n=5, c=70, h=7, w=7, m=50, hf=1, wf=1),
    pk.ConvConfig("p1s2", n=3, c=40, h=14, w=13, m=36, hf=1, wf=1, stride=2),
    pk.ConvConfig("p5", n=2, c=20, h=13, w=11, m=33, hf=5, wf=5, pad_h=2, pad_w=2),
    pk.ConvConfig("ps2", n=2, c=24, h=15, w=15, m=20, hf=3, wf=3, stride=2, pad_h=1, pad_w=1),
    pk.ConvConfig("p7", n=2, c=3, h=30, w=30, m=20, hf=7, wf=7, stride=2, pad_h=3, pad_w=3),
    pk.ConvConfig("pe", n=2, c=9, h=9, w=10, m=17, hf=2, wf=4, pad_h=1, pad_w=2),
    # pointwise with H*W % 4 == 0: 16-byte, persistent and TMA-fed families (tiles across images)
    pk.ConvConfig("p1v", n=3, c=72, h=16, w=16, m=100, hf=1, wf=1),
    # pointwise on 7x7 planes with C % 4 == 0: whole-image tiles by bulk copy (partial last tile)
    pk.ConvConfig("p1img", n=7, c=48, h=7, w=7, m=80, hf=1, wf=1),
]


@pytest.mark.parametrize("cfg", PLAN_CASES, ids=lambda c: c.name)
def test_every_family_and_split_within_tolerance_and_deterministic(cfg):
    import oracle
    import torch

    x, w = _torch_ops(cfg)
    ref = oracle.conv_f64(cfg, x.cpu().numpy(), w.cpu().numpy())
    unsplit = {}
    for fam in pk.matching_families(cfg):
        for splits in (1, 2, 3):
            try:
                layer = pk.ConvLayer(cfg, family=fam, splits=splits)
            except pk.InvalidPlan:
                continue
            a = layer(x, w).cpu().numpy()
            b = layer(x, w).cpu().numpy()
            assert a.tobytes() == b.tobytes(), "not deterministic"
            assert oracle.relative_error(a, ref) <= tol(cfg), (layer.family, splits)
            if layer.splits == 1:
                unsplit[layer.family] = a
    # unsplit plans share the per-output order: bitwise identical across families
    vals = list(unsplit.values())
    assert vals and all(v.tobytes() == vals[0].tobytes() for v in vals), list(unsplit)
    torch.cuda.synchronize()


def test_torch_conv2d_matches_oracle_and_rejects_bad_tensors():
    import oracle
    import torch

    for cfg in PLAN_CASES:
        x, w = _torch_ops(cfg, 3)
        y = pk.conv2d(x, w, stride=cfg.stride, padding=(cfg.pad_h, cfg.pad_w))
        ref = oracle.conv_f64(cfg, x.cpu().numpy(), w.cpu().numpy())
        assert oracle.relative_error(y.cpu().numpy(), ref) <= tol(cfg)
        if cfg.stride == 1:
            y2 = pk.conv2d(x, w, stride=1, padding=(cfg.pad_h, cfg.pad_w), engine="twostage")
            assert y2.cpu().numpy().tobytes() == oracle.conv_naive(cfg, x.cpu().numpy(), w.cpu().numpy()).tobytes()
    with pytest.raises(pk.ShapeMismatch):
        pk.conv2d(torch.zeros(1, 1, 3, 3), torch.zeros(1, 1, 1, 1))
    with pytest.raises(pk.ShapeMismatch):
        pk.conv2d(torch.zeros(1, 2, 3, 3, device="cuda"), torch.zeros(1, 1, 1, 1, device="cuda"))
    with pytest.raises(pk.ShapeMismatch):
        pk.conv2d(torch.zeros(1, 1, 3, 3, device="cuda", dtype=torch.float64), torch.zeros(1, 1, 1, 1, device="cuda"))


EDGE_CASES = [
    pk.ConvConfig("one", n=1, c=1, h=1, w=1, m=1, hf=1, wf=1),
    pk.ConvConfig("padonly", n=2, c=3, h=1, w=1, m=5, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("bigpad", n=1, c=2, h=3, w=4, m=3, hf=3, wf=3, pad_h=4, pad_w=5),
    pk.ConvConfig("wide", n=1, c=5, h=2, w=300, m=7, hf=1, wf=5, pad_w=2),
    pk.ConvConfig("tall", n=1, c=5, h=300, w=2, m=7, hf=5, wf=1, pad_h=2),
    pk.ConvConfig("m1", n=4, c=33, h=6, w=6, m=1, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("manyimg", n=300, c=4, h=3, w=3, m=17, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("stride3", n=2, c=6, h=17, w=13, m=9, hf=3, wf=3, stride=3),
    pk.ConvConfig("c129", n=1, c=129, h=9, w=9, m=130, hf=1, wf=1),
]


@pytest.mark.parametrize("cfg", EDGE_CASES, ids=lambda c: c.name)
def test_edge_cases(cfg):
    import oracle

    x = pk.make_tensor(pk.input_dims(cfg), "uniform", seed=5)
    w = pk.make_tensor(pk.filter_dims(cfg), "uniform", seed=6)
    got = pk.conv_forward(x, w, cfg).data
    ref = oracle.conv_f64(cfg, x.data, w.data)
    assert oracle.relative_error(got, ref) <= tol(cfg)
    if cfg.stride == 1:
        out, _ = pk.conv_twostage(x, w, cfg)
        assert out.data.tobytes() == oracle.conv_naive(cfg, x.data, w.data).tobytes()


def test_cuda_graph_capture_and_replay():
    import torch

    cfg = pk.ConvConfig("g", n=8, c=64, h=14, w=14, m=96, hf=3, wf=3, pad_h=1, pad_w=1)
    x, w = _torch_ops(cfg, 9)
    layer = pk.ConvLayer(cfg)
    y = layer(x, w)
    want = y.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            layer(x, w, out=y)
    y.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)


@pytest.mark.parametrize("wl,name", [("c5", "layer1.0.conv2"), ("c5", "layer4.0.downsample"), ("c5", "conv1"),
                                     ("c4", "vgg1_2"), ("c2", "5b-1x1")])
def test_full_size_layers_sampled_images(wl, name):
    """BASELINE full sizes: images are independent, so the per-image oracle on
    a seeded sample of images pins the whole batch."""
    import oracle
    import torch
    from paper_2103_16234_b200 import workloads as W

    n = {"c5": 256, "c4": 32, "c2": 32}[wl]
    cfg = next(c for c in W.layers(wl, n) if c.name == name)
    x, w = _torch_ops(cfg, 11)
    y = pk.conv2d(x, w, stride=cfg.stride, padding=(cfg.pad_h, cfg.pad_w))
    one = cfg.with_batch(1)
    wn = w.cpu().numpy()
    for img in (0, n // 2, n - 1):
        ref = oracle.conv_f64(one, x[img:img + 1].cpu().numpy(), wn)
        assert oracle.relative_error(y[img:img + 1].cpu().numpy(), ref) <= tol(cfg), img
    torch.cuda.synchronize()


CLUSTER_CASES = PLAN_CASES[:5] + [
    pk.ConvConfig("c1x1big", n=2, c=512, h=14, w=14, m=130, hf=1, wf=1),
    pk.ConvConfig("c3big", n=1, c=256, h=28, w=28, m=70, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("c1x1odd", n=3, c=300, h=7, w=7, m=64, hf=1, wf=1),
    # row-segment kernels park a [BM][SEG*7] tile behind their halo tables (Wo % 7 == 0)
    pk.ConvConfig("c3s2", n=2, c=40, h=28, w=28, m=130, hf=3, wf=3, stride=2, pad_h=1, pad_w=1),
    pk.ConvConfig("c5x5", n=2, c=24, h=14, w=14, m=70, hf=5, wf=5, pad_h=2, pad_w=2),
]


@pytest.mark.parametrize("cfg", CLUSTER_CASES, ids=lambda c: c.name)
def test_cluster_split_reduction_bitwise_equals_partial_planes(cfg):
    """Split-C through DSMEM clusters (reduce=2) against partial planes +
    stage2_sum (reduce=1): the same ascending-order sum, so the outputs are
    bitwise identical for every family and split count; the cluster path is
    one kernel, the planes path two."""
    import torch
    from paper_2103_16234_b200 import _native as nat

    x, w = _torch_ops(cfg, seed=7)
    n = 0
    for fam in pk.matching_families(cfg):
        for splits in (2, 3, 5, 8, 12, 16):
            try:
                planes = pk.ConvLayer(cfg, family=fam, splits=splits, reduce=1)
                dsm = pk.ConvLayer(cfg, family=fam, splits=splits, reduce=2)
            except pk.InvalidPlan:
                continue
            if planes.splits != splits:
                continue
            assert dsm.reduce == 2 and dsm.family.endswith("_dsm") and planes.reduce == 1
            a = planes(x, w)
            nat.lib().b2c_reset_launch_count()
            b = dsm(x, w)
            assert nat.lib().b2c_launch_count() == 1
            torch.cuda.synchronize()
            assert a.cpu().numpy().tobytes() == b.cpu().numpy().tobytes(), (dsm.family, splits)
            n += 1
    assert n > 0


@pytest.mark.parametrize("cfg", [
    pk.ConvConfig("pk7", n=5, c=40, h=7, w=7, m=72, hf=1, wf=1),                  # H*W % 4 != 0
    pk.ConvConfig("pks2", n=3, c=24, h=14, w=14, m=40, hf=1, wf=1, stride=2),     # projection shortcut
    pk.ConvConfig("pks2odd", n=2, c=20, h=15, w=13, m=33, hf=1, wf=1, stride=2),  # ragged Q, M tail
], ids=lambda c: c.name)
def test_packed_pointwise_through_c_abi(cfg):
    """Packed-pixel pointwise families (kind 9) through b2c_conv2d_forward: the
    plan's workspace holds the gathered pixels (+ partial planes when split);
    a forced packed plan without it fails with B2C_INVALID_ARGUMENT; results
    are bitwise those of the 4-byte-staged family with the same split ranges
    and within tol(K) of the f64 oracle."""
    import ctypes

    import oracle
    import torch

    from paper_2103_16234_b200 import _native as nat

    lib = nat.lib()
    names = pk.family_names()
    fams = [f for f in pk.matching_families(cfg) if "_1x1pk" in names[f]]
    ref_fam = next(f for f in pk.matching_families(cfg) if names[f] == "fused_1x1s_m64")
    assert fams
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
    ref = oracle.conv_f64(cfg, x.cpu().numpy(), w.cpu().numpy())
    d = nat.desc(cfg)
    stream = torch.cuda.current_stream().cuda_stream
    for splits in (1, 2):
        base = pk.ConvLayer(cfg, family=ref_fam, splits=splits, reduce=1)(x, w)
        for f in fams:
            plan = nat.TilePlanC()
            plan.family, plan.splits, plan.reduce = f, splits, 1
            if lib.b2c_select_tiles(ctypes.byref(d), nat.ENGINE_FUSED, ctypes.byref(plan)) != nat.OK:
                assert splits > -(-cfg.c // 32)  # only a 32-channel chunk family can lack a second range
                continue
            assert plan.workspace_bytes >= 4 * cfg.c * cfg.n * ((cfg.h - 1) // cfg.stride + 1) * \
                ((cfg.w - 1) // cfg.stride + 1)
            y = torch.full(base.shape, float("nan"), device="cuda")
            assert lib.b2c_conv2d_forward(ctypes.byref(d), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                          ctypes.c_void_p(y.data_ptr()), None, 0, ctypes.byref(plan),
                                          ctypes.c_void_p(stream)) == nat.INVALID_ARGUMENT
            ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
            assert lib.b2c_conv2d_forward(ctypes.byref(d), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                          ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                          plan.workspace_bytes, ctypes.byref(plan), ctypes.c_void_p(stream)) == nat.OK
            torch.cuda.synchronize()
            assert oracle.relative_error(y.cpu().numpy(), ref) <= oracle.fp32_tolerance(cfg.c, 1, 1)
            def first_bound(bc):  # end of the first split channel range
                return min(cfg.c, -(-(-(-cfg.c // bc)) // splits) * bc)

            if splits == 1 or first_bound(plan.bc) == first_bound(16):  # same ranges as the 16-channel reference
                assert torch.equal(y, base), (names[f], splits)
