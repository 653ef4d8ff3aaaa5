"""The drop-in boundary without a GPU: the C ABI library loads and exports
every symbol include/b2conv.h declares; shape/plan/precondition logic matches
the reference (golden fixtures + the reference tests' expectations); errors
surface as the reference's exception classes in the reference's order.  No
test here launches a kernel."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, cfg_from

import paper_2103_16234_b200 as pk
from paper_2103_16234_b200 import _native as nat


def header_symbols() -> list[str]:
    text = (ROOT / "include" / "b2conv.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(b2c_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(native):
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(native, s)]
    assert not missing, missing


def test_binding_covers_header(native):
    assert set(header_symbols()) == set(nat.SIGNATURES)


def test_abi_version(native):
    assert native.b2c_abi_version() == 1


def test_families_enumerable(native):
    names = pk.family_names()
    assert len(names) == native.b2c_num_families() >= 10
    assert any(n.startswith("fused_3x3") for n in names) and any(n.startswith("stage1_strict") for n in names)


# --- configs ------------------------------------------------------------------

@pytest.mark.parametrize("field,kwargs", [
    ("n", dict(n=0)), ("c", dict(c=-1)), ("stride", dict(stride=0)), ("pad_h", dict(pad_h=-1)),
    ("hf", dict(hf=9, h=3, pad_h=1)), ("wf", dict(wf=6, w=2, pad_w=1)),
])
def test_config_validation_names_field(field, kwargs):
    base = dict(name="t", n=1, c=1, h=5, w=5, m=1, hf=3, wf=3, stride=1, pad_h=0, pad_w=0)
    base.update(kwargs)
    with pytest.raises(pk.InvalidConfig) as exc:
        pk.ConvConfig(**base)
    assert exc.value.field == field


def test_c_abi_config_validation_agrees(native):
    d = nat.ConvDesc(1, 1, 3, 3, 1, 5, 3, 1, 0, 0)  # hf > h + 2*pad_h
    bad = ctypes.c_int32(-1)
    assert native.b2c_validate_config(ctypes.byref(d), ctypes.byref(bad)) == nat.INVALID_CONFIG
    assert bad.value == 5
    with pytest.raises(pk.InvalidConfig) as exc:
        nat.check(native.b2c_validate_config(ctypes.byref(d), None))
    assert exc.value.field == "hf"


def test_output_dims_and_presets():
    cfg = pk.ConvConfig("t", n=1, c=1, h=224, w=224, m=1, hf=7, wf=7, stride=2, pad_h=3, pad_w=3)
    assert pk.output_dims(cfg) == (112, 112)
    names = [c.name for c in pk.preset_configs()]
    assert names == ["1x1-A", "1x1-B", "1x1-C", "3x3-A", "3x3-B", "5x5-A", "5x5-B"]
    assert pk.same_padding(5, 5) == (2, 2)
    with pytest.raises(pk.UnsupportedFilter):
        pk.same_padding(2, 3)


def test_parse_config_file(tmp_path):
    p = tmp_path / "layers.csv"
    p.write_text("# comment\nc1, 1, 64, 56, 56, 64, 3, 3, 1, 1, 1\n\nx,2,3,4,5,6,1,1,1,0,0 # tail\n")
    cfgs = pk.parse_config_file(p)
    assert [c.name for c in cfgs] == ["c1", "x"] and cfgs[0].pad_w == 1
    p.write_text("bad,1,2\n")
    with pytest.raises(pk.ParseError) as exc:
        pk.parse_config_file(p)
    assert exc.value.line_no == 1
    p.write_text("ok,1,1,1,1,1,1,1,1,0,0\nz,1,1,1,1,1,3,1,1,0,0\n")
    with pytest.raises(pk.InvalidConfig) as exc:
        pk.parse_config_file(p)
    assert exc.value.field == "hf"


def test_tensor_file_round_trip_preserves_bits(tmp_path):
    data = np.array([np.nan, -0.0, np.inf, 1e-42, -3.5, 0.0], np.float32).reshape(1, 2, 3, 1)
    data.view(np.uint32)[0, 0, 0, 0] = 0x7FC01234  # NaN payload
    t = pk.Tensor4(data)
    pk.save_tensor(t, tmp_path / "t.c0nv")
    back = pk.load_tensor(tmp_path / "t.c0nv")
    assert back.data.tobytes() == data.tobytes()
    (tmp_path / "bad").write_bytes(b"XXXX" + bytes(18))
    with pytest.raises(pk.FormatError):
        pk.load_tensor(tmp_path / "bad")


def test_tensor_helpers():
    t = pk.make_tensor((2, 3, 4, 5), "uniform", seed=7)
    assert t.data.flags.c_contiguous and t.data.dtype == np.float32
    assert t.coords(t.flat_index(1, 2, 3, 4)) == (1, 2, 3, 4)
    assert pk.read_padded(t, 0, 0, -1, 0) == 0.0
    with pytest.raises(IndexError):
        pk.read_padded(t, 2, 0, 0, 0)
    with pytest.raises(pk.InvalidShape):
        pk.make_tensor((1, 2, 3), "zeros")


# --- the launch-plan contract (execmodel.py:36-128) ---------------------------

def test_plan_launch_matches_reference_golden(golden, native):
    for rec in golden["plans"] + golden["presets"]:
        dev = pk.DeviceModel(max_threads_per_block=rec.get("max_threads", 1024))
        p = pk.plan_launch(cfg_from(rec["cfg"]), dev)
        assert [p.blocks, p.threads_per_block, p.split_per_filter_row, p.dot_products_per_thread] == rec["plan"]
        pk.validate_plan(p, cfg_from(rec["cfg"]), dev)


def test_plan_launch_reference_expectations(native):
    presets = {c.name: c for c in pk.preset_configs()}
    a, b = pk.plan_launch(presets["1x1-A"]), pk.plan_launch(presets["1x1-B"])
    assert (a.blocks, a.threads_per_block, b.blocks, b.threads_per_block) == (256, 64, 1024, 224)  # crit. 4
    big = pk.plan_launch(pk.ConvConfig("t", n=1, c=1, h=40, w=50, m=1, hf=1, wf=1))
    assert (big.split_per_filter_row, big.threads_per_block, big.blocks) == (2, 1024, 2)
    odd = pk.plan_launch(pk.ConvConfig("t", n=1, c=1, h=10, w=10, m=1, hf=1, wf=1), pk.DeviceModel(max_threads_per_block=48))
    assert odd.threads_per_block == 32
    with pytest.raises(pk.Unsupported):
        pk.plan_launch(pk.ConvConfig("t", n=1, c=1, h=5, w=5, m=1, hf=3, wf=3, stride=2))


@pytest.mark.parametrize("override", [dict(split_per_filter_row=0), dict(blocks=3), dict(threads_per_block=2048, blocks=2),
                                      dict(threads_per_block=0, blocks=2), dict(threads_per_block=33),
                                      dict(dot_products_per_thread=0), dict(threads_per_block=32)])
def test_validate_plan_rejects(native, override):
    cfg = pk.ConvConfig("t", n=1, c=1, h=8, w=8, m=2, hf=1, wf=1)
    good = pk.plan_launch(cfg)
    fields = dict(blocks=good.blocks, threads_per_block=good.threads_per_block,
                  split_per_filter_row=good.split_per_filter_row, dot_products_per_thread=good.dot_products_per_thread)
    fields.update(override)
    with pytest.raises(pk.InvalidPlan):
        pk.validate_plan(pk.LaunchPlan(**fields), cfg)


def test_device_model_validation():
    with pytest.raises(pk.InvalidConfig) as exc:
        pk.DeviceModel(line_bytes=100, element_bytes=8)
    assert exc.value.field == "line_bytes"
    assert pk.DeviceModel().elements_per_line == 32


def test_block_position_ranges(native):
    for work, split in [(10, 3), (4096, 4), (7, 7), (1, 1), (1000, 17)]:
        r = pk.block_position_ranges(work, split)
        assert r[0][0] == 0 and r[-1][1] == work and len(r) == split
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1


def test_workspace_bytes(golden, native):
    for rec in golden["plans"] + golden["presets"]:
        cfg = cfg_from(rec["cfg"])
        assert pk.workspace_bytes(cfg) == rec["workspace_bytes"]
        assert native.b2c_workspace_bytes(ctypes.byref(nat.desc(cfg))) == rec["workspace_bytes"]


# --- preconditions, in the reference's order (twostage.py:73-79, 214-224) ------

def _ops(cfg):
    return pk.make_tensor(pk.input_dims(cfg)), pk.make_tensor(pk.filter_dims(cfg))


def test_stride_checked_before_shapes(native):
    cfg = pk.ConvConfig("t", n=1, c=1, h=5, w=5, m=1, hf=3, wf=3, stride=2)
    with pytest.raises(pk.Unsupported):
        pk.conv_twostage(pk.make_tensor((1, 9, 5, 5)), pk.make_tensor((1, 1, 3, 3)), cfg)
    with pytest.raises(pk.Unsupported):
        pk.stage1_scalar_prods(*_ops(cfg), cfg)


def test_shape_mismatch_before_plan(native):
    cfg = pk.ConvConfig("t", n=1, c=2, h=4, w=4, m=1, hf=1, wf=1)
    bad_plan = pk.LaunchPlan(blocks=1, threads_per_block=33, split_per_filter_row=1, dot_products_per_thread=1)
    with pytest.raises(pk.ShapeMismatch):
        pk.conv_twostage(pk.make_tensor((1, 3, 4, 4)), pk.make_tensor(pk.filter_dims(cfg)), cfg, plan=bad_plan)
    with pytest.raises(pk.ShapeMismatch):
        pk.conv_twostage(pk.make_tensor(pk.input_dims(cfg)), pk.make_tensor((1, 2, 3, 3)), cfg)


def test_plan_before_workspace(native):
    cfg = pk.ConvConfig("t", n=1, c=1, h=4, w=4, m=1, hf=3, wf=3, pad_h=1, pad_w=1)
    bad_plan = pk.LaunchPlan(blocks=1, threads_per_block=33, split_per_filter_row=1, dot_products_per_thread=1)
    with pytest.raises(pk.InvalidPlan):
        pk.conv_twostage(*_ops(cfg), cfg, workspace_limit=0, plan=bad_plan)


def test_workspace_exceeded_carries_sizes(native):
    cfg = next(c for c in pk.preset_configs() if c.name == "5x5-B")
    with pytest.raises(pk.WorkspaceExceeded) as exc:
        pk.conv_twostage(*_ops(cfg), cfg, workspace_limit=1000)
    assert (exc.value.required, exc.value.limit) == (5_017_600, 1000)
    with pytest.raises(pk.WorkspaceExceeded):
        pk.stage1_scalar_prods(*_ops(cfg), cfg, workspace_limit=1000)


def test_non_tensor_arguments_raise_attribute_error(native):
    cfg = pk.ConvConfig("t", n=1, c=1, h=3, w=3, m=1, hf=1, wf=1)
    with pytest.raises(AttributeError):
        pk.conv_twostage(np.zeros((1, 1, 3, 3), np.float32), pk.make_tensor((1, 1, 1, 1)), cfg)


def test_stage2_shape_mismatch(native):
    cfg = pk.ConvConfig("t", n=1, c=1, h=3, w=3, m=1, hf=3, wf=3, pad_h=1, pad_w=1)
    with pytest.raises(pk.ShapeMismatch):
        pk.stage2_sum(pk.PartialSums(np.zeros((8, 1, 1, 3, 3), np.float32)), cfg)


def test_c_abi_argument_errors(native):
    d = nat.desc(pk.ConvConfig("t", n=1, c=1, h=3, w=3, m=1, hf=1, wf=1))
    st = native.b2c_conv2d_forward(ctypes.byref(d), None, None, None, None, 0, None, None)
    assert st == nat.INVALID_ARGUMENT
    assert "null" in nat.last_error()
    d2 = nat.desc(pk.ConvConfig("t", n=1, c=1, h=3, w=3, m=1, hf=3, wf=3, stride=2))
    st = native.b2c_conv_twostage(ctypes.byref(d2), None, None, None, None, 0, None, None, 1 << 30, None, None)
    assert st == nat.UNSUPPORTED


# --- the B200 tile planner ----------------------------------------------------

def test_tile_planner_covers_every_baseline_layer(native):
    from paper_2103_16234_b200 import workloads as W

    for wl, (_, batches) in W.WORKLOADS.items():
        for n in batches:
            for cfg in W.layers(wl, n):
                t = pk.select_tiles(cfg)
                ho, wo = pk.output_dims(cfg)
                assert t.smem_bytes <= 227 * 1024
                if "_row7_" in t.family or "_rws7_" in t.family:
                    # row-segment kernels: tiles of bp/7 segments of 7 outputs of one row
                    segs = cfg.n * ho * -(-wo // 7)
                    tiles = -(-cfg.m // t.bm) * -(-segs // (t.bp // 7))
                else:
                    tiles = -(-cfg.m // t.bm) * -(-(cfg.n * ho * wo) // t.bp)
                assert t.grid == tiles * t.splits, (wl, cfg.name)
                chunks = -(-cfg.c // t.bc)
                assert 1 <= t.splits <= chunks
                # packed-pixel pointwise plans keep the gathered input x'[C][ceil4(Q)] at the head of
                # the workspace (256-byte aligned), the split-C partial planes after it
                packed = ((4 * cfg.c * (-(-(cfg.n * ho * wo) // 4) * 4) + 255) // 256 * 256
                          if "_1x1pk" in t.family else 0)
                assert (t.workspace_bytes > 0) == (t.splits > 1 or packed > 0)
                split_bytes = 4 * t.splits * cfg.n * cfg.m * ho * wo if t.splits > 1 else 0
                assert t.workspace_bytes == packed + split_bytes, (wl, cfg.name, t.family)
                if cfg.stride == 1:
                    s = pk.select_tiles(cfg, "twostage")
                    assert s.family.startswith("stage1_strict") and s.splits == 1


def test_tile_planner_forced_family_and_split(native):
    cfg = pk.ConvConfig("t", n=4, c=64, h=14, w=14, m=48, hf=3, wf=3, pad_h=1, pad_w=1)
    fams = pk.matching_families(cfg)
    names = pk.family_names()
    assert any(names[f] == "fused_3x3s1_m32" for f in fams) and any(names[f].startswith("fused_generic") for f in fams)
    for f in fams:
        assert pk.select_tiles(cfg, family=f).family_id == f
    t = pk.select_tiles(cfg, splits=4)
    assert t.splits == 4
    with pytest.raises(pk.InvalidPlan):
        pk.select_tiles(cfg, family=names.index("fused_1x1s1_m32"))


# --- the tensor-core (tcgen05) planner ------------------------------------------

def _tc_plan(native, cfg, engine, nf=0):
    import ctypes

    from paper_2103_16234_b200 import _native as nat

    plan = nat.TcPlanC()
    plan.filters_per_tile = nf
    st = native.b2c_tc_select_tiles(ctypes.byref(nat.desc(cfg)), nat.ENGINES[engine], ctypes.byref(plan))
    nat.check(st)
    return plan


def test_tensor_core_planner_covers_every_baseline_layer(native):
    from paper_2103_16234_b200 import workloads as W

    for wl, (_, batches) in W.WORKLOADS.items():
        for n in batches:
            for cfg in W.layers(wl, n):
                ho, wo = pk.output_dims(cfg)
                for engine in ("tf32x3", "tf32"):
                    p = _tc_plan(native, cfg, engine)
                    assert p.passes == (3 if engine == "tf32x3" else 1)
                    assert p.pixels_per_chunk in ((8, 16, 32) if p.mode == 1 else (0,)) and p.filters_per_tile % 16 == 0
                    assert 16 <= p.filters_per_tile <= 256 and p.filter_tiles * p.filters_per_tile >= cfg.m
                    assert p.stages >= 2 and p.smem_bytes <= 227 * 1024
                    cols = p.filters_per_tile * (2 if engine == "tf32x3" else 1) * (p.m_halves if p.mode == 2 else 1)
                    assert cols <= p.tmem_columns <= 512 and p.tmem_columns & (p.tmem_columns - 1) == 0
                    flat = cfg.hf == cfg.wf == 1 and cfg.stride == 1 and cfg.pad_h == cfg.pad_w == 0
                    assert bool(p.flattened) == flat
                    kb = -(-cfg.c // 16) * cfg.hf * cfg.wf
                    assert bool(p.k_packed) == (cfg.c < 16 and cfg.hf * cfg.wf > 1)
                    if p.k_packed:
                        kb = -(-(cfg.c * cfg.hf * cfg.wf) // 16)
                    assert p.mode in (1, 2)
                    if p.mode == 1:  # gather: 128-pixel tiles of 32-pixel chunks
                        width = ho * wo if flat else wo
                        rows = 1 if flat else ho
                        xw = p.pixels_per_chunk
                        chunks = cfg.n * -(-rows // (32 // xw)) * -(-width // xw)
                        tiles = -(-chunks // 4)
                        assert 1 <= p.splits <= kb
                        kbps = -(-kb // p.splits)
                    else:  # halo: 128 positions of the flattened padded stack
                        assert cfg.stride == 1
                        hp, wp = cfg.h + 2 * cfg.pad_h, cfg.w + 2 * cfg.pad_w
                        mh = p.m_halves
                        assert mh in (1, 2, 4)
                        assert p.halo_positions == -(-(128 * mh + (cfg.hf - 1) * wp + cfg.wf - 1) // 8) * 8
                        tiles = -(-(cfg.n * hp * wp) // (128 * mh))
                        cbl = -(-cfg.c // 16)
                        assert 1 <= p.splits <= cbl
                        kbps = -(-cbl // p.splits) * cfg.hf * cfg.wf
                    assert p.grid == tiles * p.filter_tiles * p.splits, (wl, cfg.name)
                    planes = 2 if engine == "tf32x3" else 1
                    if engine == "tf32x3":
                        assert kbps <= max(72, cfg.hf * cfg.wf)  # <= 1152 products per split (accuracy rule)
                    wpl = planes
                    filt = 4 * kb * 16 * p.filter_tiles * p.filters_per_tile * wpl
                    part = 4 * p.splits * cfg.n * cfg.m * ho * wo if p.splits > 1 else 0
                    assert p.workspace_bytes == -(-filt // 256) * 256 + part


def test_tensor_core_planner_forced_tiles_and_errors(native):
    import ctypes

    from paper_2103_16234_b200 import _native as nat

    cfg = pk.ConvConfig("t", n=2, c=40, h=12, w=12, m=96, hf=3, wf=3, pad_h=1, pad_w=1)
    for nf in (16, 32, 48, 96, 256):
        p = _tc_plan(native, cfg, "tf32x3", nf)
        assert p.filters_per_tile == nf and p.filter_tiles == -(-96 // nf)
    for bad in (8, 24, 272):
        with pytest.raises(pk.InvalidPlan):
            _tc_plan(native, cfg, "tf32", bad)
    plan = nat.TcPlanC()
    assert native.b2c_tc_select_tiles(ctypes.byref(nat.desc(cfg)), nat.ENGINE_FUSED, ctypes.byref(plan)) \
        == nat.INVALID_ARGUMENT
    # device compute entry validates before touching the GPU
    assert native.b2c_conv2d_forward_tc(ctypes.byref(nat.desc(cfg)), None, None, None, None, 0, nat.ENGINE_TF32X3,
                                        None, None) == nat.INVALID_ARGUMENT
    p = nat.TcPlanC()
    p.splits = 3
    assert native.b2c_tc_select_tiles(ctypes.byref(nat.desc(cfg)), nat.ENGINE_TF32, ctypes.byref(p)) == nat.OK
    assert p.splits == 3


# --- harness I/O compatibility ------------------------------

def test_harness_csv_header_is_reference_prefix_and_skips(tmp_path):
    from paper_2103_16234_b200 import harness as H

    assert H.CSV_HEADER == ("config,algorithm,batch,repeats,mean_us,min_us,stddev_us,speedup,validated,"
                            "workspace_bytes,txn_per_warp")  # convkit bench.py:37
    s2 = pk.ConvConfig("s2", n=1, c=3, h=9, w=9, m=4, hf=3, wf=3, stride=2, pad_h=1, pad_w=1)
    assert H.skip_reason("twostage", s2) == "Unsupported: stride"
    big = pk.ConvConfig("big", n=128, c=64, h=224, w=224, m=64, hf=3, wf=3, pad_h=1, pad_w=1)
    assert H.skip_reason("twostage", big) == "WorkspaceExceeded"
    assert H.skip_reason("tf32x3", s2) is None and H.skip_reason("fused", big) is None
    with pytest.raises(pk.ConvKitError):
        H.skip_reason("winograd", s2)
    rec = H.BenchRecord(config="s2", algorithm="twostage", batch=1, skipped=True, skip_reason="Unsupported: stride")
    out = tmp_path / "r.csv"
    H.emit_report([rec], out)
    lines = out.read_text().splitlines()
    assert lines[0].startswith(H.CSV_HEADER + ",") and lines[1].startswith("s2,twostage,1,0,,,,,skipped(Unsupported: stride)")
    with pytest.raises(pk.ConvKitError):
        H.emit_report([], out)


def test_harness_analyze_plan_dump_runs_on_host(tmp_path):
    """``analyze`` (reference cli.py:97-120): reference ANALYZE_HEADER prefix,
    the reference plan in its columns, the B200 plan of every engine after it;
    planner-only, so it runs without a GPU."""
    from paper_2103_16234_b200 import harness as H

    assert H.ANALYZE_HEADER == ("config,batch,blocks,threads_per_block,split,dot_products_per_thread,"
                                "warps_total,transactions_total,txn_per_warp,perfectly_coalesced_warps")
    out = tmp_path / "plans.csv"
    assert H.main(["analyze", "--batches", "1,8", "--algos", "fused,twostage,tf32x3", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == H.ANALYZE_HEADER + "," + H.ANALYZE_GPU_COLUMNS
    rows = [l.split(",") for l in lines[1:]]
    presets = pk.preset_configs()
    assert len(rows) == len(presets) * 2 * 3  # every preset is stride 1: all three engines plan
    for r, cfg in zip(rows[::6], presets):
        plan = pk.plan_launch(cfg.with_batch(1))
        assert r[0] == cfg.name and r[2:6] == [str(plan.blocks), str(plan.threads_per_block),
                                               str(plan.split_per_filter_row), str(plan.dot_products_per_thread)]
    for r in rows:
        assert r[10] in ("fused", "twostage", "tf32x3") and r[11] and int(r[12]) > 0 and int(r[14]) >= 1
    assert H.main(["analyze", "--algos", "winograd", "--out", str(out)]) == 1


def test_split_reduction_mode_plumbing():
    """b2c_tile_plan.reduce: planner default = partial planes + stage 2 (1);
    forced DSMEM cluster (2) for <= 16 splits and tiles that fit shared
    memory, InvalidPlan beyond; tuned plans carry their mode."""
    import ctypes

    from paper_2103_16234_b200 import _native as nat

    cfg = pk.ConvConfig("red", n=2, c=512, h=14, w=14, m=130, hf=1, wf=1)
    assert pk.select_tiles(cfg, splits=1).reduce == 0
    p1, p2 = pk.select_tiles(cfg, splits=8, reduce=1), pk.select_tiles(cfg, splits=8, reduce=2)
    assert (p1.reduce, p2.reduce) == (1, 2) and p2.smem_bytes >= 4 * p2.bm * p2.bp
    assert pk.select_tiles(cfg, splits=8).reduce in (1, 2)
    assert pk.select_tiles(cfg, splits=32).reduce == 1
    with pytest.raises(pk.InvalidPlan):
        pk.select_tiles(cfg, splits=32, reduce=2)
    with pytest.raises(pk.ConvKitError):
        pk.select_tiles(cfg, splits=8, reduce=3)
    one = pk.ConvConfig("red1", n=3, c=520, h=14, w=14, m=130, hf=1, wf=1)
    fam = pk.select_tiles(one, splits=4, reduce=2).family_id
    lib = nat.lib()
    assert lib.b2c_register_tuned_plan(ctypes.byref(nat.desc(one)), nat.ENGINE_FUSED, fam, 4, 2) == nat.OK
    auto = pk.select_tiles(one)
    assert (auto.family_id, auto.splits, auto.reduce) == (fam, 4, 2)
    assert pk.ConvLayer(one).family.endswith("_dsm")
    assert lib.b2c_register_tuned_plan(ctypes.byref(nat.desc(one)), nat.ENGINE_FUSED, fam, 4, 7) != nat.OK
    twostage = pk.select_tiles(pk.ConvConfig("t", n=1, c=64, h=8, w=8, m=8, hf=3, wf=3, pad_h=1, pad_w=1),
                               engine="twostage")
    assert twostage.reduce == 0


def test_bench_dominant_kernel_roofline_fields(tmp_path, monkeypatch):
    """bench.py's roofline object is about the dominant kernel family: the one
    with the largest share of the step's kernel time; traffic comes from the
    committed ncu capture only when it covers exactly those layers."""
    import json
    import sys

    sys.path.insert(0, str(pk.__file__).rsplit("/", 2)[0])
    import bench
    from paper_2103_16234_b200 import workloads as W

    cfgs = W.layers("c2", 32)[:6]
    layers = [pk.ConvLayer(c) for c in cfgs]
    ms = [0.01] * len(cfgs)
    ms[2] = 1.0  # one slow layer makes its family dominant
    fam = layers[2].family.replace("_dsm", "")
    idx = [i for i, L in enumerate(layers) if L.family.replace("_dsm", "") == fam]
    path = tmp_path / "traffic.json"
    path.write_text(json.dumps({"c2": {cfgs[i].name: {"family": layers[i].family, "dram_bytes": 1000 + i}
                                       for i in idx}}))
    monkeypatch.setattr(bench, "TRAFFIC_PATH", str(path))
    d = bench.dominant_kernel(cfgs, layers, ms, "c2", 72.0, 6500.0)
    assert d["kernel"] == fam and d["launches"] == len(idx)
    ridge = 72.0e12 / 6500.0e9
    fl, by = sum(cfgs[i].flops for i in idx), sum(cfgs[i].compulsory_bytes for i in idx)
    assert d["bound"] == ("fp32" if fl / by >= ridge else "hbm")
    assert abs(d["share"] - sum(ms[i] for i in idx) / sum(ms)) < 1e-4
    assert abs(d["achieved_tflops"] - sum(cfgs[i].flops for i in idx) / (sum(ms[i] for i in idx) * 1e-3) / 1e12) < 1e-9
    assert d["traffic"] == round(sum(1000 + i for i in idx) / len(idx)) and d["traffic_source"]
    assert bench.dominant_kernel(cfgs, layers, ms, "c3", 72.0, 6500.0)["traffic"] is None  # no capture for it
    rows = bench.layer_rooflines(cfgs, layers, ms, 72.0, 6500.0)
    assert [r["layer"] for r in rows] == [c.name for c in cfgs]
    for r, c, t in zip(rows, cfgs, ms):
        want = (c.flops / (t * 1e-3) / 72.0e12) if r["bound"] == "fp32" else c.compulsory_bytes / (t * 1e-3) / 6500.0e9
        assert abs(r["roofline_frac"] - want) < 1e-4


def test_bench_reference_arm_contract_line():
    """`bench.py --impl reference` runs on the host (no GPU) and prints one JSON
    line with the contract keys, its own cpu_baseline and a zero-copy e2e."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "1",
                        "--warmup", "3"], cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in d["config"] and "model" not in d["config"]


def test_every_shipped_tuned_plan_is_what_the_planner_returns():
    """tuned_plans.json (measured on B200, registered at import) must be live:
    for every entry the planner's automatic choice for that exact shape is the
    recorded plan (a stale or rejected entry would silently fall back to the
    cost model)."""
    import json

    from paper_2103_16234_b200 import _native as nat

    entries = json.loads(nat.TUNED_PATH.read_text())["plans"]
    assert len(entries) > 200
    keys = ("n", "c", "h", "w", "m", "hf", "wf", "stride", "pad_h", "pad_w")
    for e in entries:
        cfg = pk.ConvConfig("tuned", **dict(zip(keys, e["desc"])))
        L = pk.ConvLayer(cfg, e["engine"])
        if e["engine"] == "fused":
            assert L.family.replace("_dsm", "") == e["family"], e["layer"]
            if e.get("splits", 0) > 0:
                assert L.splits == e["splits"], e["layer"]
            if L.splits > 1 and e.get("reduce", 0) > 0:
                assert L.reduce == e["reduce"], e["layer"]
        else:
            t = L._tc
            assert (t.mode == 2) == (e["mode"] == 2), e["layer"]
            if e["nf"] > 0:
                assert t.filters_per_tile == e["nf"], e["layer"]
            if e["splits"] > 0:
                assert t.splits == e["splits"], e["layer"]


def test_tc_forced_m_halves():
    """b2c_tc_plan.m_halves on input forces the halo plan's M slices (1/2/4);
    other values are rejected; gather plans ignore it."""
    import ctypes

    from paper_2103_16234_b200 import _native as nat

    cfg = pk.ConvConfig("mh", n=8, c=64, h=28, w=28, m=64, hf=3, wf=3, pad_h=1, pad_w=1)
    lib = nat.lib()
    for mh in (1, 2, 4):
        p = nat.TcPlanC()
        p.mode, p.m_halves = 2, mh
        assert lib.b2c_tc_select_tiles(ctypes.byref(nat.desc(cfg)), nat.ENGINE_TF32X3, ctypes.byref(p)) == nat.OK
        assert p.mode == 2 and p.m_halves == mh
        L = pk.ConvLayer(cfg, "tf32x3", tc_mode=2, tc_m_halves=mh)
        assert L._tc.m_halves == mh
    p = nat.TcPlanC()
    p.m_halves = 3
    assert lib.b2c_tc_select_tiles(ctypes.byref(nat.desc(cfg)), nat.ENGINE_TF32X3, ctypes.byref(p)) != nat.OK
    p = nat.TcPlanC()
    p.mode, p.m_halves = 1, 4
    assert lib.b2c_tc_select_tiles(ctypes.byref(nat.desc(cfg)), nat.ENGINE_TF32X3, ctypes.byref(p)) == nat.OK
    assert p.mode == 1


def _segment_banks(cfg, t, rx=7):
    """Banks of the 32 segment origins of each warp of the first tiles of a
    row-segment plan (the planner's pick_row_stride objective)."""
    ho, wo = pk.output_dims(cfg)
    nb = -(-wo // rx)
    hp = cfg.h + 2 * cfg.pad_h
    seg = t.bp // rx
    segs = cfg.n * ho * nb
    worst = 1
    for s0 in range(0, min(segs, 8 * seg), seg):
        r0 = s0 // nb
        v0 = (r0 // ho) * hp + (r0 % ho) * cfg.stride
        for w0 in range(s0, min(s0 + seg, segs), 32):
            banks = {}
            for sg in range(w0, min(w0 + 32, segs)):
                r, b = divmod(sg, nb)
                v = (r // ho) * hp + (r % ho) * cfg.stride
                bank = ((v - v0) * t.smem_row_stride + b * rx * cfg.stride) % 32
                banks[bank] = banks.get(bank, 0) + 1
            worst = max(worst, max(banks.values()))
    return worst


def test_row_segment_plans_layout(native):
    """Row-segment families (conv_row.cuh): the band row stride keeps every row
    16-byte congruent with its global row at stride 1 (RS == W mod 4), spreads each warp's
    32 segment origins over the shared-memory banks (at most 2-way on the
    BASELINE 3x3 stride-1 layers, 3-way at stride 2), and split-C through DSMEM is offered only when 7
    divides the output width (the tile is then a contiguous pixel range)."""
    from paper_2103_16234_b200 import workloads as W

    names = pk.family_names()
    checked = 0
    for wl, n in (("c5", 256), ("c4", 8), ("c1", 1)):
        for cfg in W.layers(wl, n):
            for f in pk.matching_families(cfg):
                if "_rws7_" not in names[f] and "_row7_" not in names[f]:
                    continue
                t = pk.select_tiles(cfg, family=f, splits=1)
                if cfg.stride == 1:
                    assert t.smem_row_stride % 4 == cfg.w % 4, (cfg.name, t.family)
                assert t.smem_bytes <= 227 * 1024
                if cfg.hf == 3:  # stride 2: output rows are 2 band rows apart, at best 2-3 way
                    assert _segment_banks(cfg, t) <= (2 if cfg.stride == 1 else 3), (cfg.name, t.family,
                                                                                      t.smem_row_stride)
                checked += 1
    assert checked > 20
    odd = pk.ConvConfig("odd", n=2, c=32, h=11, w=11, m=32, hf=3, wf=3, pad_h=1, pad_w=1)  # Wo = 11
    even = pk.ConvConfig("even", n=2, c=32, h=14, w=14, m=32, hf=3, wf=3, pad_h=1, pad_w=1)  # Wo = 14
    rws = names.index("fused_3x3s1_rws7_m64")
    assert pk.select_tiles(even, family=rws, splits=2, reduce=2).reduce == 2
    with pytest.raises(pk.InvalidPlan):
        pk.select_tiles(odd, family=rws, splits=2, reduce=2)
    assert pk.select_tiles(odd, family=rws, splits=2, reduce=1).reduce == 1
