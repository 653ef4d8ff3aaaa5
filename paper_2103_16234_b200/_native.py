"""ctypes binding of the C ABI (include/b2conv.h) — the only way Python
reaches the CUDA kernels.  There is no CPU fallback: if ``libb2conv.so`` is
missing or fails to load, every compute entry point raises ``DeviceError``.

The same binding is what a convkit maintainer would add to call the B200
engine from the reference package.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import (ConvKitError, DeviceError, InvalidConfig, InvalidPlan, ShapeMismatch,
                     Unsupported, WorkspaceExceeded)

LIB_PATH = Path(__file__).resolve().parent / "libb2conv.so"
if os.environ.get("B2C_LIB_VARIANT"):  # development A/B of two in-tree builds (libb2conv_<variant>.so)
    LIB_PATH = LIB_PATH.with_name(f"libb2conv_{os.environ['B2C_LIB_VARIANT']}.so")

OK, UNSUPPORTED, SHAPE_MISMATCH, INVALID_PLAN, WORKSPACE_EXCEEDED, INVALID_CONFIG, CUDA_ERROR, INVALID_ARGUMENT = range(8)
ENGINE_FUSED, ENGINE_TWOSTAGE, ENGINE_TF32X3, ENGINE_TF32 = 0, 1, 2, 3
ENGINES = {"fused": ENGINE_FUSED, "twostage": ENGINE_TWOSTAGE, "tf32x3": ENGINE_TF32X3, "tf32": ENGINE_TF32}
FIELD_NAMES = ("n", "c", "h", "w", "m", "hf", "wf", "stride", "pad_h", "pad_w")


class ConvDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in FIELD_NAMES]


class DeviceModelC(ctypes.Structure):
    _fields_ = [("warp_width", ctypes.c_int32), ("line_bytes", ctypes.c_int32),
                ("max_threads_per_block", ctypes.c_int32), ("element_bytes", ctypes.c_int32)]


class LaunchPlanC(ctypes.Structure):
    _fields_ = [("blocks", ctypes.c_int64), ("threads_per_block", ctypes.c_int32),
                ("split_per_filter_row", ctypes.c_int32), ("dot_products_per_thread", ctypes.c_int32)]


class RunStatsC(ctypes.Structure):
    _fields_ = [("stage1_tasks_run", ctypes.c_int64), ("stage2_invoked", ctypes.c_int32),
                ("filter_row_global_loads", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64)]


class TilePlanC(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("bm", ctypes.c_int32), ("bp", ctypes.c_int32),
                ("bc", ctypes.c_int32), ("threads", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("smem_rows", ctypes.c_int32), ("smem_row_stride", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int32), ("grid", ctypes.c_int64), ("splits", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64), ("reduce", ctypes.c_int32)]


class TcPlanC(ctypes.Structure):
    _fields_ = [("pixels_per_chunk", ctypes.c_int32), ("filters_per_tile", ctypes.c_int32),
                ("filter_tiles", ctypes.c_int32), ("stages", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("tmem_columns", ctypes.c_int32), ("flattened", ctypes.c_int32), ("passes", ctypes.c_int32),
                ("grid", ctypes.c_int64), ("splits", ctypes.c_int32), ("workspace_bytes", ctypes.c_int64),
                ("mode", ctypes.c_int32), ("halo_positions", ctypes.c_int32), ("m_halves", ctypes.c_int32),
                ("bf16_corrections", ctypes.c_int32), ("k_packed", ctypes.c_int32)]


_P = ctypes.POINTER
_fp = ctypes.c_void_p  # raw float* (device or host address)

# name -> (restype, argtypes); every symbol declared in include/b2conv.h
SIGNATURES = {
    "b2c_abi_version": (ctypes.c_int32, []),
    "b2c_last_error": (ctypes.c_char_p, []),
    "b2c_family_name": (ctypes.c_char_p, [ctypes.c_int32]),
    "b2c_num_families": (ctypes.c_int32, []),
    "b2c_family_matches": (ctypes.c_int32, [_P(ConvDesc), ctypes.c_int32, ctypes.c_int32]),
    "b2c_launch_count": (ctypes.c_int64, []),
    "b2c_reset_launch_count": (None, []),
    "b2c_validate_config": (ctypes.c_int, [_P(ConvDesc), _P(ctypes.c_int32)]),
    "b2c_output_dims": (ctypes.c_int, [_P(ConvDesc), _P(ctypes.c_int32), _P(ctypes.c_int32)]),
    "b2c_workspace_bytes": (ctypes.c_int64, [_P(ConvDesc)]),
    "b2c_plan_launch": (ctypes.c_int, [_P(ConvDesc), _P(DeviceModelC), _P(LaunchPlanC)]),
    "b2c_validate_plan": (ctypes.c_int, [_P(ConvDesc), _P(DeviceModelC), _P(LaunchPlanC)]),
    "b2c_block_position_ranges": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, _P(ctypes.c_int64)]),
    "b2c_select_tiles": (ctypes.c_int, [_P(ConvDesc), ctypes.c_int32, _P(TilePlanC)]),
    "b2c_register_tuned_plan": (ctypes.c_int, [_P(ConvDesc), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                               ctypes.c_int32]),
    "b2c_conv2d_forward": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, _fp, ctypes.c_void_p, ctypes.c_int64,
                                          _P(TilePlanC), ctypes.c_void_p]),
    "b2c_conv2d_forward_tc": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, _fp, ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_int32, _P(TcPlanC), ctypes.c_void_p]),
    "b2c_tc_select_tiles": (ctypes.c_int, [_P(ConvDesc), ctypes.c_int32, _P(TcPlanC)]),
    "b2c_register_tuned_tc_plan": (ctypes.c_int, [_P(ConvDesc), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                  ctypes.c_int32, ctypes.c_int32]),
    "b2c_conv_twostage": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, _fp, _fp, ctypes.c_int64, _P(LaunchPlanC),
                                         _P(DeviceModelC), ctypes.c_int64, ctypes.c_void_p, _P(RunStatsC)]),
    "b2c_stage1_scalar_prods": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, _fp, _P(LaunchPlanC), _P(DeviceModelC),
                                               ctypes.c_int64, ctypes.c_void_p, _P(RunStatsC)]),
    "b2c_stage2_sum": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, ctypes.c_void_p, _P(RunStatsC)]),
    "b2c_conv_host": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, _fp, ctypes.c_int32, _P(LaunchPlanC),
                                     _P(DeviceModelC), ctypes.c_int64, ctypes.c_int32, _P(RunStatsC)]),
    "b2c_conv_host_layers": (ctypes.c_int, [ctypes.c_int32, _P(ConvDesc), _P(ctypes.c_void_p), _P(ctypes.c_void_p),
                                            _P(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int32]),
    "b2c_stage1_host": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, _fp, _P(LaunchPlanC), _P(DeviceModelC),
                                       ctypes.c_int64, ctypes.c_int32, _P(RunStatsC)]),
    "b2c_stage2_host": (ctypes.c_int, [_P(ConvDesc), _fp, _fp, ctypes.c_int32, _P(RunStatsC)]),
    "b2c_probe_fp32_peak": (ctypes.c_int, [ctypes.c_int32, _P(ctypes.c_double), _P(ctypes.c_double),
                                           _P(ctypes.c_double)]),
    "b2c_host_alloc": (ctypes.c_void_p, [ctypes.c_size_t]),
    "b2c_host_free": (None, [ctypes.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libb2conv.so (once).  Raises DeviceError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeviceError(f"{LIB_PATH.name} is not built; run `python -m paper_2103_16234_b200.build` "
                                  "(the B200 engine has no CPU fallback)")
            try:
                l = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(l, name)
                fn.restype = res
                fn.argtypes = args
            _lib = l
            _register_tuned(l)
    return _lib


TUNED_PATH = Path(__file__).resolve().parent / "tuned_plans.json"


def _register_tuned(l) -> None:
    """Register the measured plans shipped with the package (if any)."""
    import json

    if not TUNED_PATH.exists():
        return
    try:
        entries = json.loads(TUNED_PATH.read_text()).get("plans", [])
    except (OSError, ValueError):
        return
    names = [l.b2c_family_name(i).decode() for i in range(l.b2c_num_families())]
    for e in entries:
        if e.get("engine") in ("tf32x3", "tf32"):
            d = ConvDesc(*[int(v) for v in e["desc"]])
            l.b2c_register_tuned_tc_plan(ctypes.byref(d), ENGINES[e["engine"]], int(e["mode"]), int(e["nf"]),
                                         int(e["splits"]), int(e.get("mh", 0)))
            continue
        if e.get("family") not in names:
            continue
        d = ConvDesc(*[int(v) for v in e["desc"]])
        eng = ENGINE_TWOSTAGE if e.get("engine") == "twostage" else ENGINE_FUSED
        l.b2c_register_tuned_plan(ctypes.byref(d), eng, names.index(e["family"]), int(e.get("splits", 1)),
                                  int(e.get("reduce", 0)))


def last_error() -> str:
    return lib().b2c_last_error().decode("utf-8", "replace")


def desc(cfg) -> ConvDesc:
    vals = cfg.as_tuple() if hasattr(cfg, "as_tuple") else tuple(int(v) for v in cfg)
    return ConvDesc(*vals)


def check(status: int, *, required: int = 0, limit: int = 0, field: str = "") -> None:
    """Raise the reference exception class matching a b2c_status."""
    if status == OK:
        return
    msg = last_error()
    if status == UNSUPPORTED:
        raise Unsupported(msg)
    if status == SHAPE_MISMATCH:
        raise ShapeMismatch(msg)
    if status == INVALID_PLAN:
        raise InvalidPlan(msg)
    if status == WORKSPACE_EXCEEDED:
        raise WorkspaceExceeded(required, limit)
    if status == INVALID_CONFIG:
        name = field or (msg.split(":", 1)[0] if ":" in msg else "config")
        raise InvalidConfig(name, msg.split(": ", 1)[-1])
    if status == CUDA_ERROR:
        raise DeviceError(msg)
    raise ConvKitError(msg or f"b2c status {status}")
