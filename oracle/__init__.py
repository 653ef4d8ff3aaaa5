"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's forward-convolution path (convkit 0.1.0).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package, and only as the checker or the
timed CPU baseline.  The product package ``paper_2103_16234_b200`` never imports
it and has no CPU fallback.

The arithmetic lives in ``conv_oracle.c`` (built into ``liboracle.so`` by
``oracle/Makefile``; compiled with ``-ffp-contract=off`` so every fp32 multiply
and add rounds separately, like numpy's float32 ufuncs).  This module adds the
numpy-level helpers the reference tests rely on:

* ``make_uniform``    — restates ``tensor.make_tensor(..., "uniform", seed)``
                         (/root/reference/pkg/src/convkit/tensor.py:80-109)
* ``bench_seeds``     — restates the harness seed derivation
                         (/root/reference/pkg/src/convkit/bench.py:119-121)
* ``relative_error``  — restates reference.py:254-271
* ``conv_naive`` / ``conv_f64`` / ``stage1`` / ``stage2`` / ``conv_twostage`` /
  ``plan_launch``      — thin ctypes wrappers over conv_oracle.c, each citing
                         the reference function it restates.

Parity of this oracle against the reference itself is pinned by
``tests/test_oracle.py`` using fixtures in ``tests/golden/`` that were produced
by importing the reference (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_f32p = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> Path:
    """Compile liboracle.so with the committed Makefile (gcc, no CUDA)."""
    src = _HERE / "conv_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE), "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        l = ctypes.CDLL(str(_LIB_PATH))
        for name in ("oracle_conv_naive", "oracle_conv_f64", "oracle_conv_twostage", "oracle_stage1"):
            fn = getattr(l, name)
            fn.argtypes = [_i32p, _f32p, _f32p, _f32p, ctypes.c_int]
            fn.restype = ctypes.c_int
        l.oracle_stage2.argtypes = [_i32p, _f32p, _f32p, ctypes.c_int]
        l.oracle_stage2.restype = ctypes.c_int
        l.oracle_plan_launch.argtypes = [_i32p, ctypes.c_int32, ctypes.c_int32, _i64p]
        l.oracle_plan_launch.restype = None
        l.oracle_max_threads.argtypes = []
        l.oracle_max_threads.restype = ctypes.c_int
        _lib = l
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


# ---------------------------------------------------------------------------
# shapes
# ---------------------------------------------------------------------------

def desc_of(cfg) -> np.ndarray:
    """int32[10] {n,c,h,w,m,hf,wf,stride,pad_h,pad_w} from any object with
    those attributes (ConvConfig field order, configs.py:17-40) or a tuple."""
    if isinstance(cfg, (tuple, list, np.ndarray)):
        vals = [int(v) for v in cfg]
        if len(vals) == 7:  # n,c,h,w,m,hf,wf with stride 1, pad 0
            vals += [1, 0, 0]
    else:
        vals = [int(getattr(cfg, f)) for f in ("n", "c", "h", "w", "m", "hf", "wf", "stride", "pad_h", "pad_w")]
    return np.ascontiguousarray(np.array(vals, dtype=np.int32))


def out_dims(d) -> tuple[int, int]:
    """configs.output_dims (configs.py:60-64)."""
    n, c, h, w, m, hf, wf, s, ph, pw = (int(v) for v in d)
    return (h + 2 * ph - hf) // s + 1, (w + 2 * pw - wf) // s + 1


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _prep(cfg, x, w):
    d = desc_of(cfg)
    x = np.ascontiguousarray(x, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    n, c, h, ww, m, hf, wf = (int(v) for v in d[:7])
    if x.shape != (n, c, h, ww) or w.shape != (m, c, hf, wf):
        raise ValueError(f"oracle: operand shapes {x.shape}/{w.shape} do not match {d.tolist()}")
    return d, x, w


def _run(name, cfg, x, w, threads):
    d, x, w = _prep(cfg, x, w)
    ho, wo = out_dims(d)
    y = np.empty((int(d[0]), int(d[4]), ho, wo), dtype=np.float32)
    rc = getattr(lib(), name)(_ptr(d, _i32p), _ptr(x, _f32p), _ptr(w, _f32p), _ptr(y, _f32p), int(threads))
    if rc:
        raise MemoryError(f"{name} failed")
    return y


def conv_naive(cfg, x, w, threads: int = 0) -> np.ndarray:
    """reference.conv_naive (reference.py:58-83): pinned-order fp32, any stride."""
    return _run("oracle_conv_naive", cfg, x, w, threads)


def conv_f64(cfg, x, w, threads: int = 0) -> np.ndarray:
    """reference.conv_naive_f64 (reference.py:86-103): f64 accumulation, one rounding."""
    return _run("oracle_conv_f64", cfg, x, w, threads)


def conv_twostage(cfg, x, w, threads: int = 0) -> np.ndarray:
    """twostage.conv_twostage arithmetic (twostage.py:208-239), stride 1."""
    return _run("oracle_conv_twostage", cfg, x, w, threads)


def stage1(cfg, x, w, threads: int = 0) -> np.ndarray:
    """twostage.stage1_scalar_prods arithmetic (twostage.py:148-172): (k,n,m,ho,wo)."""
    d, x, w = _prep(cfg, x, w)
    ho, wo = out_dims(d)
    k = int(d[5]) * int(d[6])
    p = np.empty((k, int(d[0]), int(d[4]), ho, wo), dtype=np.float32)
    rc = lib().oracle_stage1(_ptr(d, _i32p), _ptr(x, _f32p), _ptr(w, _f32p), _ptr(p, _f32p), int(threads))
    if rc:
        raise MemoryError("oracle_stage1 failed")
    return p


def stage2(cfg, partials, threads: int = 0) -> np.ndarray:
    """twostage.stage2_sum arithmetic (twostage.py:175-205)."""
    d = desc_of(cfg)
    ho, wo = out_dims(d)
    p = np.ascontiguousarray(partials, dtype=np.float32)
    y = np.empty((int(d[0]), int(d[4]), ho, wo), dtype=np.float32)
    lib().oracle_stage2(_ptr(d, _i32p), _ptr(p, _f32p), _ptr(y, _f32p), int(threads))
    return y


def plan_launch(cfg, warp: int = 32, max_threads: int = 1024) -> tuple[int, int, int, int]:
    """execmodel.plan_launch (execmodel.py:73-98) →
    (blocks, threads_per_block, split_per_filter_row, dot_products_per_thread)."""
    d = desc_of(cfg)
    out = np.zeros(4, dtype=np.int64)
    lib().oracle_plan_launch(_ptr(d, _i32p), int(warp), int(max_threads), _ptr(out, _i64p))
    return tuple(int(v) for v in out)


# ---------------------------------------------------------------------------
# numpy-level restatements
# ---------------------------------------------------------------------------

def make_uniform(dims, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """tensor.make_tensor(dims, "uniform", seed=seed) (tensor.py:100-109):
    PCG64(seed).uniform(lo, hi) in f64, then cast to fp32, C-contiguous NCHW."""
    gen = np.random.Generator(np.random.PCG64(int(seed)))
    return np.ascontiguousarray(gen.uniform(lo, hi, size=tuple(int(v) for v in dims)).astype(np.float32))


def bench_seeds(seed: int, idx: int, batch: int) -> tuple[int, int]:
    """Input/filter seeds of run_bench (bench.py:119)."""
    a, b = np.random.SeedSequence([seed, idx, batch]).generate_state(2)
    return int(a), int(b)


def relative_error(result, reference) -> float:
    """reference.relative_error (reference.py:254-271): max|a-b| / max|ref| in f64."""
    a = np.asarray(result, dtype=np.float64)
    b = np.asarray(reference, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.size == 0:
        return 0.0
    diff = float(np.max(np.abs(a - b)))
    if diff == 0.0:
        return 0.0
    scale = float(np.max(np.abs(b)))
    return float("inf") if scale == 0.0 else diff / scale


def fp32_tolerance(c: int, hf: int, wf: int) -> float:
    """Fused-FFMA engine gate from BASELINE.json north_star / SURVEY §8(d):
    relative_error vs conv_naive_f64 <= 1e-5 * max(1, K/4096), K = C*hf*wf."""
    return 1e-5 * max(1.0, (c * hf * wf) / 4096.0)


def max_ulp_diff(a, b) -> int:
    """Largest distance in fp32 ulps (ordered-integer metric), NaNs must match."""
    ai = np.asarray(a, dtype=np.float32).view(np.int32).astype(np.int64)
    bi = np.asarray(b, dtype=np.float32).view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return int(np.max(np.abs(ai - bi))) if ai.size else 0
