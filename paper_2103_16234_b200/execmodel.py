"""Launch-plan contract of the drop-in.

``DeviceModel``/``LaunchPlan``/``plan_launch``/``validate_plan``/
``block_position_ranges`` keep the reference's semantics
(execmodel.py:36-128): the plan is the paper's one-filter-row-per-block
decomposition, validated before any work and used for ``RunStats``.  The
arithmetic runs in the C ABI (``b2c_plan_launch``/``b2c_validate_plan``), the
same code the CUDA entry points use for their precondition checks.

The grid the B200 kernels actually run is chosen separately by the tile
planner (``select_tiles``): per (filter size, stride, channels, plane, batch)
it picks a kernel family and CTA tile for 148 SMs.  Outputs never depend on
either plan.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native as nat
from .configs import ConvConfig, output_dims
from .errors import InvalidConfig, Unsupported


@dataclass(frozen=True)
class DeviceModel:
    """Device limits of the reference's analytical model (warp 32, 128 B line,
    1024 threads per block, 4 B elements)."""

    warp_width: int = 32
    line_bytes: int = 128
    max_threads_per_block: int = 1024
    element_bytes: int = 4

    def __post_init__(self):
        for f in ("warp_width", "line_bytes", "max_threads_per_block", "element_bytes"):
            if getattr(self, f) < 1:
                raise InvalidConfig(f, f"must be >= 1, got {getattr(self, f)}")
        if self.line_bytes % self.element_bytes:
            raise InvalidConfig("line_bytes", f"{self.line_bytes} not a multiple of element size "
                                              f"{self.element_bytes}")

    @property
    def elements_per_line(self) -> int:
        return self.line_bytes // self.element_bytes

    def _c(self) -> nat.DeviceModelC:
        return nat.DeviceModelC(self.warp_width, self.line_bytes, self.max_threads_per_block, self.element_bytes)


@dataclass(frozen=True)
class LaunchPlan:
    """Stage-1 block decomposition: blocks = m*hf*wf*split."""

    blocks: int
    threads_per_block: int
    split_per_filter_row: int
    dot_products_per_thread: int

    def _c(self) -> nat.LaunchPlanC:
        return nat.LaunchPlanC(self.blocks, self.threads_per_block, self.split_per_filter_row,
                               self.dot_products_per_thread)


@dataclass(frozen=True)
class TilePlan:
    """The B200 grid for one layer (b2c_tile_plan)."""

    family: str
    family_id: int
    bm: int
    bp: int
    bc: int
    threads: int
    stages: int
    smem_rows: int
    smem_row_stride: int
    smem_bytes: int
    grid: int
    splits: int
    workspace_bytes: int
    reduce: int = 0  # split-C reduction: 0 none, 1 partial planes + stage 2, 2 DSMEM cluster


def _plan_from_c(p: nat.LaunchPlanC) -> LaunchPlan:
    return LaunchPlan(int(p.blocks), int(p.threads_per_block), int(p.split_per_filter_row),
                      int(p.dot_products_per_thread))


def plan_launch(cfg: ConvConfig, device: DeviceModel | None = None) -> LaunchPlan:
    """One filter row per block; split = ceil(n*h_out*w_out / max_threads);
    threads rounded up to whole warps (execmodel.py:73-98).  Stride 1 only."""
    if cfg.stride != 1:
        raise Unsupported(f"launch planning covers stride 1, got {cfg.stride}")
    device = device or DeviceModel()
    out = nat.LaunchPlanC()
    nat.check(nat.lib().b2c_plan_launch(ctypes.byref(nat.desc(cfg)), ctypes.byref(device._c()), ctypes.byref(out)))
    return _plan_from_c(out)


def validate_plan(plan: LaunchPlan, cfg: ConvConfig, device: DeviceModel | None = None) -> None:
    """Raise InvalidPlan unless blocks = m*hf*wf*split, threads are a warp
    multiple within the device limit, and the plan covers every dot product."""
    device = device or DeviceModel()
    nat.check(nat.lib().b2c_validate_plan(ctypes.byref(nat.desc(cfg)), ctypes.byref(device._c()),
                                          ctypes.byref(plan._c())))


def block_position_ranges(work: int, split: int) -> list[tuple[int, int]]:
    """Balanced contiguous [lo, hi) ranges of one filter row's positions."""
    if split < 1:
        return []
    buf = (ctypes.c_int64 * (2 * split))()
    nat.check(nat.lib().b2c_block_position_ranges(int(work), int(split), buf))
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(split)]


def theoretical_reuse(cfg: ConvConfig) -> tuple[int, int]:
    """(row_reuse, max_element_reuse) = (h_out*w_out, hf*wf) at stride 1
    (execmodel.py:218-228)."""
    if cfg.stride != 1:
        raise Unsupported(f"reuse model covers stride 1, got {cfg.stride}")
    ho, wo = output_dims(cfg)
    return ho * wo, cfg.hf * cfg.wf


def family_names() -> list[str]:
    l = nat.lib()
    return [l.b2c_family_name(i).decode() for i in range(l.b2c_num_families())]


def matching_families(cfg: ConvConfig, engine: str = "fused") -> list[int]:
    """Kernel families able to run ``cfg`` under ``engine`` ("fused"|"twostage")."""
    l = nat.lib()
    e = nat.ENGINE_TWOSTAGE if engine == "twostage" else nat.ENGINE_FUSED
    d = nat.desc(cfg)
    return [i for i in range(l.b2c_num_families()) if l.b2c_family_matches(ctypes.byref(d), e, i)]


def select_tiles(cfg: ConvConfig, engine: str = "fused", family: int = -1, splits: int = 0,
                 reduce: int = 0) -> TilePlan:
    """The B200 tile plan for ``cfg`` (planner's choice, or a forced family / split / reduction)."""
    out = nat.TilePlanC()
    out.family = int(family)
    out.splits = int(splits)
    out.reduce = int(reduce)
    e = nat.ENGINE_TWOSTAGE if engine == "twostage" else nat.ENGINE_FUSED
    nat.check(nat.lib().b2c_select_tiles(ctypes.byref(nat.desc(cfg)), e, ctypes.byref(out)))
    return TilePlan(nat.lib().b2c_family_name(out.family).decode(), int(out.family), int(out.bm), int(out.bp),
                    int(out.bc), int(out.threads), int(out.stages), int(out.smem_rows), int(out.smem_row_stride),
                    int(out.smem_bytes), int(out.grid), int(out.splits), int(out.workspace_bytes), int(out.reduce))
