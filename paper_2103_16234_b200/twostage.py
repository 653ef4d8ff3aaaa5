"""The drop-in forward-convolution entry point: ``conv_twostage`` and its
stage-wise siblings, with convkit's signatures, return types, exception
classes and precondition order (twostage.py:33-239), running on B200.

Two engines sit behind the same call:

``engine="twostage"`` (default)
    The paper's scheme on the GPU: a stage-1 kernel computes one partial-sum
    plane per filter row k=(yf,xf) (channels ascending, separately rounded
    multiply and add, +0.0 start) into a device workspace of
    4*hf*wf*n*m*h_out*w_out bytes, and a stage-2 kernel adds the planes in
    ascending k.  1x1 layers are fused (stage 1 writes the output, no
    workspace).  Bitwise identical to the reference's ``conv_twostage`` and
    ``conv_naive``; RunStats, InvalidPlan and WorkspaceExceeded behave exactly
    as in the reference.

``engine="fused"``
    The B200 fast path: one FFMA2 kernel reduces channels and filter rows in
    registers, no workspace (so ``workspace_limit`` never trips), within
    tol(K) = 1e-5*max(1, K/4096) of ``conv_naive_f64`` (K = c*hf*wf).

``engine="tf32x3"`` / ``engine="tf32"``
    The optional tensor-core variant (tcgen05 implicit GEMM, TMA-shifted
    input rows, TMEM accumulators): 3xTF32 operand splitting is fp32-class
    (within tol(K)); plain TF32 has its own 5e-3 tolerance.  Stride 1 and
    W % 4 == 0 (or unpadded 1x1 with H*W % 4 == 0) only: Unsupported otherwise.

``workers`` is accepted for signature compatibility; the GPU result is
independent of it (as the reference's is).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .configs import ConvConfig, filter_dims, input_dims, output_dims
from .errors import ShapeMismatch, Unsupported, WorkspaceExceeded
from .execmodel import DeviceModel, LaunchPlan, plan_launch, validate_plan
from .tensor import Tensor4

DEFAULT_WORKSPACE_LIMIT = 1_073_741_824
ENGINES = ("twostage", "fused", "tf32x3", "tf32")


def workspace_bytes(cfg: ConvConfig) -> int:
    """Bytes of the stage-1 partial-sum buffer: 4*hf*wf*n*m*h_out*w_out, 0 for 1x1."""
    if cfg.hf == 1 and cfg.wf == 1:
        return 0
    ho, wo = output_dims(cfg)
    return 4 * cfg.hf * cfg.wf * cfg.n * cfg.m * ho * wo


@dataclass
class RunStats:
    """Counters of a two-stage run (twostage.py:48-55).  Task and load counts
    follow the reference launch plan (one task = one filter row x position
    range) so they are comparable across engines and with the reference."""

    stage1_tasks_run: int = 0
    stage2_invoked: bool = False
    filter_row_global_loads: int = 0
    workspace_bytes: int = 0


@dataclass
class PartialSums:
    """Stage-1 output laid out (k, n, m, h_out, w_out), x fastest."""

    data: np.ndarray

    @property
    def dims(self) -> tuple[int, int, int, int, int]:
        return self.data.shape

    @property
    def byte_size(self) -> int:
        return self.data.nbytes


def _check_operands(inp: Tensor4, filters: Tensor4, cfg: ConvConfig, *, stride1: bool) -> None:
    # reference order: stride first, then input dims, then filter dims (twostage.py:73-79)
    if stride1 and cfg.stride != 1:
        raise Unsupported(f"two-stage convolution requires stride 1, got {cfg.stride}")
    if inp.dims != input_dims(cfg):
        raise ShapeMismatch(f"input dims {inp.dims} != config {input_dims(cfg)}")
    if filters.dims != filter_dims(cfg):
        raise ShapeMismatch(f"filter dims {filters.dims} != config {filter_dims(cfg)}")


def _stats(s: nat.RunStatsC) -> RunStats:
    return RunStats(int(s.stage1_tasks_run), bool(s.stage2_invoked), int(s.filter_row_global_loads),
                    int(s.workspace_bytes))


def _resolve_plan(cfg, device, plan) -> LaunchPlan:
    device = device or DeviceModel()
    plan = plan or plan_launch(cfg, device)
    validate_plan(plan, cfg, device)
    return plan


def conv_twostage(inp: Tensor4, filters: Tensor4, cfg: ConvConfig, device: DeviceModel | None = None,
                  workspace_limit: int = DEFAULT_WORKSPACE_LIMIT, *, plan: LaunchPlan | None = None,
                  workers: int = 1, engine: str = "twostage", gpu: int = -1) -> tuple[Tensor4, RunStats]:
    """Forward convolution of ``inp`` [n,c,h,w] with ``filters`` [m,c,hf,wf];
    returns the fresh [n,m,h_out,w_out] output and its RunStats.

    Preconditions, in the reference's order: stride 1 (Unsupported) ->
    operand dims (ShapeMismatch) -> launch plan (InvalidPlan) -> workspace
    limit (WorkspaceExceeded, two-stage engine only)."""
    if engine not in ENGINES:
        raise ValueError(f"unknown engine {engine!r} (choose from {ENGINES})")
    _check_operands(inp, filters, cfg, stride1=True)
    device = device or DeviceModel()
    plan = _resolve_plan(cfg, device, plan)
    required = workspace_bytes(cfg)
    if engine == "twostage" and required > workspace_limit:
        raise WorkspaceExceeded(required, workspace_limit)
    ho, wo = output_dims(cfg)
    out = np.empty((cfg.n, cfg.m, ho, wo), dtype=np.float32)
    stats = nat.RunStatsC()
    e = nat.ENGINES[engine]
    st = nat.lib().b2c_conv_host(ctypes.byref(nat.desc(cfg)), inp.data.ctypes.data, filters.data.ctypes.data,
                                 out.ctypes.data, e, ctypes.byref(plan._c()), ctypes.byref(device._c()),
                                 int(workspace_limit), int(gpu), ctypes.byref(stats))
    nat.check(st, required=required, limit=workspace_limit)
    if engine != "twostage":
        return Tensor4(out), RunStats(plan.blocks, False, plan.blocks, 0)
    return Tensor4(out), _stats(stats)


def stage1_scalar_prods(inp: Tensor4, filters: Tensor4, cfg: ConvConfig, plan: LaunchPlan | None = None, *,
                        device: DeviceModel | None = None, workspace_limit: int = DEFAULT_WORKSPACE_LIMIT,
                        workers: int = 1, gpu: int = -1) -> tuple[PartialSums, RunStats]:
    """Stage 1 alone (twostage.py:148-172): every filter-row dot product into a
    (k, n, m, h_out, w_out) PartialSums buffer.  The buffer counts against
    ``workspace_limit`` except for 1x1 filters."""
    _check_operands(inp, filters, cfg, stride1=True)
    device = device or DeviceModel()
    plan = _resolve_plan(cfg, device, plan)
    required = workspace_bytes(cfg)
    if required > workspace_limit:
        raise WorkspaceExceeded(required, workspace_limit)
    ho, wo = output_dims(cfg)
    parts = np.empty((cfg.hf * cfg.wf, cfg.n, cfg.m, ho, wo), dtype=np.float32)
    stats = nat.RunStatsC()
    st = nat.lib().b2c_stage1_host(ctypes.byref(nat.desc(cfg)), inp.data.ctypes.data, filters.data.ctypes.data,
                                   parts.ctypes.data, ctypes.byref(plan._c()), ctypes.byref(device._c()),
                                   int(workspace_limit), int(gpu), ctypes.byref(stats))
    nat.check(st, required=required, limit=workspace_limit)
    return PartialSums(parts), RunStats(plan.blocks, False, plan.blocks, required)


def stage2_sum(partials: PartialSums, cfg: ConvConfig, *, workers: int = 1,
               gpu: int = -1) -> tuple[Tensor4, RunStats]:
    """Stage 2 alone (twostage.py:175-205): out = +0 + sum over k ascending."""
    ho, wo = output_dims(cfg)
    expected = (cfg.hf * cfg.wf, cfg.n, cfg.m, ho, wo)
    if partials.data.shape != expected:
        raise ShapeMismatch(f"partials dims {partials.data.shape} != {expected} implied by config")
    parts = np.ascontiguousarray(partials.data, dtype=np.float32)
    out = np.empty((cfg.n, cfg.m, ho, wo), dtype=np.float32)
    stats = nat.RunStatsC()
    st = nat.lib().b2c_stage2_host(ctypes.byref(nat.desc(cfg)), parts.ctypes.data, out.ctypes.data, int(gpu),
                                   ctypes.byref(stats))
    nat.check(st)
    return Tensor4(out), RunStats(stage2_invoked=True)


def conv_forward(inp: Tensor4, filters: Tensor4, cfg: ConvConfig, *, gpu: int = -1,
                 engine: str = "fused") -> Tensor4:
    """Fused-engine convolution for any stride >= 1 and any padding (the
    operand contract of reference.conv_naive, reference.py:58-83), host in /
    host out."""
    _check_operands(inp, filters, cfg, stride1=False)
    ho, wo = output_dims(cfg)
    out = np.empty((cfg.n, cfg.m, ho, wo), dtype=np.float32)
    st = nat.lib().b2c_conv_host(ctypes.byref(nat.desc(cfg)), inp.data.ctypes.data, filters.data.ctypes.data,
                                 out.ctypes.data, nat.ENGINES[engine], None, None, 0, int(gpu), None)
    nat.check(st)
    return Tensor4(out)


def conv_forward_layers(layers, *, engine: str = "fused", gpu: int = -1) -> list[Tensor4]:
    """A sequence of independent convolutions ``[(inp, filters, cfg), ...]``
    (e.g. every layer of a network for one batch) from host buffers: the
    host-to-device copies, the convolutions and the device-to-host copies of
    consecutive layers overlap (b2c_conv_host_layers).  The batched form of
    calling ``conv_forward`` in a loop, as the reference harness does
    (bench.py:91-163)."""
    if engine not in ("fused", "tf32x3", "tf32"):
        raise ValueError(f"conv_forward_layers runs the fused or tensor-core engines, got {engine!r}")
    n = len(layers)
    descs = (nat.ConvDesc * max(n, 1))()
    outs, keep = [], []
    xp = (ctypes.c_void_p * max(n, 1))()
    wp = (ctypes.c_void_p * max(n, 1))()
    yp = (ctypes.c_void_p * max(n, 1))()
    for i, (inp, filters, cfg) in enumerate(layers):
        _check_operands(inp, filters, cfg, stride1=False)
        descs[i] = nat.desc(cfg)
        ho, wo = output_dims(cfg)
        out = np.empty((cfg.n, cfg.m, ho, wo), dtype=np.float32)
        outs.append(Tensor4(out))
        keep += [inp.data, filters.data, out]
        xp[i], wp[i], yp[i] = inp.data.ctypes.data, filters.data.ctypes.data, out.ctypes.data
    st = nat.lib().b2c_conv_host_layers(n, descs, xp, wp, yp, nat.ENGINES[engine], int(gpu))
    nat.check(st)
    return outs
