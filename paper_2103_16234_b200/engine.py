"""Torch-facing entry: convolution of CUDA-resident tensors through the C ABI.

``conv2d(x, w, stride, padding)`` takes exactly ``torch.nn.functional.conv2d``'s
(stride, padding) arguments with dilation=1, groups=1, no bias, on fp32 NCHW
contiguous CUDA tensors, and launches the hand-written sm_100a kernels on the
caller's current stream (so it composes with CUDA graphs and multi-stream
code).  PyTorch provides only device memory and the stream: there is no torch
compute and no fallback — if the native library is absent this raises.

``conv2d`` dispatches through the registered PyTorch operator
``torch.ops.b2conv.conv2d`` (csrc/torch_ext.cpp, with a Meta kernel for
fake-tensor tracing); ``ConvLayer`` pre-resolves the descriptor and tile plan
once for repeated calls on one shape (the per-call overhead is then one ctypes
call) and is what the benchmark and the sharded wrapper use.
"""

from __future__ import annotations

import ctypes

from . import _native as nat
from .configs import ConvConfig, output_dims
from .errors import ShapeMismatch, Unsupported


def _pair(v) -> tuple[int, int]:
    if isinstance(v, (tuple, list)):
        if len(v) != 2:
            raise ValueError(f"expected an int or a pair, got {v!r}")
        return int(v[0]), int(v[1])
    return int(v), int(v)


def config_for(x, w, stride=1, padding=0, name: str = "torch") -> ConvConfig:
    if x.dim() != 4 or w.dim() != 4:
        raise ShapeMismatch(f"expected 4-D NCHW input and MCHW filters, got {tuple(x.shape)} / {tuple(w.shape)}")
    n, c, h, wd = (int(v) for v in x.shape)
    m, cw, hf, wf = (int(v) for v in w.shape)
    if cw != c:
        raise ShapeMismatch(f"filter depth {cw} != input channels {c}")
    sh, sw = _pair(stride)
    if sh != sw:
        raise Unsupported(f"one stride for both axes is supported (configs.py:26), got {(sh, sw)}")
    ph, pw = _pair(padding)
    return ConvConfig(name, n=n, c=c, h=h, w=wd, m=m, hf=hf, wf=wf, stride=sh, pad_h=ph, pad_w=pw)


def _check_tensor(t, what: str) -> None:
    import torch

    if not t.is_cuda:
        raise ShapeMismatch(f"{what} must be a CUDA tensor (the B200 engine has no CPU path)")
    if t.dtype != torch.float32:
        raise ShapeMismatch(f"{what} must be float32, got {t.dtype}")
    if not t.is_contiguous():
        raise ShapeMismatch(f"{what} must be contiguous NCHW")


class ConvLayer:
    """A resolved forward convolution for one configuration."""

    def __init__(self, cfg: ConvConfig, engine: str = "fused", family: int = -1, splits: int = 0,
                 filters_per_tile: int = 0, tc_mode: int = 0, reduce: int = 0, tc_m_halves: int = 0):
        if engine not in nat.ENGINES:
            raise ValueError(f"unknown engine {engine!r}")
        if engine == "twostage" and cfg.stride != 1:
            raise Unsupported(f"two-stage convolution requires stride 1, got {cfg.stride}")
        self.cfg = cfg
        self.engine = engine
        self._desc = nat.desc(cfg)
        self._lib = nat.lib()
        self._tiles = nat.TilePlanC()
        self._tiles.family = int(family)
        self._tiles.splits = int(splits)
        self._tiles.reduce = int(reduce)  # split-C: 0 planner, 1 partial planes + stage 2, 2 DSMEM cluster
        self._engine_id = nat.ENGINES[engine]
        self.tensor_core = engine in ("tf32x3", "tf32")
        if self.tensor_core:
            self._tc = nat.TcPlanC()
            self._tc.filters_per_tile = int(filters_per_tile)
            self._tc.splits = int(splits)
            self._tc.mode = int(tc_mode)
            self._tc.m_halves = int(tc_m_halves)  # halo plans: 128-pixel M slices per tile (0 = planner)
            nat.check(self._lib.b2c_tc_select_tiles(ctypes.byref(self._desc), self._engine_id, ctypes.byref(self._tc)))
        else:
            e = nat.ENGINE_TWOSTAGE if engine == "twostage" else nat.ENGINE_FUSED
            nat.check(self._lib.b2c_select_tiles(ctypes.byref(self._desc), e, ctypes.byref(self._tiles)))
        self.out_hw = output_dims(cfg)
        self.workspace_bytes = 0
        if self.tensor_core:
            self.workspace_bytes = int(self._tc.workspace_bytes)
        if engine == "twostage" and not (cfg.hf == 1 and cfg.wf == 1):
            self.workspace_bytes = int(self._lib.b2c_workspace_bytes(ctypes.byref(self._desc)))
        self.split_workspace_bytes = int(self._tiles.workspace_bytes) if engine == "fused" else 0
        self._ws_by_stream: dict = {}

    @property
    def family(self) -> str:
        if self.tensor_core:
            t = self._tc
            shape = f"h{t.halo_positions}" if t.mode == 2 else f"x{t.pixels_per_chunk}"
            return (f"{self.engine}_{shape}_n{t.filters_per_tile}_s{t.stages}_k{t.splits}"
                    + ("_flat" if t.flattened else "") + ("_b16c" if t.bf16_corrections else "")
                    + ("_kpack" if t.k_packed else ""))
        name = self._lib.b2c_family_name(self._tiles.family).decode()
        return name + ("_dsm" if self._tiles.splits > 1 and self._tiles.reduce == 2 else "")

    @property
    def grid(self) -> int:
        return int(self._tc.grid if self.tensor_core else self._tiles.grid)

    @property
    def reduce(self) -> int:
        """Split-C reduction of the plan: 0 none, 1 partial planes + stage 2, 2 DSMEM cluster."""
        return 0 if self.tensor_core else int(self._tiles.reduce)

    @property
    def splits(self) -> int:
        return int(self._tc.splits if self.tensor_core else self._tiles.splits)

    def output_shape(self) -> tuple[int, int, int, int]:
        return (self.cfg.n, self.cfg.m, *self.out_hw)

    def _check_operands(self, x, w, out) -> None:
        """The operands must match the resolved configuration exactly: the
        kernels index raw device pointers by ``cfg``, so a mismatch is a
        ShapeMismatch here, never an out-of-bounds access on the device."""
        _check_tensor(x, "input")
        _check_tensor(w, "filters")
        c = self.cfg
        if tuple(x.shape) != (c.n, c.c, c.h, c.w):
            raise ShapeMismatch(f"input has shape {tuple(x.shape)}, layer expects {(c.n, c.c, c.h, c.w)}")
        if tuple(w.shape) != (c.m, c.c, c.hf, c.wf):
            raise ShapeMismatch(f"filters have shape {tuple(w.shape)}, layer expects {(c.m, c.c, c.hf, c.wf)}")
        if w.device != x.device:
            raise ShapeMismatch("input and filters must be on the same device")
        if out is not None:
            _check_tensor(out, "out")
            if tuple(out.shape) != self.output_shape():
                raise ShapeMismatch(f"out has shape {tuple(out.shape)}, expected {self.output_shape()}")
            if out.device != x.device:
                raise ShapeMismatch("out must be on the input's device")

    def _workspace(self, nbytes: int, device, stream_handle: int):
        """Scratch (split-C partial planes, pre-tiled filters) private to one
        (device, stream): calls on different streams never share it, calls on
        one stream are ordered by the stream."""
        import torch

        key = (device.index, stream_handle)
        buf = self._ws_by_stream.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = self._ws_by_stream[key] = torch.empty(nbytes, dtype=torch.uint8, device=device)
        return buf.data_ptr()

    def __call__(self, x, w, out=None, stream=None):
        import torch

        self._check_operands(x, w, out)
        if out is None:
            out = torch.empty(self.output_shape(), dtype=torch.float32, device=x.device)
        s = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
        if self.engine == "fused":
            ws_ptr, ws_len = None, 0
            if self.split_workspace_bytes:
                ws_len = self.split_workspace_bytes
                ws_ptr = self._workspace(ws_len, x.device, s)
            st = self._lib.b2c_conv2d_forward(ctypes.byref(self._desc), x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                              ws_ptr, ws_len, ctypes.byref(self._tiles), ctypes.c_void_p(s))
            nat.check(st)
        elif self.tensor_core:
            ws_ptr = self._workspace(self.workspace_bytes, x.device, s) if self.workspace_bytes else None
            st = self._lib.b2c_conv2d_forward_tc(ctypes.byref(self._desc), x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                                 ws_ptr, self.workspace_bytes, self._engine_id, ctypes.byref(self._tc),
                                                 ctypes.c_void_p(s))
            nat.check(st)
        else:
            ws_ptr = self._workspace(self.workspace_bytes, x.device, s) if self.workspace_bytes else None
            stats = nat.RunStatsC()
            st = self._lib.b2c_conv_twostage(ctypes.byref(self._desc), x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                             ws_ptr, self.workspace_bytes, None, None, 1 << 62, ctypes.c_void_p(s),
                                             ctypes.byref(stats))
            nat.check(st)
        return out


_ops_loaded = False


def torch_ops():
    """``torch.ops.b2conv`` — the PyTorch operator library (csrc/torch_ext.cpp,
    built in-tree as _b2conv_torch.so next to libb2conv.so).  Raises
    DeviceError if it is missing: there is no fallback."""
    global _ops_loaded
    import torch

    if not _ops_loaded:
        from .build import TORCH_LIB

        nat.lib()  # libb2conv.so first: the operator library links it
        if not TORCH_LIB.exists():
            raise nat.DeviceError(f"{TORCH_LIB.name} is not built (python -m paper_2103_16234_b200.build)")
        torch.ops.load_library(str(TORCH_LIB))
        _ops_loaded = True
    return torch.ops.b2conv


def conv2d(x, w, stride=1, padding=0, *, engine: str = "fused", out=None):
    """``F.conv2d(x, w, stride=stride, padding=padding)`` on B200 kernels,
    through the registered operator ``torch.ops.b2conv.conv2d`` (traceable by
    torch.compile / torch.export through its Meta kernel).  Operand errors
    raise the reference's exception classes first (ShapeMismatch,
    Unsupported, InvalidConfig)."""
    if engine not in nat.ENGINES:
        raise ValueError(f"unknown engine {engine!r}")
    _check_tensor(x, "input")
    _check_tensor(w, "filters")
    if w.device != x.device:
        raise ShapeMismatch("input and filters must be on the same device")
    cfg = config_for(x, w, stride, padding)
    if engine == "twostage" and cfg.stride != 1:
        raise Unsupported(f"two-stage convolution requires stride 1, got {cfg.stride}")
    st, pd = [cfg.stride, cfg.stride], [cfg.pad_h, cfg.pad_w]
    ops = torch_ops()
    if out is None:
        return ops.conv2d(x, w, st, pd, engine)
    _check_tensor(out, "out")
    want = (cfg.n, cfg.m, *output_dims(cfg))
    if tuple(out.shape) != want:
        raise ShapeMismatch(f"out has shape {tuple(out.shape)}, expected {want}")
    return ops.conv2d_out(x, w, st, pd, engine, out=out)
