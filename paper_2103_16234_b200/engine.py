"""Torch-facing entry: convolution of CUDA-resident tensors through the C ABI.

``conv2d(x, w, stride, padding)`` takes exactly ``torch.nn.functional.conv2d``'s
(stride, padding) arguments with dilation=1, groups=1, no bias, on fp32 NCHW
contiguous CUDA tensors, and launches the hand-written sm_100a kernels on the
caller's current stream (so it composes with CUDA graphs and multi-stream
code).  PyTorch provides only device memory and the stream: there is no torch
compute and no fallback — if the native library is absent this raises.

``ConvLayer`` pre-resolves the descriptor and tile plan once for repeated
calls on one shape (the per-call overhead is then one ctypes call).
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
        self._ws = None
        self.split_workspace_bytes = int(self._tiles.workspace_bytes) if engine == "fused" else 0
        self._split_ws = None

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

    def __call__(self, x, w, out=None, stream=None):
        import torch

        if out is None:
            out = torch.empty(self.output_shape(), dtype=torch.float32, device=x.device)
        s = stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
        if self.engine == "fused":
            ws_ptr, ws_len = None, 0
            if self.split_workspace_bytes:
                if self._split_ws is None or self._split_ws.device != x.device:
                    self._split_ws = torch.empty(self.split_workspace_bytes, dtype=torch.uint8, device=x.device)
                ws_ptr, ws_len = self._split_ws.data_ptr(), self.split_workspace_bytes
            st = self._lib.b2c_conv2d_forward(ctypes.byref(self._desc), x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                              ws_ptr, ws_len, ctypes.byref(self._tiles), ctypes.c_void_p(s))
            nat.check(st)
        elif self.tensor_core:
            if self.workspace_bytes and (self._ws is None or self._ws.device != x.device):
                self._ws = torch.empty(self.workspace_bytes // 4, dtype=torch.float32, device=x.device)
            ws_ptr = self._ws.data_ptr() if self.workspace_bytes else None
            st = self._lib.b2c_conv2d_forward_tc(ctypes.byref(self._desc), x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                                 ws_ptr, self.workspace_bytes, self._engine_id, ctypes.byref(self._tc),
                                                 ctypes.c_void_p(s))
            nat.check(st)
        else:
            if self.workspace_bytes and (self._ws is None or self._ws.device != x.device):
                self._ws = torch.empty(self.workspace_bytes // 4, dtype=torch.float32, device=x.device)
            ws_ptr = self._ws.data_ptr() if self.workspace_bytes else None
            stats = nat.RunStatsC()
            st = self._lib.b2c_conv_twostage(ctypes.byref(self._desc), x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                             ws_ptr, self.workspace_bytes, None, None, 1 << 62, ctypes.c_void_p(s),
                                             ctypes.byref(stats))
            nat.check(st)
        return out


_layer_cache: dict = {}


def conv2d(x, w, stride=1, padding=0, *, engine: str = "fused", out=None):
    """``F.conv2d(x, w, stride=stride, padding=padding)`` on B200 kernels."""
    _check_tensor(x, "input")
    _check_tensor(w, "filters")
    if w.device != x.device:
        raise ShapeMismatch("input and filters must be on the same device")
    cfg = config_for(x, w, stride, padding)
    key = (cfg.as_tuple(), engine, x.device.index)
    layer = _layer_cache.get(key)
    if layer is None:
        layer = _layer_cache[key] = ConvLayer(cfg, engine)
    if out is not None:
        _check_tensor(out, "out")
        if tuple(out.shape) != layer.output_shape():
            raise ShapeMismatch(f"out has shape {tuple(out.shape)}, expected {layer.output_shape()}")
    return layer(x, w, out=out)
