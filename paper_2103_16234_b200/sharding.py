"""Batch-sharded forward convolution over the GPUs of one node.

The path shards naturally: out[n] depends only on inp[n] and the full filter
bank.  Each rank (one process per GPU, torchrun) convolves a
contiguous slab of images [lo, hi) with a replicated filter bank — no
collective on the hot path.  Only when a single-device result is requested is
the NCHW output gathered (NCCL over NVLink on GPUs; any torch.distributed
backend works, gloo is used by the CPU tests).

Per image, the arithmetic does not depend on the shard (the
reference's worker independence, test_acceptance.py:179-213):
the two-stage engine's order is fixed by (c, hf, wf); the fused engine's by
(c, hf, wf, splits) and the tensor-core engines' by (mode, splits).  The
planner would adapt the split to the per-rank batch, so ``shard_layer`` pins
every order-relevant plan field to the plan of the GLOBAL batch: a rank's slab
is then bitwise identical to the same images of the unsharded result for any
world size (tests/test_gpu_sharding.py).
"""

from __future__ import annotations

from typing import Callable, Optional

from .configs import ConvConfig


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced image range [lo, hi) of ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    return rank * n // world, (rank + 1) * n // world


def shard_config(cfg: ConvConfig, world: int, rank: int) -> ConvConfig:
    lo, hi = shard_range(cfg.n, world, rank)
    return cfg.with_batch(max(hi - lo, 0)) if hi > lo else cfg.with_batch(1)


def _split_bounds(layer, c: int) -> tuple:
    """First input channel of each split range of a fused plan."""
    bc, splits = int(layer._tiles.bc), int(layer.splits)
    per = -(-(-(-c // bc)) // splits) * bc  # chunks per split x channels per chunk
    return tuple(min(c, s * per) for s in range(splits))


def shard_layer(cfg: ConvConfig, local_cfg: ConvConfig, engine: str = "fused"):
    """The ConvLayer a rank runs for its slab ``local_cfg`` of the global
    layer ``cfg``, with the summation-order fields of its plan pinned to the
    global plan (fused: the channel ranges of the split-C reduction, set by
    the split count and the kernel family's channels per chunk; tensor core:
    A-operand mode and split-K count), so its outputs do not depend on the
    world size.  The slab's own plan (measured registry or planner) is kept
    whenever it already agrees; otherwise its kernel family (else the global
    plan's) is kept and only the order-relevant fields are forced."""
    from .engine import ConvLayer
    from .errors import InvalidPlan

    local = ConvLayer(local_cfg, engine)
    if local_cfg.as_tuple() == cfg.as_tuple() or engine == "twostage":
        return local
    ref = ConvLayer(cfg, engine)
    if engine == "fused":
        # the summation order is fixed by the channel ranges of the splits,
        # which follow from (splits, channels per pipeline chunk)
        if _split_bounds(local, cfg.c) == _split_bounds(ref, cfg.c):
            return local
        reduce = ref.reduce if ref.splits > 1 else 0
        for fam in (int(local._tiles.family), int(ref._tiles.family)):
            try:
                cand = ConvLayer(local_cfg, engine, family=fam, splits=ref.splits, reduce=reduce)
            except InvalidPlan:
                continue
            if _split_bounds(cand, cfg.c) == _split_bounds(ref, cfg.c):
                return cand
        raise InvalidPlan(f"no plan for the {local_cfg.n}-image shard reproduces the channel split of {cfg.name}")
    if local.splits == ref.splits and int(local._tc.mode) == int(ref._tc.mode):
        return local
    try:
        return ConvLayer(local_cfg, engine, splits=ref.splits, tc_mode=int(ref._tc.mode),
                         filters_per_tile=int(local._tc.filters_per_tile))
    except InvalidPlan:
        return ConvLayer(local_cfg, engine, splits=ref.splits, tc_mode=int(ref._tc.mode))


class ShardedConv:
    """Forward convolution of a global batch split across ``world`` ranks.

    ``compute(cfg_local, x_local, w) -> y_local`` defaults to the B200 engine
    (``ConvLayer``) on the rank's current CUDA device; tests inject another
    callable to exercise the sharding/gather plumbing on CPU.
    """

    def __init__(self, cfg: ConvConfig, group=None, engine: str = "fused", compute: Optional[Callable] = None):
        import torch.distributed as dist

        self.cfg = cfg
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.lo, self.hi = shard_range(cfg.n, self.world, self.rank)
        self.local_cfg = cfg.with_batch(self.hi - self.lo) if self.hi > self.lo else None
        self._compute = compute
        if compute is None and self.local_cfg is not None:
            self._layer = shard_layer(cfg, self.local_cfg, engine)
            self._compute = lambda c, x, w: self._layer(x, w)

    def local_slice(self, x_global):
        """This rank's images of a global batch tensor."""
        return x_global[self.lo:self.hi]

    def broadcast_filters(self, w, src: int = 0):
        """Replicate the filter bank from ``src`` (once, at setup)."""
        import torch.distributed as dist

        if self.world > 1:
            if w.is_cuda and dist.get_backend(self.group) == "gloo":
                h = w.cpu()
                dist.broadcast(h, src, group=self.group)
                w.copy_(h)
            else:
                dist.broadcast(w, src, group=self.group)
        return w

    def forward(self, x_local, w):
        """The hot path: this rank's slab only, no communication."""
        if self.local_cfg is None:
            return None
        return self._compute(self.local_cfg, x_local, w)

    def gather(self, y_local, dst: Optional[int] = None):
        """Assemble the global [n, m, ho, wo] output on every rank
        (``dst=None``: one all_gather) or on rank ``dst`` only (one gather:
        the other ranks send their slab and get None).  Slabs are padded to
        the largest shard so every rank moves the same byte count; NCCL over
        NVLink on GPUs, gloo on CPU."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return y_local
        biggest = -(-self.cfg.n // self.world)
        from .configs import output_dims

        ho, wo = output_dims(self.cfg)
        dev = y_local.device if y_local is not None else torch.device("cpu")
        if y_local is not None and y_local.shape[0] == biggest and y_local.is_contiguous():
            pad = y_local
        else:
            pad = torch.zeros((biggest, self.cfg.m, ho, wo), dtype=torch.float32, device=dev)
            if y_local is not None:
                pad[: y_local.shape[0]].copy_(y_local)
        on_host = pad.is_cuda and dist.get_backend(self.group) == "gloo"
        if on_host:  # gloo moves host memory; NCCL (the GPU backend) gathers device memory directly
            pad = pad.cpu()
        if dst is None:
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(parts, pad, group=self.group)
        else:
            parts = [torch.empty_like(pad) for _ in range(self.world)] if self.rank == dst else None
            dist.gather(pad, parts, dst=dst, group=self.group)
            if self.rank != dst:
                return None
        sizes = [shard_range(self.cfg.n, self.world, r) for r in range(self.world)]
        out = torch.cat([p[: hi - lo] for (lo, hi), p in zip(sizes, parts)], dim=0)
        return out.to(dev) if on_host else out

    def __call__(self, x_local, w, gather: bool = False, dst: Optional[int] = None):
        y = self.forward(x_local, w)
        return self.gather(y, dst) if gather else y
