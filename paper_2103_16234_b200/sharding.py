"""Batch-sharded forward convolution over the GPUs of one node.

The path shards naturally: out[n] depends only on inp[n] and the full filter
bank.  Each rank (one process per GPU, torchrun) convolves a
contiguous slab of images [lo, hi) with a replicated filter bank — no
collective on the hot path.  Only when a single-device result is requested is
the NCHW output gathered (NCCL over NVLink on GPUs; any torch.distributed
backend works, gloo is used by the CPU tests).

Per image, the arithmetic does not depend on the shard: the two-stage engine
is bitwise identical for any world size, and the fused engine is too when the
reduction split is pinned (``splits=``), since its planner otherwise adapts
the split to the per-rank batch.
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


class ShardedConv:
    """Forward convolution of a global batch split across ``world`` ranks.

    ``compute(cfg_local, x_local, w) -> y_local`` defaults to the B200 engine
    (``ConvLayer``) on the rank's current CUDA device; tests inject another
    callable to exercise the sharding/gather plumbing on CPU.
    """

    def __init__(self, cfg: ConvConfig, group=None, engine: str = "fused", splits: int = 0,
                 compute: Optional[Callable] = None):
        import torch.distributed as dist

        self.cfg = cfg
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.lo, self.hi = shard_range(cfg.n, self.world, self.rank)
        self.local_cfg = cfg.with_batch(self.hi - self.lo) if self.hi > self.lo else None
        self._compute = compute
        if compute is None and self.local_cfg is not None:
            from .engine import ConvLayer

            self._layer = ConvLayer(self.local_cfg, engine, splits=splits)
            self._compute = lambda c, x, w: self._layer(x, w)

    def local_slice(self, x_global):
        """This rank's images of a global batch tensor."""
        return x_global[self.lo:self.hi]

    def broadcast_filters(self, w, src: int = 0):
        """Replicate the filter bank from ``src`` (once, at setup)."""
        import torch.distributed as dist

        if self.world > 1:
            dist.broadcast(w, src, group=self.group)
        return w

    def forward(self, x_local, w):
        """The hot path: this rank's slab only, no communication."""
        if self.local_cfg is None:
            return None
        return self._compute(self.local_cfg, x_local, w)

    def gather(self, y_local, dst: Optional[int] = None):
        """Assemble the global [n, m, ho, wo] output on every rank
        (``dst=None``) or on rank ``dst`` only (others get None).  Slabs are
        padded to the largest shard so one all_gather suffices."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return y_local
        biggest = -(-self.cfg.n // self.world)
        from .configs import output_dims

        ho, wo = output_dims(self.cfg)
        dev = y_local.device if y_local is not None else torch.device("cpu")
        pad = torch.zeros((biggest, self.cfg.m, ho, wo), dtype=torch.float32, device=dev)
        if y_local is not None:
            pad[: y_local.shape[0]].copy_(y_local)
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        if dst is not None and self.rank != dst:
            return None
        out = [p[: shard_range(self.cfg.n, self.world, r)[1] - shard_range(self.cfg.n, self.world, r)[0]]
               for r, p in enumerate(parts)]
        return torch.cat(out, dim=0)

    def __call__(self, x_local, w, gather: bool = False, dst: Optional[int] = None):
        y = self.forward(x_local, w)
        return self.gather(y, dst) if gather else y
