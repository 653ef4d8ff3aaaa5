"""Batch sharding on the GPU engine.

Outputs must be bitwise identical for G = 1 vs 2/4/8 (the reference's
worker/plan independence, /root/reference/SPEC.md:314-315;
pkg/tests/test_acceptance.py:179-213).  One GPU is available, so the shards
of ResNet-50 at N=256 (BASELINE config 5) run one after another on it, each
through ``shard_layer`` exactly as a rank would; a world-2 ``ShardedConv``
(two processes, gloo, both on cuda:0) exercises the real wrapper with the
CUDA engine, including the output gather.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch

import paper_2103_16234_b200 as pk
from paper_2103_16234_b200 import workloads as W
from paper_2103_16234_b200.sharding import ShardedConv, shard_layer, shard_range

pytestmark = pytest.mark.gpu


def _operands(cfg, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
    return x, w


@pytest.mark.parametrize("engine", ["fused", "tf32x3"])
def test_resnet50_n256_shards_bitwise_equal_unsharded(engine):
    bad = []
    for i, cfg in enumerate(W.layers("c5", 256)):
        x, w = _operands(cfg, 500 + i)
        full = shard_layer(cfg, cfg, engine)(x, w)
        for world in (2, 4, 8):
            for r in range(world):
                lo, hi = shard_range(cfg.n, world, r)
                layer = shard_layer(cfg, cfg.with_batch(hi - lo), engine)
                y = layer(x[lo:hi], w)
                if not torch.equal(y, full[lo:hi]):
                    bad.append(f"{cfg.name} G={world} rank {r} ({layer.family})")
        del x, w, full
        torch.cuda.empty_cache()
    assert not bad, bad


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    outs = []
    for name in ("layer3.0.conv2", "layer4.1.conv1", "layer1.0.downsample"):
        cfg = next(c for c in W.layers("c5", 6) if c.name == name)
        x, w = _operands(cfg, 77)
        sc = ShardedConv(cfg)
        sc.broadcast_filters(w)
        y_all = sc(sc.local_slice(x), w, gather=True)
        y_root = sc(sc.local_slice(x), w, gather=True, dst=0)
        if rank == 0:
            outs.append((name, y_all.cpu(), y_root.cpu()))
        else:
            assert y_root is None
    if rank == 0:
        q.put(outs)
    dist.barrier()
    dist.destroy_process_group()


def test_world2_sharded_conv_cuda_engine_gathers_the_unsharded_result():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for name, y_all, y_root in outs:
        cfg = next(c for c in W.layers("c5", 6) if c.name == name)
        x, w = _operands(cfg, 77)
        want = shard_layer(cfg, cfg)(x, w).cpu()
        assert torch.equal(y_all, want) and torch.equal(y_root, want), name
