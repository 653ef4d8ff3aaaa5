"""Batch sharding across ranks: world_size-2 gloo processes on
CPU exercise the shard arithmetic, the filter broadcast and the output gather;
the per-rank compute is injected (the oracle here — tests may use it as the
checker), so the plumbing is verified without a GPU.  The sharded result
must be bitwise identical to the single-process result."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_16234_b200 import ConvConfig
from paper_2103_16234_b200.sharding import ShardedConv, shard_range


def test_shard_range_partitions():
    for n in (1, 2, 7, 32, 256, 255):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [h - l for l, h in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    cfg = ConvConfig("s", n=n, c=5, h=9, w=7, m=6, hf=3, wf=3, pad_h=1, pad_w=1)
    x = torch.from_numpy(oracle.make_uniform((n, 5, 9, 7), 11))
    w = torch.zeros((6, 5, 3, 3)) if rank else torch.from_numpy(oracle.make_uniform((6, 5, 3, 3), 12))

    def compute(c, xl, wl):
        return torch.from_numpy(oracle.conv_naive(c, xl.numpy(), wl.numpy()))

    sc = ShardedConv(cfg, compute=compute)
    sc.broadcast_filters(w)
    y_all = sc(sc.local_slice(x), w, gather=True)
    y_root = sc(sc.local_slice(x), w, gather=True, dst=0)
    if rank == 0:
        q.put((y_all.numpy().tobytes(), y_root.numpy().tobytes(), tuple(y_all.shape)))
    else:
        assert y_root is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [4, 5])
def test_gloo_world2_gather_is_bitwise_single_process(n):
    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got_all, got_root, shape = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = ConvConfig("s", n=n, c=5, h=9, w=7, m=6, hf=3, wf=3, pad_h=1, pad_w=1)
    want = oracle.conv_naive(cfg, oracle.make_uniform((n, 5, 9, 7), 11), oracle.make_uniform((6, 5, 3, 3), 12))
    assert shape == want.shape
    assert got_all == want.tobytes() and got_root == want.tobytes()


@pytest.mark.gpu
def test_sharded_engine_single_rank_matches_unsharded():
    """With one rank the sharded wrapper runs the B200 engine on the whole batch."""
    import oracle
    import paper_2103_16234_b200 as pk

    cfg = ConvConfig("s", n=6, c=16, h=14, w=14, m=24, hf=3, wf=3, pad_h=1, pad_w=1)
    x = torch.from_numpy(oracle.make_uniform(pk.input_dims(cfg), 1)).cuda()
    w = torch.from_numpy(oracle.make_uniform(pk.filter_dims(cfg), 2)).cuda()
    sc = ShardedConv(cfg, engine="twostage")
    y = sc(sc.local_slice(x), w, gather=True)
    assert y.cpu().numpy().tobytes() == oracle.conv_naive(cfg, x.cpu().numpy(), w.cpu().numpy()).tobytes()
    # per-image arithmetic is shard independent: a 2-image slab equals the batch slice
    part = pk.ConvLayer(cfg.with_batch(2), "twostage")(x[2:4], w)
    assert torch.equal(part, y[2:4])
