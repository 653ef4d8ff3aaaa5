"""Scaling proxy on ONE GPU (this pool has one GPU per call): the C5 step of
one rank of a G-way batch-sharded run (N = 256/G images, plans pinned to the
global plan by sharding.shard_layer, exactly what bench.py runs under
torchrun), timed as a captured CUDA graph.  Per-GPU throughput at each G, and
the weak-case efficiency G * t(G) vs t(1) if the ranks ran in parallel with no
interference (the gather is not on the step).

    python tools/shard_proxy.py [workload] [global_batch]
"""
import json, os, sys
from types import SimpleNamespace
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2103_16234_b200 import _native as nat
from paper_2103_16234_b200 import workloads as W
from paper_2103_16234_b200.sharding import shard_layer, shard_range

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
nglob = int(sys.argv[2]) if len(sys.argv) > 2 else 256
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
lib = nat.lib()
gcfgs = W.layers(wl, nglob)
flops = sum(c.flops for c in gcfgs)
out = {"workload": wl, "global_batch": nglob, "ranks": {}}
t1 = None
for G in (1, 2, 4, 8):
    lo, hi = shard_range(nglob, G, 0)
    cfgs = [c.with_batch(hi - lo) for c in gcfgs]
    layers = [shard_layer(g, c, "fused") for g, c in zip(gcfgs, cfgs)]
    xs, ws, ys = bench.make_operands(cfgs, dev, 0)
    groups = W.schedule(wl, cfgs)
    ms, launches, _ = bench.time_graph(lib, layers, xs, ws, ys, SimpleNamespace(steps=10, warmup=3), 1, dev, 0, groups)
    ms /= 10
    t1 = t1 or ms
    out["ranks"][G] = {"per_rank_batch": hi - lo, "ms_per_step": round(ms, 4),
                       "per_gpu_tflops": round(flops / G / (ms * 1e-3) / 1e12, 2),
                       "ideal_efficiency": round(t1 / (G * ms), 4)}
    print(json.dumps({G: out["ranks"][G]}), flush=True)
    del xs, ws, ys, layers
    torch.cuda.empty_cache()
print(json.dumps(out))
