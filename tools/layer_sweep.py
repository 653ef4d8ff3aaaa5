"""Time one layer under every matching kernel family x split (CUDA-graph
replays, CUDA events).  Development aid for the planner.
    python tools/layer_sweep.py WORKLOAD N LAYER [LAYER...]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, ConvConfig, workloads as W, matching_families, select_tiles, family_names

def time_layer(L, x, w, y, reps=50):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        L(x, w, out=y); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                L(x, w, out=y)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); b.synchronize()
    return a.elapsed_time(b) / reps * 1e3

wl, n = sys.argv[1], int(sys.argv[2])
names = sys.argv[3:]
fams = family_names()
for cfg in W.layers(wl, n):
    if names and cfg.name not in names and names != ["all"]:
        continue
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda")
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
    auto = ConvLayer(cfg)
    y = torch.empty(auto.output_shape(), device="cuda")
    res = {"layer": cfg.name, "gflop": cfg.flops / 1e9, "auto": [auto.family, auto.splits, round(time_layer(auto, x, w, y), 2)]}
    trials = []
    for f in matching_families(cfg):
        for sp in (1, 2, 4, 8, 16):
            try:
                L = ConvLayer(cfg, family=f, splits=sp)
            except Exception:
                continue
            trials.append((round(time_layer(L, x, w, y), 2), fams[f], L.splits))
    trials.sort()
    res["best"] = trials[:6]
    print(json.dumps(res), flush=True)
