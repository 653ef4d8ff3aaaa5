"""A/B of kernel families per layer (GPU): every matching fused family (or
those matching --only), split 1 unless --splits, timed as 20 back-to-back
launches in a CUDA graph (median of 3 replays).

    python tools/fam_ab.py c5 256 [--layers a,b] [--only 1x1] [--splits 1,2,4]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, matching_families
from paper_2103_16234_b200 import workloads as W
from autotune import time_layer

ap = argparse.ArgumentParser()
ap.add_argument("wl"); ap.add_argument("n", type=int)
ap.add_argument("--layers", default=""); ap.add_argument("--only", default="")
ap.add_argument("--splits", default="1")
ap.add_argument("--reduce", default="0", help="split-C reduction modes to try (0 planner, 1 planes, 2 DSMEM)")
a = ap.parse_args()
cfgs = W.layers(a.wl, a.n)
if a.layers:
    keep = a.layers.split(",")
    cfgs = [c for c in cfgs if c.name in keep]
seen = set()
for c in cfgs:
    if c.as_tuple() in seen:
        continue
    seen.add(c.as_tuple())
    x = torch.rand((c.n, c.c, c.h, c.w), device="cuda") * 2 - 1
    w = torch.rand((c.m, c.c, c.hf, c.wf), device="cuda") * 2 - 1
    auto = ConvLayer(c)
    y = torch.empty(auto.output_shape(), device="cuda")
    res = []
    for fam in matching_families(c):
        for sp, red in ((int(s), int(r)) for s in a.splits.split(",") for r in a.reduce.split(",")):
            try:
                L = ConvLayer(c, family=fam, splits=sp, reduce=red)
            except Exception:  # noqa: BLE001
                continue
            if a.only and a.only not in L.family:
                continue
            us = time_layer(L, x, w, y)
            res.append((us, L.family, sp))
    ta = time_layer(auto, x, w, y)
    res.sort()
    line = "  ".join(f"{f}/s{sp}:{us:.1f}({c.flops / us / 1e6:.1f})" for us, f, sp in res[:6])
    print(f"{c.name:22s} auto {auto.family}/s{auto.splits} {ta:.1f}us ({c.flops / ta / 1e6:.1f} TF) | {line}", flush=True)
    del x, w, y
    torch.cuda.empty_cache()
