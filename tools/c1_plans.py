"""Time forced fused plans on one layer (graph of 20 launches, median of 3):
    python tools/c1_plans.py WL N LAYER"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, family_names, matching_families, workloads as W
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
from autotune import time_layer
wl, n, name = sys.argv[1], int(sys.argv[2]), sys.argv[3]
cfg = next(c for c in W.layers(wl, n) if c.name == name)
x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda"); w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
names = family_names()
auto = ConvLayer(cfg); y = torch.empty(auto.output_shape(), device="cuda")
print(json.dumps({"plan": "auto:" + auto.family, "splits": auto.splits, "us": round(time_layer(auto, x, w, y), 2)}))
rows = []
for f in matching_families(cfg):
    for sp in (1, 2, 4, 8, 16):
        for red in ((0,) if sp == 1 else (1, 2)):
            try:
                L = ConvLayer(cfg, family=f, splits=sp, reduce=red)
            except Exception:
                continue
            if L.splits != sp:
                continue
            rows.append((time_layer(L, x, w, y), L.family, sp))
for t, fam, sp in sorted(rows)[:12]:
    print(json.dumps({"plan": fam, "splits": sp, "us": round(t, 2)}))
