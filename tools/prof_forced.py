"""Run one layer with a forced family/split a few times (ncu target).
    python tools/prof_forced.py WORKLOAD N LAYER FAMILY_NAME SPLITS"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, workloads as W, family_names

wl, n, name, fam, sp = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
cfg = next(c for c in W.layers(wl, n) if c.name == name)
L = ConvLayer(cfg, family=family_names().index(fam), splits=sp)
print(cfg, L.family, L.grid, L.splits, flush=True)
x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda")
w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
y = L(x, w)
for _ in range(4):
    L(x, w, out=y)
torch.cuda.synchronize()
