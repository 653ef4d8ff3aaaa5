"""Run one layer with a forced family a few times (ncu target):
python tools/prof_layer_fam.py WORKLOAD N LAYER FAMILY [SPLITS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, family_names
from paper_2103_16234_b200 import workloads as W

wl, n, name, fam = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
sp = int(sys.argv[5]) if len(sys.argv) > 5 else 1
cfg = next(c for c in W.layers(wl, n) if c.name == name)
L = ConvLayer(cfg, family=family_names().index(fam), splits=sp)
print(cfg, L.family, L.grid, flush=True)
x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda") * 2 - 1
w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda") * 2 - 1
y = L(x, w)
for _ in range(4):
    L(x, w, out=y)
torch.cuda.synchronize()
