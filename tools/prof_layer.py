"""Run one layer a few times (ncu target): python tools/prof_layer.py WORKLOAD N LAYER_NAME [engine]
(B2C_FAMILY=<family name> [B2C_SPLITS=k] forces the plan)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, workloads as W

wl, n, name = sys.argv[1], int(sys.argv[2]), sys.argv[3]
engine = sys.argv[4] if len(sys.argv) > 4 else "fused"
cfg = next(c for c in W.layers(wl, n) if c.name == name)
fam = os.environ.get("B2C_FAMILY")
from paper_2103_16234_b200.execmodel import family_names
sp = int(os.environ.get("B2C_SPLITS", "0"))
L = ConvLayer(cfg, engine, family=family_names().index(fam), splits=sp) if fam else ConvLayer(cfg, engine)
print(cfg, L.family, L.grid, flush=True)
x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda") * 2 - 1
w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda") * 2 - 1
y = L(x, w)
for _ in range(4):
    L(x, w, out=y)
torch.cuda.synchronize()
