"""Per-CTA trace of one forced launch: python tools/trace_layer.py WL N LAYER FAMILY SPLITS OUT.csv"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, workloads as W, family_names
wl, n, name, fam, sp, out = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5]), sys.argv[6]
cfg = next(c for c in W.layers(wl, n) if c.name == name)
L = ConvLayer(cfg, family=family_names().index(fam), splits=sp)
x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda"); w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
y = L(x, w); y = L(x, w); torch.cuda.synchronize()
os.environ["B2C_TRACE_FILE"] = out
L(x, w, out=y); torch.cuda.synchronize()
