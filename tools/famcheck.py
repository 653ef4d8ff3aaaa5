"""Check every family x split on one BASELINE layer against each other and the
f64 oracle (GPU): python tools/famcheck.py WORKLOAD N LAYER [splits,...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2103_16234_b200 as pk
from paper_2103_16234_b200 import workloads as W

wl, n, name = sys.argv[1], int(sys.argv[2]), sys.argv[3]
splits = [int(s) for s in (sys.argv[4] if len(sys.argv) > 4 else "1,2,3").split(",")]
reduces = [int(s) for s in (sys.argv[5] if len(sys.argv) > 5 else "0").split(",")]
cfg = next(c for c in W.layers(wl, n) if c.name == name)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
ref = torch.nn.functional.conv2d(x.double(), w.double(), stride=cfg.stride, padding=(cfg.pad_h, cfg.pad_w))
outs = {}
for fam in pk.matching_families(cfg):
    for sp, red in ((a, b) for a in splits for b in reduces):
        try:
            L = pk.ConvLayer(cfg, family=fam, splits=sp, reduce=red)
        except Exception:
            continue
        print("run", L.family, sp, red, flush=True)
        if L.splits != sp:
            continue
        y = L(x, w)
        err = ((y.double() - ref).abs().max() / ref.abs().max()).item()
        key = (sp, L._tiles.bc)
        same = [f for (f, s2, b2), v in outs.items() if (s2, b2) == key and torch.equal(v, y)]
        diff = [f for (f, s2, b2), v in outs.items() if (s2, b2) == key and not torch.equal(v, y)]
        outs[(L.family, sp, L._tiles.bc)] = y
        print(f"{L.family:26s} s{sp} bc{L._tiles.bc} err {err:.2e} same={same[:2]} DIFF={diff[:3]}", flush=True)
