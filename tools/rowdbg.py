import sys, torch
sys.path.insert(0, '.')
import paper_2103_16234_b200 as pk
cfgs = [pk.ConvConfig("p3", n=3, c=37, h=14, w=14, m=40, hf=3, wf=3, pad_h=1, pad_w=1),
        pk.ConvConfig("p5", n=2, c=20, h=13, w=11, m=33, hf=5, wf=5, pad_h=2, pad_w=2),
        pk.ConvConfig("p4", n=3, c=64, h=14, w=14, m=64, hf=3, wf=3, pad_h=1, pad_w=1),
        pk.ConvConfig("ps2", n=2, c=24, h=15, w=15, m=20, hf=3, wf=3, stride=2, pad_h=1, pad_w=1),
        pk.ConvConfig("p7", n=2, c=3, h=30, w=30, m=20, hf=7, wf=7, stride=2, pad_h=3, pad_w=3),
        pk.ConvConfig("p1", n=5, c=70, h=7, w=7, m=50, hf=1, wf=1),
        pk.ConvConfig("p1s2", n=3, c=40, h=14, w=13, m=36, hf=1, wf=1, stride=2),
        pk.ConvConfig("p1v", n=3, c=64, h=14, w=14, m=80, hf=1, wf=1),
        pk.ConvConfig("p1t", n=5, c=72, h=16, w=16, m=100, hf=1, wf=1),
        pk.ConvConfig("p1big", n=3, c=32, h=28, w=28, m=64, hf=1, wf=1)]
for cfg in cfgs:
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), generator=g, device="cuda") * 2 - 1
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), generator=g, device="cuda") * 2 - 1
    ref = torch.nn.functional.conv2d(x.double(), w.double(), padding=(cfg.pad_h, cfg.pad_w), stride=cfg.stride)
    for fam in pk.matching_families(cfg):
        L = pk.ConvLayer(cfg, family=fam, splits=2 if cfg.c >= 64 else 1)
        if not any(k in L.family for k in ('row', 'rws', '1x1ws', '1x1t')): continue
        print(cfg.name, fam, L.grid, flush=True)
        y = L(x, w); torch.cuda.synchronize()
        print("  err", ((y.double()-ref).abs().max()/ref.abs().max()).item(), flush=True)
