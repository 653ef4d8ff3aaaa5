"""Development: per-role cycle breakdown of CTA 0 of the tensor-core kernel (B2C_TC_DEBUG dump)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["B2C_TC_DEBUG"] = "/tmp/tc_roles.bin"
import torch
from paper_2103_16234_b200 import ConvLayer, workloads as W
for spec in sys.argv[1:]:
    wl, n, name, eng = spec.split(":")
    cfg = next(c for c in W.layers(wl, int(n)) if c.name == name)
    L = ConvLayer(cfg, eng)
    x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda")
    w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
    L(x, w); torch.cuda.synchronize()
    d = np.fromfile("/tmp/tc_roles.bin", dtype=np.uint32)
    kb = (cfg.c + 15) // 16 * cfg.hf * cfg.wf
    names = ["mma_total", "mma_wait", "mma_issue", "prod_wait_empty", "prod_total", "ld_wait_empty", "ld_store",
             "ld_wait_full", "ld_split", "ld_fence_arrive", "ld_gather", "ld_total"]
    print(spec, L.family, "k-blocks", kb)
    for i, nm in enumerate(names):
        print(f"   {nm:18s} {d[2 + i]:12d} clk  {d[2 + i] / kb:8.1f} clk/kb")
