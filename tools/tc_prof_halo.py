"""Development: per-role cycles of CTA (0,0) of the halo tensor-core kernel."""
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
    d = np.fromfile("/tmp/tc_roles.bin", dtype=np.uint32).astype(np.int64)
    t = L._tc
    ncb = -(-(-(-cfg.c // 16)) // t.splits)
    taps = cfg.hf * cfg.wf
    print(spec, L.family, "grid", t.grid, "cblocks/CTA", ncb, "taps", taps, "mode", os.environ.get("B2C_TC_MODE", "0"))
    for nm, i in [("mma_total", 2), ("mma_wait_b", 3), ("mma_wait_a", 4), ("prod_wait", 5), ("prod_total", 6),
                  ("ld_wait_a_empty", 7), ("ld_fill", 8), ("ld_total", 13), ("epi_wait_accum", 9)]:
        print(f"   {nm:16s} {d[i]:10d} clk  {d[i] / (ncb * taps):8.1f} /tap")
    print(f"   {'cta_span':16s} {(d[10] - d[11]) & 0xffffffff:10d} clk (setup end -> before teardown)")
