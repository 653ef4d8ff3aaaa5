"""Development: time tensor-core plans (forced mode / filters / splits) per layer.
    python tools/tc_plan_cmp.py ENGINE WL:N[:name,...] ..."""
import itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, InvalidPlan, workloads as W

eng = sys.argv[1]
for spec in sys.argv[2:]:
    parts = spec.split(":")
    wl, n = parts[0], int(parts[1])
    names = set(parts[2].split(",")) if len(parts) > 2 and parts[2] else None
    for cfg in W.layers(wl, n):
        if names and cfg.name not in names:
            continue
        x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda")
        w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
        res = {}
        auto = ConvLayer(cfg, eng)
        cands = [("auto", auto)]
        for mode, nf, sp in itertools.product((1, 2), (0, 64, 128, 256), (0, 1, 2, 4)):
            try:
                cands.append((f"m{mode}n{nf}k{sp}", ConvLayer(cfg, eng, tc_mode=mode, filters_per_tile=nf, splits=sp)))
            except (InvalidPlan, Exception):  # noqa: BLE001
                pass
        best = None
        for tag, L in cands:
            y = L(x, w)
            for _ in range(2):
                L(x, w, out=y)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                L(x, w, out=y)
            b.record()
            b.synchronize()
            us = a.elapsed_time(b) / 10 * 1e3
            res[tag] = (round(us, 1), L.family)
            if best is None or us < best[1]:
                best = (tag, us, L.family)
        print(json.dumps({"layer": cfg.name, "n": n, "auto": res["auto"], "best": [best[0], round(best[1], 1), best[2]],
                          "gflop": round(cfg.flops / 1e9, 3)}), flush=True)
