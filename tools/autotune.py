"""Measure every (kernel family x reduction split) for the BASELINE layers on
the GPU and write paper_2103_16234_b200/tuned_plans.json ("find" results the
planner uses for exact shape matches; other shapes use its cost model).

    python tools/autotune.py [--workloads c2,c3,...] [--out PATH]

Timing: each candidate is captured as a CUDA graph of 20 launches and replayed
twice; the median of 3 replays (CUDA events) is kept.  The winner must beat
the cost model's own choice by >3% to be recorded.
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2103_16234_b200 import ConvLayer, family_names, matching_families
from paper_2103_16234_b200 import workloads as W


def time_layer(L, x, w, y, reps=20):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        L(x, w, out=y)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                L(x, w, out=y)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b) / reps * 1e3)
    return sorted(ts)[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="c1,c2,c3,c4,c5")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                   "paper_2103_16234_b200", "tuned_plans.json"))
    ap.add_argument("--budget-s", type=float, default=1500)
    args = ap.parse_args()
    names = family_names()
    plans, seen = [], set()
    t_start = time.time()
    for wl in args.workloads.split(","):
        for n in W.WORKLOADS[wl][1]:
            for cfg in W.layers(wl, n):
                key = cfg.as_tuple()
                if key in seen:
                    continue
                seen.add(key)
                if time.time() - t_start > args.budget_s:
                    break
                x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda")
                w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
                auto = ConvLayer(cfg)
                y = torch.empty(auto.output_shape(), device="cuda")
                t_auto = time_layer(auto, x, w, y)
                best = (t_auto, auto.family, auto.splits)
                for f in matching_families(cfg):
                    for sp in (1, 2, 3, 4, 6, 8, 12, 16, 24):
                        try:
                            L = ConvLayer(cfg, family=f, splits=sp)
                        except Exception:
                            continue
                        if L.splits != sp:
                            continue
                        t = time_layer(L, x, w, y)
                        if t < best[0]:
                            best = (t, names[f], L.splits)
                rec = {"layer": f"{wl}/{cfg.name}/N{n}", "desc": list(key), "engine": "fused",
                       "family": best[1], "splits": best[2], "us": round(best[0], 2), "model_us": round(t_auto, 2)}
                print(json.dumps(rec), flush=True)
                if best[0] < t_auto * 0.97:
                    plans.append(rec)
                del x, w, y
                torch.cuda.empty_cache()
    with open(args.out, "w") as fh:
        json.dump({"generator": "tools/autotune.py", "device": torch.cuda.get_device_name(),
                   "plans": plans}, fh, indent=0)
    print(f"wrote {len(plans)} tuned plans to {args.out}")


if __name__ == "__main__":
    main()
