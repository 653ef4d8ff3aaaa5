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


def tc_accurate(cfg, L):
    """3xTF32 accuracy rule: <= 72 k-blocks of 16 channels per
    TMEM accumulator (halo mode keeps whole channel blocks, so at least one)."""
    t = L._tc
    cb = -(-cfg.c // 16)
    taps = cfg.hf * cfg.wf
    if t.mode == 2:
        return -(-cb // t.splits) * taps <= max(72, taps)
    return -(-(cb * taps) // t.splits) <= 72


def tune_tc(cfg, eng, x, w, label, desc):
    auto = ConvLayer(cfg, eng)
    y = torch.empty(auto.output_shape(), device="cuda")
    t_auto = time_layer(auto, x, w, y)
    best = (t_auto, auto._tc.mode, 0, 0, auto.family, 0)
    seen = {(auto.family, auto._tc.m_halves)}
    for mode, mh in ((1, 0), (2, 1), (2, 2), (2, 4)):
        for nf in (0, 32, 64, 96, 128, 192, 256):
            for sp in (0, 1, 2, 3, 4, 6, 8, 12):
                try:
                    L = ConvLayer(cfg, eng, tc_mode=mode, filters_per_tile=nf, splits=sp, tc_m_halves=mh)
                except Exception:  # noqa: BLE001
                    continue
                key = (L.family, L._tc.m_halves)
                if key in seen or (eng == "tf32x3" and not tc_accurate(cfg, L)):
                    continue
                seen.add(key)
                t = time_layer(L, x, w, y)
                if t < best[0]:
                    best = (t, L._tc.mode, L._tc.filters_per_tile, L._tc.splits, L.family, L._tc.m_halves)
    del y
    if best[2] == 0:
        return {"layer": label, "desc": desc, "engine": eng, "mode": best[1], "nf": 0, "splits": 0,
                "plan": best[4], "us": round(best[0], 2), "model_us": round(t_auto, 2)}
    return {"layer": label, "desc": desc, "engine": eng, "mode": best[1], "nf": best[2], "splits": best[3],
            "mh": best[5] if best[1] == 2 else 0, "plan": best[4], "us": round(best[0], 2),
            "model_us": round(t_auto, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="c1,c2,c3,c4,c5")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                   "paper_2103_16234_b200", "tuned_plans.json"))
    ap.add_argument("--budget-s", type=float, default=1500)
    ap.add_argument("--engines", default="fused", help="comma list of fused, tf32x3, tf32")
    ap.add_argument("--batches", default="", help="override the batch sizes per workload (comma list)")
    ap.add_argument("--all-records", action="store_true",
                    help="write every tuned layer (keep=false where the cost model's plan won) for tools/merge_plans.py")
    ap.add_argument("--layers", default="", help="only these layer names (comma list)")
    ap.add_argument("--families", default="", help="only fused families whose name contains one of these (comma list)")
    ap.add_argument("--splits", default="1,2,3,4,6,8,12,16,24", help="fused split counts to try")
    args = ap.parse_args()
    engines = args.engines.split(",")
    names = family_names()
    plans, seen = [], set()
    t_start = time.time()
    for wl in args.workloads.split(","):
        batches = [int(b) for b in args.batches.split(",")] if args.batches else W.WORKLOADS[wl][1]
        for n in batches:
            for cfg in W.layers(wl, n):
                key = cfg.as_tuple()
                if key in seen or (args.layers and cfg.name not in args.layers.split(",")):
                    continue
                seen.add(key)
                if args.families and "fused" in engines and not any(
                        any(k in names[f] for k in args.families.split(",")) for f in matching_families(cfg)):
                    continue  # no candidate family for this shape
                if time.time() - t_start > args.budget_s:
                    break
                x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda")
                w = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda")
                for eng in engines:
                    if eng != "fused":
                        rec = tune_tc(cfg, eng, x, w, f"{wl}/{cfg.name}/N{n}", list(key))
                        if rec:
                            print(json.dumps(rec), flush=True)
                            if rec["us"] < rec["model_us"] * 0.97:
                                plans.append(rec)
                if "fused" not in engines:
                    continue
                auto = ConvLayer(cfg)
                y = torch.empty(auto.output_shape(), device="cuda")
                t_auto = time_layer(auto, x, w, y)
                best = (t_auto, names[auto._tiles.family], auto.splits, auto.reduce)
                for f in matching_families(cfg):
                    if args.families and not any(k in names[f] for k in args.families.split(",")):
                        continue
                    for sp in (int(v) for v in args.splits.split(",")):
                        for red in ((0,) if sp == 1 else (1, 2) if sp <= 16 else (1,)):
                            try:
                                L = ConvLayer(cfg, family=f, splits=sp, reduce=red)
                            except Exception:
                                continue
                            if L.splits != sp:
                                continue
                            t = time_layer(L, x, w, y)
                            if t < best[0]:
                                best = (t, names[f], L.splits, L.reduce)
                rec = {"layer": f"{wl}/{cfg.name}/N{n}", "desc": list(key), "engine": "fused",
                       "family": best[1], "splits": best[2], "reduce": best[3], "us": round(best[0], 2),
                       "model_us": round(t_auto, 2)}
                rec["keep"] = best[0] < t_auto * 0.97
                print(json.dumps(rec), flush=True)
                if rec["keep"] or args.all_records:
                    plans.append(rec)
                del x, w, y
                torch.cuda.empty_cache()
    with open(args.out, "w") as fh:
        json.dump({"generator": "tools/autotune.py", "device": torch.cuda.get_device_name(),
                   "plans": plans}, fh, indent=0)
    print(f"wrote {len(plans)} tuned plans to {args.out}")


if __name__ == "__main__":
    main()
