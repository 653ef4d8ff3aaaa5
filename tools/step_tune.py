"""Schedule-aware plan tuning (development tool, GPU box).

tools/autotune.py measures every layer alone, with the whole GPU to itself.
In bench.py's dataflow step the branches of an inception module (and a
bottleneck's projection shortcut) run concurrently, so a layer that needed
split-C to fill 148 SMs alone may do better with fewer splits (less partial
traffic, no stage-2 pass) or another tile.  This tool does coordinate descent
over the per-layer fused plans, timing the WHOLE captured step
(bench.time_graph) for each candidate, and writes the winners in the
tuned-plan format (merged into paper_2103_16234_b200/tuned_plans.json).

    python tools/step_tune.py --workload c2 --batch 32 --out gpurun_out/st/c2.json
"""
import argparse
import json
import os
import sys
import time
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
from paper_2103_16234_b200 import ConvLayer, family_names, matching_families
from paper_2103_16234_b200 import _native as nat
from paper_2103_16234_b200 import workloads as W

SPLITS = (1, 2, 3, 4, 6, 8, 12, 16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--sweeps", type=int, default=2)
    ap.add_argument("--budget-s", type=float, default=1500)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    t0 = time.time()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    lib = nat.lib()
    names = family_names()
    cfgs = W.layers(a.workload, a.batch)
    groups = W.schedule(a.workload, cfgs)
    xs, ws, ys = bench.make_operands(cfgs, dev, 0)
    targs = SimpleNamespace(steps=a.steps, warmup=3)
    # the tuned-plan registry is keyed by shape, so layers with identical shapes
    # (e.g. GoogLeNet 3b-1x1 and 3b-3x3red) must share one plan
    twins = {i: [j for j, d in enumerate(cfgs) if d.as_tuple() == c.as_tuple()] for i, c in enumerate(cfgs)}
    plans = []
    for cfg in cfgs:
        L = ConvLayer(cfg)
        plans.append((L._tiles.family, L.splits, L.reduce))

    def measure(pl, reps=2):
        layers = [ConvLayer(c, family=f, splits=s, reduce=r) for c, (f, s, r) in zip(cfgs, pl)]
        best = float("inf")
        for _ in range(reps):
            ms, _, _ = bench.time_graph(lib, layers, xs, ws, ys, targs, 1, dev, 0, groups)
            best = min(best, ms / a.steps)
        return best

    base0 = measure(plans, 3)
    cur = base0
    print(json.dumps({"start_ms": round(base0, 4)}), flush=True)
    for sweep in range(a.sweeps):
        changed = 0
        for i, cfg in enumerate(cfgs):
            if time.time() - t0 > a.budget_s:
                break
            f0, s0, r0 = plans[i]
            cands = {(f0, s) for s in SPLITS}
            for f in matching_families(cfg):
                for s in {s0, max(1, s0 // 2), s0 * 2}:
                    cands.add((f, s))
            cands = {(f, s, r) for f, s in cands for r in ((0,) if s == 1 else (1, 2) if s <= 16 else (1,))}
            best = (cur, plans[i])
            for f, s, r in sorted(cands):
                if (f, s, r) == plans[i]:
                    continue
                try:
                    L = ConvLayer(cfg, family=f, splits=s, reduce=r)
                except Exception:  # noqa: BLE001
                    continue
                if L.splits != s:
                    continue
                trial = list(plans)
                for j in twins[i]:
                    trial[j] = (f, s, L.reduce)
                t = measure(trial)
                if t < best[0] * 0.996:
                    best = (t, (f, s, L.reduce))
            if best[1] != plans[i]:
                trial = list(plans)
                for j in twins[i]:
                    trial[j] = best[1]
                # confirm against a fresh measurement of the incumbent
                t_new, t_old = measure(trial, 3), measure(plans, 3)
                if t_new < t_old * 0.997:
                    plans = trial
                    cur = t_new
                    changed += 1
                    print(json.dumps({"sweep": sweep, "layer": cfg.name, "from": [names[f0], s0, r0],
                                      "to": [names[best[1][0]], best[1][1], best[1][2]], "step_ms": round(t_new, 4),
                                      "was_ms": round(t_old, 4)}), flush=True)
                else:
                    cur = t_old
        print(json.dumps({"sweep": sweep, "changed": changed, "step_ms": round(cur, 4)}), flush=True)
        if not changed:
            break
    final = measure(plans, 3)
    out = []
    for cfg, (f, s, r) in zip(cfgs, plans):
        out.append({"layer": f"{a.workload}/{cfg.name}/N{a.batch}", "desc": list(cfg.as_tuple()), "engine": "fused",
                    "family": names[f], "splits": s, "reduce": r, "us": None, "model_us": None, "step_ms": round(final, 4),
                    "source": "tools/step_tune.py (dataflow step)"})
    with open(a.out, "w") as fh:
        json.dump({"generator": "tools/step_tune.py", "device": torch.cuda.get_device_name(), "start_ms": base0,
                   "final_ms": final, "plans": out}, fh, indent=0)
    print(json.dumps({"start_ms": round(base0, 4), "final_ms": round(final, 4)}), flush=True)


if __name__ == "__main__":
    main()
