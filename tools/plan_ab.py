"""A/B of whole-step plan sets (tools/step_tune.py outputs) in one process:
    python tools/plan_ab.py c2 32 A.json B.json [...]"""
import json, os, sys
from types import SimpleNamespace
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2103_16234_b200 import ConvLayer, family_names
from paper_2103_16234_b200 import _native as nat
from paper_2103_16234_b200 import workloads as W

wl, n, files = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
names = family_names()
cfgs = W.layers(wl, n)
groups = W.schedule(wl, cfgs)
xs, ws, ys = bench.make_operands(cfgs, dev, 0)
sets = {}
for f in files:
    by = {tuple(p["desc"]): p for p in json.load(open(f))["plans"]}
    sets[f] = [ConvLayer(c, family=names.index(by[c.as_tuple()]["family"]), splits=by[c.as_tuple()]["splits"],
                         reduce=by[c.as_tuple()].get("reduce", 0)) for c in cfgs]
sets["auto"] = [ConvLayer(c) for c in cfgs]
res = {k: [] for k in sets}
args = SimpleNamespace(steps=100, warmup=3)
for rep in range(5):
    for k, layers in sets.items():
        ms, _, _ = bench.time_graph(nat.lib(), layers, xs, ws, ys, args, 1, dev, 0, groups)
        res[k].append(ms / args.steps)
for k, v in res.items():
    print(json.dumps({"set": k, "min_ms": round(min(v), 4), "median_ms": round(sorted(v)[len(v) // 2], 4)}))
