"""Summarise bench lines: python tools/bline.py FILE.json [...]"""
import json, sys
from collections import defaultdict
for path in sys.argv[1:]:
    lines = [l for l in open(path) if l.startswith("{")]
    if not lines:
        print(path, "no line"); continue
    d = json.loads(lines[-1])
    r = d.get("roofline", {})
    print(f"== {path}: value {d['value']:.0f} {d['unit']} ms/step {d['ms_per_step']} | dom {r.get('kernel')} "
          f"{r.get('achieved')} frac {r.get('frac')} share {r.get('kernel_share_of_step')} | "
          f"step frac {r.get('step', {}).get('frac')} | clocks {d.get('clocks')}")
    fam = defaultdict(lambda: [0.0, 0.0, 0])
    for row in d.get("per_layer", []):
        f = fam[row["family"]]
        f[0] += row["us"]; f[1] += row["gflops"] * row["us"]; f[2] += 1
    for k, (us, gw, n) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
        print(f"   {k:28s} n={n:3d} {us/1e3:8.3f} ms  {gw/us/1e3:6.1f} TFLOP/s")
    tc = d.get("tensor_core_variant")
    if tc:
        print(f"   tc {tc['engine']}: {tc['value']:.0f} GFLOP/s, frac {tc['roofline']['frac']}")
