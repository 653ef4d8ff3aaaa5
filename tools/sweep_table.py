"""Summarise a bench.py --report sweep JSON into a markdown table (per workload x batch)."""
import json, sys
from collections import defaultdict
d = json.load(open(sys.argv[1]))
peak = d["peak_fp32_tflops"]
agg = defaultdict(lambda: defaultdict(float))
for r in d["rows"]:
    k = (r["workload"], r["batch"])
    fl = r["gflops"] * r["us"] * 1e-6  # GFLOP
    agg[k]["gflop"] += fl
    agg[k]["fused_us"] += r["us"]
    agg[k]["tc_us"] += r.get("tf32x3_us", 0)
    agg[k]["cudnn_us"] += r.get("cudnn_fp32_us", 0)
    agg[k]["layers"] += 1
print(f"| workload | batch | layers | fused µs | fused TFLOP/s | % FFMA2 peak | tf32x3 µs | tf32x3 TFLOP/s | cuDNN fp32 µs | fused vs cuDNN | tf32x3 vs cuDNN |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for (wl, n), a in sorted(agg.items()):
    f = a["gflop"] / a["fused_us"] * 1e3
    t = a["gflop"] / a["tc_us"] * 1e3 if a["tc_us"] else 0
    cu = a["cudnn_us"]
    print(f"| {wl} | {n} | {int(a['layers'])} | {a['fused_us']:.0f} | {f:.1f} | {100 * f / peak:.0f}% | {a['tc_us']:.0f} | {t:.1f} | "
          f"{cu:.0f} | {cu / a['fused_us']:.2f}x | {cu / a['tc_us']:.2f}x |")
