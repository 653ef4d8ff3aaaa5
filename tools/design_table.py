"""DESIGN.md §7 table from a final_round.sh output directory.

    python tools/design_table.py gpurun_out/r1final
"""
import json
import os
import sys

ROWS = [("bench.json", "C2 GoogLeNet 1×1 ×36, N=32/GPU (headline)"), ("bench_c1.json", "C1 ResNet conv2_x 3×3, N=1"),
        ("bench_c3.json", "C3 AlexNet conv2 + inception 5×5, N=128"), ("bench_c4.json", "C4 VGG-16 3×3 ×13, N=8"),
        ("bench_c5.json", "C5 ResNet-50 ×53, N=256")]


def last_json(path):
    with open(path) as fh:
        lines = [l for l in fh if l.startswith("{")]
    return json.loads(lines[-1])


def main(d):
    print("| workload (bench.py --workload) | fused FFMA2 engine (TFLOP/s) | dominant kernel: achieved / frac of "
          "FFMA2 peak / DRAM traffic vs algorithmic bytes per launch | tf32x3 variant | e2e (host buffers) |")
    print("|---|---|---|---|---|")
    for f, label in ROWS:
        p = os.path.join(d, f)
        if not os.path.exists(p):
            continue
        b = last_json(p)
        r = b["roofline"]
        tc = b.get("tensor_core_variant") or {}
        e2e = (b.get("e2e") or {}).get("value")
        traffic = (f"{r['traffic'] / 1e6:.1f} / {r['algorithmic_bytes_per_launch'] / 1e6:.1f} MB"
                   if r.get("traffic") else "n/a")
        print(f"| {label} | {b['value'] / 1e3:.1f} | `{r['kernel']}` ({r['kernel_share_of_step']:.0%} of kernel time): "
              f"{r['achieved']:.1f} TFLOP/s, {r['frac']:.0%}, {traffic} | "
              f"{tc.get('value', 0) / 1e3:.1f} | {e2e / 1e3 if e2e else 0:.2f} |")


if __name__ == "__main__":
    main(sys.argv[1])
