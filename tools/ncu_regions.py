"""Stall reasons by code region of a --set full capture (run here on the CPU host):
    python tools/ncu_regions.py REPORT.ncu-rep
Regions = runs of consecutive SASS lines with the same execution count; the
hottest FFMA2 run is the inner loop.  Prints instructions and the per-reason
warp-stall samples of every region holding > 2 % of the samples."""
import csv
import io
import subprocess
import sys

REASONS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_lg", "stall_long_sb", "stall_math",
           "stall_mio", "stall_no_inst", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_wait",
           "stall_drain", "stall_membar", "stall_misc", "stall_sleep"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[0][1])
    hdr, data = rows[1], rows[2:]
    ia, ss, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    ri = {r: hdr.index(r) for r in REASONS if r in hdr}

    def num(v):
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return 0.0

    regions, cur = [], None
    for i, r in enumerate(data):
        c = num(r[ia])
        if cur is None or c != cur["count"]:
            cur = {"start": i, "count": c, "inst": 0.0, "samples": 0.0, "ffma2": 0, "first": r[src].strip()[:48],
                   "reasons": {k: 0.0 for k in ri}}
            regions.append(cur)
        cur["end"] = i
        cur["inst"] += c
        cur["samples"] += num(r[ss])
        cur["ffma2"] += "FFMA2" in r[src]
        for k, j in ri.items():
            cur["reasons"][k] += num(r[j])
    tot_s = sum(g["samples"] for g in regions) or 1
    tot_i = sum(g["inst"] for g in regions) or 1
    print(f"instructions {tot_i:.4g}, stall samples {tot_s:.0f}")
    for g in regions:
        if g["samples"] / tot_s < 0.02:
            continue
        top = sorted(g["reasons"].items(), key=lambda kv: -kv[1])[:5]
        print(f"lines {g['start']:5d}-{g['end']:5d} x{g['count']:.0f}  inst {100*g['inst']/tot_i:5.1f}%  "
              f"samples {100*g['samples']/tot_s:5.1f}%  ffma2 {g['ffma2']:3d}  [{g['first']}]  "
              + ", ".join(f"{k[6:]} {100*v/tot_s:.1f}" for k, v in top if v))


if __name__ == "__main__":
    main(sys.argv[1])
