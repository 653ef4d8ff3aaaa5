"""Summarise ncu output for profiles/ (run here, on the CPU host).

    python tools/ncu_summary.py launches LAUNCHES.csv            # per-kernel share of device time
    python tools/ncu_summary.py full REPORT.ncu-rep              # key metrics of a --set full capture
"""
from __future__ import annotations

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEY_METRICS = [
    r"gpu__time_duration\.sum$", r"dram__bytes_(read|write)\.sum$", r"sm__cycles_elapsed\.avg\.per_second$",
    r"sm__pipe_fma_cycles_active\.avg\.pct_of_peak_sustained_active$",
    r"sm__inst_executed_pipe_fma\.avg\.pct_of_peak_sustained_active$",
    r"sm__pipe_tensor.*cycles_active\.avg\.pct_of_peak_sustained_(active|elapsed)$",
    r"sm__throughput\.avg\.pct_of_peak_sustained_elapsed$", r"launch__registers_per_thread$",
    r"launch__grid_size$", r"launch__block_size$", r"sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"lts__t_bytes\.sum$", r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum$",
    r"smsp__inst_executed\.sum$", r"launch__shared_mem_per_block_dynamic$",
    r"smsp__average_warp_latency_issue_stalled_.*\.ratio$",
]


def launches(path):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if not l.startswith("==")]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        if v != v:  # nan (ncu could not time the launch)
            continue
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        rows.append((name, v * scale))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for n, t in rows:
        tot[n] += t
        cnt[n] += 1
    total = sum(tot.values())
    print(f"# {len(rows)} launches, {total:.1f} us total device time (ncu: serialised, cold-cache)")
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for n in sorted(tot, key=lambda k: -tot[k]):
        print(f"{n[:60]:60s} {cnt[n]:8d} {tot[n]:10.1f} {tot[n] / cnt[n]:9.2f} {tot[n] / total:6.1%}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units, vals = r[0], r[1], r[2:]
    kcol = head.index("Kernel Name") if "Kernel Name" in head else None
    for v in vals:
        if kcol is not None:
            print(f"## {v[kcol][:120]}")
        for i, k in enumerate(head):
            if any(re.search(p, k) for p in KEY_METRICS):
                print(f"{k:80s} {v[i]:>16s} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
