"""Summarise B2C_TRACE_FILE per-CTA phase records."""
import csv, sys, collections
for f in sys.argv[1:]:
    rows = [(int(r[1]), int(r[2]), *[int(v) for v in r[3:7]]) for r in csv.reader(open(f))]
    t0 = min(r[2] for r in rows)
    tend = max(r[5] for r in rows)
    ph = lambda a, b: sorted((r[b] - r[a]) / 1e3 for r in rows)
    med = lambda v: v[len(v) // 2]
    tab, loop, epi = ph(2, 3), ph(3, 4), ph(4, 5)
    starts = sorted((r[2] - t0) / 1e3 for r in rows)
    print(f"{f}: ctas={len(rows)} span={ (tend - t0) / 1e3:.1f}us  start(last)={starts[-1]:.1f}  "
          f"tables med/max={med(tab):.2f}/{tab[-1]:.2f}  loop med/max={med(loop):.2f}/{loop[-1]:.2f}  "
          f"epilogue med/max={med(epi):.2f}/{epi[-1]:.2f}  sms={len(set(r[1] for r in rows))}")
