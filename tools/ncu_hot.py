"""Top SASS instructions by warp-stall samples from an ncu report: python tools/ncu_hot.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr_i]
si, ai, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
tot = sum(int(r[ai] or 0) for r in body)
print(f"total samples {tot}")
for idx, r in sorted(enumerate(body), key=lambda t: -int(t[1][ai] or 0))[:n]:
    print(f"{idx:5d} {int(r[ai]):6d} {100*int(r[ai])/tot:5.1f}%  exec={r[ei]:>8s}  {r[si].strip()[:90]}")
