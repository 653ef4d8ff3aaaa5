import json, sys
d = sys.argv[1]
for f in ["check.log", "roles.log", "time.log"]:
    try:
        lines = open(f"{d}/{f}").read().splitlines()
    except OSError:
        continue
    for l in lines:
        if not l.startswith("{"):
            print(l[:200]); continue
        r = json.loads(l)
        if "case" in r:
            print(f"{r['case']:14s} x3={r.get('tf32x3')!s:24.24s} x1={r.get('tf32')!s:24.24s}")
        else:
            print(f"{r['layer']:16s} {r['n']:4d} fused {r.get('fused_tf')!s:6} x3 {r.get('tf32x3_tf')!s:6} x1 {r.get('tf32_tf')!s:6} {r.get('tf32x3_plan')}")
