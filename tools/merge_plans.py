"""Merge autotune.py --all-records output into paper_2103_16234_b200/tuned_plans.json.

    python tools/merge_plans.py NEW.json [NEW2.json ...]

For every (shape, engine) a new file tuned: its record replaces the old one
(or is added) when keep is true — the measured winner beat the plan the
library resolved at tuning time (the registry's record, else the cost model's
pick) by >3 %.  keep=false means that resolved plan is still the measured
best, so the existing record (if any) stays."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH = os.path.join(ROOT, "paper_2103_16234_b200", "tuned_plans.json")


def main(paths):
    cur = json.load(open(PATH))
    plans = cur["plans"]
    key = lambda r: (tuple(r["desc"]), r["engine"])  # noqa: E731
    idx = {key(r): i for i, r in enumerate(plans)}
    added, replaced = 0, 0
    for p in paths:
        for r in json.load(open(p))["plans"]:
            k = key(r)
            keep = r.pop("keep", True)
            if not keep:
                continue
            if k in idx:
                plans[idx[k]] = r
                replaced += 1
            else:
                idx[k] = len(plans)
                plans.append(r)
                added += 1
    cur["plans"] = plans
    with open(PATH, "w") as fh:
        json.dump(cur, fh, indent=0)
    print(f"replaced {replaced}, added {added}; {len(cur['plans'])} plans")


if __name__ == "__main__":
    main(sys.argv[1:])
