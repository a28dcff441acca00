"""Summarise tools/gpu_ab.sh output: ms/step per arm (median of rounds) and phase split."""
import glob
import json
import os
import statistics
import sys

d = sys.argv[1]
arms = {}
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    arm = os.path.basename(f).rsplit("_", 1)[0]
    try:
        rec = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print("bad", f)
        continue
    arms.setdefault(arm, []).append(rec)
for arm, recs in arms.items():
    ms = [r["ms_per_step"] for r in recs]
    ph = {k: round(statistics.median(r["phases"][k]["ms_per_step"] for r in recs), 3) for k in recs[0].get("phases", {})}
    print(f"{arm:28s} ms/step {statistics.median(ms):.3f}  all {[round(x, 3) for x in ms]}  {ph}")
