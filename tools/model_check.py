"""Compare the cost model (libcct.so, no GPU needed) with a measured sweep (tools/sweep.py output)."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402

hits = tot = 0
err = []
for line in open(sys.argv[1]):
    r = json.loads(line)
    desc = cct.ConvDesc(r["n"], r["k"], r["d"], r["o"], r["b"], r["stride"], r["pad"])
    choice, est = cct.select_lowering(desc, 3)
    meas = {int(t): v["ms"] for t, v in r["types"].items()}
    best = min(meas, key=meas.get)
    regret = meas[choice] / meas[best]
    tot += 1
    hits += choice == best
    for t in (1, 2, 3):
        err.append(est[t - 1].model_seconds * 1e3 / meas[t])
    print(f"n={r['n']:3d} d={r['d']:5d} o={r['o']:5d} d/o={r['d']/r['o']:7.3f} measured "
          + " ".join(f"T{t}={meas[t]:7.3f}" for t in (1, 2, 3)) + " | model "
          + " ".join(f"T{t}={est[t-1].model_seconds*1e3:7.3f}" for t in (1, 2, 3))
          + f" | best T{best} model T{choice} regret {regret:.3f}")
err.sort()
print(f"choice == measured best on {hits}/{tot}; model/measured median {err[len(err)//2]:.2f} "
      f"[{err[0]:.2f}, {err[-1]:.2f}]")
