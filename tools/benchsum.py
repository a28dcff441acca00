"""Print a one-line summary of the bench.py JSON line read from stdin (tag = argv[1])."""
import json
import sys

lines = [l for l in sys.stdin.read().strip().splitlines() if l.startswith("{")]
l = json.loads(lines[-1])
ph = l.get("phases", {})
print(sys.argv[1] if len(sys.argv) > 1 else "", round(l["value"]), "img/s", round(l["ms_per_step"], 3), "ms",
      " ".join(f"{k}={v['ms_per_step']:.3f}" for k, v in ph.items()), "clk", l.get("clocks", {}).get("sm_mhz"))
