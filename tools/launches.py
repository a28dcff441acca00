"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per cct kernel."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if not any(s in d["Kernel Name"] for s in ("cct", "unnamed>", "gk::", "_kernel")) and "--all" not in sys.argv:
            continue
        key = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void ", "").replace("cct::<unnamed>::", "").replace("gk::", ""))
        agg.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = 0.0
for (i, k), v in sorted(agg.items()):
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    by = (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e6
    tot += t
    print(f"{i:>4} {k[:44]:44s} {t:9.1f} us {by:9.1f} MB {by / t if t else 0:6.2f} TB/s")
print(f"total {tot:.1f} us")
