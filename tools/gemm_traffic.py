"""profiles/rNN/gemm_traffic.json from an ncu launch list of `bench.py --steps 1 --warmup 1`:
average DRAM bytes (read + write) per tensor-core GEMM launch (gemm3xtf32 and the fused conv1
gather / hfold kernels: the GEMM phase of the step) over the last (timed) step."""
import csv
import json
import sys

path, out, per_step = sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 15
rows = list(csv.reader(open(path)))
hdr = None
agg = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if any(t in d["Kernel Name"] for t in ("gemm3xtf32", "gather_kernel", "hfold_kernel")):
            agg.setdefault(int(d["ID"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
last = [agg[i] for i in sorted(agg)][-per_step:]
by = [v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in last]
ns = [v.get("gpu__time_duration.sum", 0) for v in last]
json.dump({"kernel": f"gemm3xtf32_kernel + fused conv1 gather / hfold kernels (the {len(last)} launches of one "
                     f"conv1-5 fwd+bwd step, b=256)",
           "launches": len(last), "avg_dram_bytes_per_launch": sum(by) / len(by),
           "avg_duration_ns_under_ncu": sum(ns) / len(ns),
           "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     f"--clock-control none python bench.py --steps 1 --warmup 1 ({path}; last {len(last)} GEMM launches)"},
          open(out, "w"), indent=1)
print(open(out).read())
