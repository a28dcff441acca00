"""Side-by-side raw metrics of the first kernel in two ncu reports (differences only)."""
import csv
import io
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2]))


a, b = load(sys.argv[1]), load(sys.argv[2])
pat = sys.argv[3].split(",") if len(sys.argv) > 3 else ["inst_executed.sum", "dram__bytes", "duration",
                                                         "op_st.sum", "stalled", "tensor_cycles_active.avg.pct"]
for k in a:
    if any(t in k for t in pat) and a.get(k) != b.get(k):
        print(f"{k[:96]:96s} {a.get(k, '')[:16]:>16s} {b.get(k, '')[:16]:>16s}")
print("A:", a.get("Kernel Name", "")[:110])
print("B:", b.get("Kernel Name", "")[:110])
