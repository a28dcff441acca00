"""Step time of the bench workload eager vs replayed from a CUDA graph (A/B, no phase events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200.stack import CAFFENET, ConvStack  # noqa: E402

dev = torch.device("cuda")
st = ConvStack(256, dev, CAFFENET)
L = cct.lib()
L.cct_profile_enable(0)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(3):
        st.step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    st.step()
torch.cuda.synchronize()
print("captured", flush=True)


def timed(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for _ in range(2):
    print(f"eager {timed(st.step):.3f} ms/step  graph {timed(g.replay):.3f} ms/step", flush=True)
