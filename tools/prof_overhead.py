"""Step time of the bench workload with and without the per-launch phase events (A/B)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200.stack import CAFFENET, ConvStack  # noqa: E402

dev = torch.device("cuda")
st = ConvStack(256, dev, CAFFENET)
L = cct.lib()
for _ in range(3):
    st.step()
torch.cuda.synchronize()
for prof in (0, 1, 0, 1):
    L.cct_profile_read(None, None, None, None, 1)
    L.cct_profile_enable(prof)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    L.cct_profile_enable(0)
    print(f"profiling {prof}: {e0.elapsed_time(e1) / 20:.3f} ms/step", flush=True)
