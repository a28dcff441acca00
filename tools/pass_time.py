"""CUDA-event time of one pass of one CaffeNet layer (after warm-up), for A/B runs.

python tools/pass_time.py --layer conv1 --pass fwd [--type 1] [--reps 10]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from phase_profile import LAYERS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layer", default="conv1")
ap.add_argument("--pass", dest="pass_", default="fwd")
ap.add_argument("--type", type=int, default=1)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tune", default="", help="comma list key=value of cct tuning switches")
ap.add_argument("--layout", type=int, default=0, help="0 NCHW y / dy, 1 NHWC")
a = ap.parse_args()
for kv in filter(None, a.tune.split(",")):
    k_, v_ = kv.split("=")
    cct.set_tuning(k_, int(v_))
n, k, d, o, s, p = LAYERS[a.layer]
desc = cct.ConvDesc(n, k, d, o, a.batch, s, p, a.layout)
dev = torch.device("cuda")
x = torch.rand((a.batch, n, n, d), device=dev) * 2 - 1
w = torch.rand((o, k, k, d), device=dev) * 2 - 1
dy = torch.rand(desc.y_shape(), device=dev) * 2 - 1
fn = {"fwd": lambda: conv.conv_fwd(x, w, desc, a.type), "dgrad": lambda: conv.conv_bwd_data(dy, w, desc, a.type),
      "wgrad": lambda: conv.conv_bwd_weight(x, dy, desc, a.type)}[a.pass_]
for _ in range(3):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

e0.record()
for _ in range(a.reps):
    fn()
e1.record()
torch.cuda.synchronize()
print(f"{a.layer} {a.pass_} T{a.type}: {e0.elapsed_time(e1) / a.reps * 1e3:.1f} us per pass", flush=True)
