"""Run fwd / bwd-data / bwd-weight once per selected layer (for ncu launch lists).

python tools/phase_profile.py --layer conv2 --type 1 [--passes fwd,dgrad,wgrad] [--warm 1]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402

LAYERS = {  # CaffeNet conv1-5 (n, k, d, o, stride, pad)
    "conv1": (227, 11, 3, 96, 4, 0),
    "conv2": (27, 5, 96, 256, 1, 2),
    "conv3": (13, 3, 256, 384, 1, 1),
    "conv4": (13, 3, 384, 384, 1, 1),
    "conv5": (13, 3, 384, 256, 1, 1),
}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="conv2")
    ap.add_argument("--type", type=int, default=1)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--passes", default="fwd,dgrad,wgrad")
    ap.add_argument("--warm", type=int, default=1)
    a = ap.parse_args()
    n, k, d, o, s, p = LAYERS[a.layer]
    desc = cct.ConvDesc(n, k, d, o, a.batch, s, p)
    m = desc.m
    dev = torch.device("cuda")
    x = torch.rand((a.batch, n, n, d), device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), device=dev) * 2 - 1
    dy = torch.rand((a.batch, o, m, m), device=dev) * 2 - 1
    fns = {"fwd": lambda: conv.conv_fwd(x, w, desc, a.type),
           "dgrad": lambda: conv.conv_bwd_data(dy, w, desc, a.type),
           "wgrad": lambda: conv.conv_bwd_weight(x, dy, desc, a.type)}
    for _ in range(a.warm + 1):
        for ps in a.passes.split(","):
            fns[ps]()
    torch.cuda.synchronize()
    print("done", a.layer, a.type, flush=True)
