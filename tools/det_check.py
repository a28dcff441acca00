"""Diagnostic: repeatability of conv1 backward-weight (b=32)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402

b = 32
desc = cct.ConvDesc(227, 11, 3, 96, b, 4, 0)
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(17)
x = torch.rand((b, 227, 227, 3), generator=g, device=dev) * 2 - 1
dy = torch.rand((b, 96, desc.m, desc.m), generator=g, device=dev) * 2 - 1
w = torch.rand((96, 11, 11, 3), generator=g, device=dev) * 2 - 1
ref = conv.conv_bwd_weight(x, dy, desc, 1)
for i in range(6):
    if i % 2:
        big = torch.empty(3 << 28, device=dev)  # flush L2 / shift allocations
        big.fill_(1.0)
        del big
    dw = conv.conv_bwd_weight(x, dy, desc, 1)
    print(i, "equal" if torch.equal(dw, ref) else f"DIFF {float((dw - ref).norm() / ref.norm()):.3e}", flush=True)
