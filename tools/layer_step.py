"""One training step (fwd cached + combined bwd) of one conv layer, for ncu launch lists.

python tools/layer_step.py n k d o stride pad type [batch]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402

n, k, d, o, s, p, t = (int(v) for v in sys.argv[1:8])
b = int(sys.argv[8]) if len(sys.argv) > 8 else 256
desc = cct.ConvDesc(n, k, d, o, b, s, p)
dev = torch.device("cuda")
x = torch.rand((b, n, n, d), device=dev) * 2 - 1
w = torch.rand((o, k, k, d), device=dev) * 2 - 1
dy = torch.rand((b, o, desc.m, desc.m), device=dev) * 2 - 1
cache = conv.alloc_cache(desc, t, dev)
y = conv.conv_fwd_cached(x, w, desc, t, cache=cache)
dx, dw = conv.conv_bwd(dy, w, desc, t, x=x, cache=cache)
torch.cuda.synchronize()
print("done")
