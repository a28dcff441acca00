"""Diagnostic: conv1 backward-weight (b=32) vs fp64 torch under env variants."""
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n, k, d, o, s, p = 227, 11, 3, 96, 4, 0
desc = cct.ConvDesc(n, k, d, o, b, s, p)
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(17)
x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
xd = x.double().permute(0, 3, 1, 2).contiguous()
rdw = torch.nn.grad.conv2d_weight(xd, (o, d, k, k), dy.double(), stride=s, padding=p).permute(0, 2, 3, 1)
def cached():
    cache = conv.alloc_cache(desc, 1, dev)
    conv.conv_fwd_cached(x, w, desc, 1, cache=cache)
    return conv.conv_bwd(dy, w, desc, 1, x=x, cache=cache)[1]


for name, fn in (("wgrad", lambda: conv.conv_bwd_weight(x, dy, desc, 1)),
                 ("train", lambda: conv.conv_bwd(dy, w, desc, 1, x=x, cache=None)[1]), ("cached", cached)):
    dw = fn()
    print(name, os.environ.get("TAG", ""), float(torch.linalg.norm(dw.double() - rdw) / torch.linalg.norm(rdw)), flush=True)

dwc = cached()
dwt = conv.conv_bwd(dy, w, desc, 1, x=x, cache=None)[1]
diff = (dwc - dwt).abs().reshape(o, -1)
bad_rows = (diff.amax(1) > 1e-3 * dwt.abs().max()).nonzero().ravel().tolist()
bad_cols = (diff.amax(0) > 1e-3 * dwt.abs().max()).nonzero().ravel().tolist()
print("bad rows (o)", bad_rows[:10], len(bad_rows), "bad cols (tap*d+ch)", bad_cols[:10], bad_cols[-5:], len(bad_cols))

# dw only, with the cache (no dx part)
cache = conv.alloc_cache(desc, 1, dev)
conv.conv_fwd_cached(x, w, desc, 1, cache=cache)
_, dwo = conv.conv_bwd(dy, w, desc, 1, x=x, cache=cache, want_dx=False)
print("cached dw-only", float(torch.linalg.norm(dwo.double() - rdw) / torch.linalg.norm(rdw)))
dhat = conv.lower(x, desc, 1, cct.ROWS_INTERNAL)
rows, cols = dhat.shape[0], dhat.shape[1]
cv = cache.view(rows, -1)[:, :cols]
print("cache == lower:", bool(torch.equal(cv, dhat)), cache.numel(), rows * ((cols + 3) // 4 * 4))
