"""GPU parity at BASELINE sizes for every lowering type.

* configs[1]: the lowering-type sweep (n = 13, k = 3, pad 1, b = 256) at all nine
  (d, o) points of SURVEY 8(a) a12 -- d/o = 1/16 .. 16 -- for Type 1, 2 and 3, the
  stand-alone passes and the cached training step (fwd + bwd-data + bwd-weight).
  Forward and backward-data are checked against the oracle on a two-image slice of
  the full-batch outputs (images are independent in those passes); backward-weight
  (a reduction over all 256 images) against fp64 torch on the GPU (checker only).
  The result must not depend on the lowering.
* configs[2] / [3]: CaffeNet conv1 at b = 256 through the bench's exact path (the
  cached training step, cost-model lowering).
Tolerance: relative L2 <= 1e-4 per tensor (north star).
"""
import pytest
import torch

from oracle_py import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-4
SWEEP = [(64, 1024), (128, 512), (256, 256), (512, 128), (1024, 64),
         (128, 1024), (256, 512), (512, 256), (1024, 128)]


def _data(dev, desc, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    b, n, d, o, k, m = desc.b, desc.n, desc.d, desc.o, desc.k, desc.m
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, m, m), generator=g, device=dev) * 2 - 1
    return x, w, dy


def _fp64_wgrad(x, w, dy, s, p):
    xd = x.double().permute(0, 3, 1, 2).contiguous()
    wd = w.double().permute(0, 3, 1, 2)
    return torch.nn.grad.conv2d_weight(xd, wd.shape, dy.double(), stride=s, padding=p).permute(0, 2, 3, 1)


def _rel(a, r):
    return float(torch.linalg.norm(a.double() - r) / torch.linalg.norm(r))


@pytest.mark.timeout(900, method="thread")
@pytest.mark.parametrize("d,o", SWEEP, ids=[f"d{d}_o{o}" for d, o in SWEEP])
def test_ratio_sweep_b256_every_type(cct, dev, orc, d, o):
    from paper_1504_04343_b200 import conv
    n, k, s, p, b = 13, 3, 1, 1, 256
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x, w, dy = _data(dev, desc, d * 7 + o)
    q = 2  # oracle slice
    xs, ws, dys = x[:q].cpu().numpy().ravel(), w.cpu().numpy().ravel(), dy[:q].cpu().numpy().ravel()
    ry = orc.conv_fwd(xs, ws, q, n, d, k, o, s, p)
    rdx = orc.conv_bwd_data(dys, ws, q, n, d, k, o, s, p)
    rdw = _fp64_wgrad(x, w, dy, s, p)
    errs = {}
    for t in (1, 2, 3):
        y = conv.conv_fwd(x, w, desc, t)
        dx = conv.conv_bwd_data(dy, w, desc, t)
        dw = conv.conv_bwd_weight(x, dy, desc, t)
        cache = conv.alloc_cache(desc, t, dev)
        yc = conv.conv_fwd_cached(x, w, desc, t, cache=cache)
        dxc, dwc = conv.conv_bwd(dy, w, desc, t, x=x, cache=cache)
        errs[t] = (rel_l2(y[:q].cpu().numpy().ravel(), ry), rel_l2(dx[:q].cpu().numpy().ravel(), rdx),
                   _rel(dw, rdw), rel_l2(yc[:q].cpu().numpy().ravel(), ry),
                   rel_l2(dxc[:q].cpu().numpy().ravel(), rdx), _rel(dwc, rdw))
        del cache
    worst = max(max(e) for e in errs.values())
    assert worst <= TOL, errs


@pytest.mark.timeout(900, method="thread")
def test_conv1_b256_bench_path(cct, dev):
    """conv1 (227x227x3 -> 96, k11, s4) at b = 256 exactly as bench.py runs it: the cost
    model's lowering (and its space-to-depth / slab-major decisions at this batch), the
    lowered cache, the full-batch backward-weight split count -- against fp64 torch."""
    import torch.nn.functional as F
    from paper_1504_04343_b200 import conv
    from paper_1504_04343_b200.stack import CAFFENET, ConvStack
    st = ConvStack(256, dev, CAFFENET[:1])
    st.step()
    torch.cuda.synchronize()
    x, w, dy = st.x[0], st.w[0], st.dy[0]
    xd = x.double().permute(0, 3, 1, 2).contiguous()
    wd = w.double().permute(0, 3, 1, 2).contiguous()
    ry = F.conv2d(xd, wd, stride=4)
    rdx = torch.nn.grad.conv2d_input(xd.shape, wd, dy.double(), stride=4).permute(0, 2, 3, 1)
    rdw = torch.nn.grad.conv2d_weight(xd, wd.shape, dy.double(), stride=4).permute(0, 2, 3, 1)
    e = (_rel(st.y[0], ry), _rel(st.dx[0], rdx), _rel(st.dw[0], rdw))
    assert max(e) <= TOL, e
    # and the stand-alone passes agree with the training step within the tolerance
    desc = st.descs[0]
    assert _rel(conv.conv_fwd(x, w, desc, st.types[0]), ry) <= TOL
