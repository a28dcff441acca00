"""The y / dy layout option of the boundary (cct_layout {NCHW, NHWC}).

NCHW is the reference's OutputBatch (tensor.hpp:135-150); NHWC is the DataBatch
order of the next layer's input (tensor.hpp:28-35).  Every pass, every lowering
type and every internal form (materialised, implicit, swapped, space-to-depth,
the cached training step, batch chunks) must give the same numbers in both
layouts (NHWC = the NCHW result transposed) and match the oracle.
"""
import ctypes as C

import numpy as np
import pytest

from oracle_py import rel_l2

TOL = 1e-4


def test_desc_layout_validation():
    """CPU: cct_conv_desc_init defaults to NCHW; set_layout range-checks; y_shape follows."""
    import paper_1504_04343_b200 as cct
    d = cct.ConvDesc(13, 3, 8, 16, 2, 1, 1)
    assert d.c().layout == cct.NCHW and d.y_shape() == (2, 16, 13, 13)
    dn = cct.ConvDesc(13, 3, 8, 16, 2, 1, 1, cct.NHWC)
    assert dn.c().layout == cct.NHWC and dn.y_shape() == (2, 13, 13, 16)
    raw = dn.c()
    assert cct.lib().cct_conv_desc_set_layout(C.byref(raw), 7) == cct.ERR_CONFIG
    raw.layout = 5  # a corrupted descriptor is rejected by every entry point
    out = C.c_size_t()
    assert cct.lib().cct_workspace_size(C.byref(raw), 1, 0, C.byref(out)) == cct.ERR_CONFIG


CASES = [
    # name, (n, k, d, o, b, s, p), types, tuning
    ("pad1", (13, 3, 64, 96, 3, 1, 1), (1, 2, 3), {}),
    ("conv1like", (23, 11, 3, 96, 2, 4, 0), (1, 2, 3), {}),
    ("conv2like", (27, 5, 96, 256, 2, 1, 2), (1, 2, 3), {}),
    ("implicit_bwd", (13, 3, 64, 96, 3, 1, 1), (1,), {"implicit_bwd": 2}),
    ("dgrad_swap", (13, 3, 96, 64, 3, 1, 1), (1,), {"implicit_bwd": 2, "dgrad_swap": 2}),
    ("s2d", (23, 11, 3, 96, 2, 4, 0), (1,), {"s2d": 2}),
    ("fwd_swap", (19, 3, 16, 64, 4, 1, 1), (1,), {"fwd_swap": 1}),
    ("stride2", (15, 5, 8, 12, 3, 2, 2), (1, 2, 3), {}),
    ("odd_o", (11, 3, 8, 10, 2, 1, 1), (1, 2, 3), {}),
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_nhwc_matches_nchw_and_oracle(cct, dev, orc, case):
    import torch
    from paper_1504_04343_b200 import conv
    name, (n, k, d, o, b, s, p), types, tune = case
    x, w = orc.random_problem(31, b, n, d, k, o)
    m = (n + 2 * p - k) // s + 1
    dy = orc.uniform(32, b * o * m * m)
    ry = orc.conv_fwd(x, w, b, n, d, k, o, s, p)
    rdx = orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p)
    rdw = orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p)
    xt = torch.from_numpy(x).to(dev).view(b, n, n, d)
    wt = torch.from_numpy(w).to(dev).view(o, k, k, d)
    dyc = torch.from_numpy(dy).to(dev).view(b, o, m, m)
    dyn = dyc.permute(0, 2, 3, 1).contiguous()
    dc = cct.ConvDesc(n, k, d, o, b, s, p)
    dn = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    with cct.tuning(**tune):
        for t in types:
            yc, yn = conv.conv_fwd(xt, wt, dc, t), conv.conv_fwd(xt, wt, dn, t)
            dxc, dxn = conv.conv_bwd_data(dyc, wt, dc, t), conv.conv_bwd_data(dyn, wt, dn, t)
            dwc, dwn = conv.conv_bwd_weight(xt, dyc, dc, t), conv.conv_bwd_weight(xt, dyn, dn, t)
            cache = conv.alloc_cache(dn, t, dev)
            ytn = conv.conv_fwd_cached(xt, wt, dn, t, cache=cache)
            dxt, dwt = conv.conv_bwd(dyn, wt, dn, t, x=xt, cache=cache)
            yn_c = yn.permute(0, 3, 1, 2).contiguous()
            ytn_c = ytn.permute(0, 3, 1, 2).contiguous()
            for a, bb in ((yn_c, yc), (ytn_c, yc), (dxn, dxc), (dxt, dxc), (dwn, dwc), (dwt, dwc)):
                assert rel_l2(a.cpu().numpy().ravel(), bb.cpu().numpy().ravel()) <= 1e-6, (name, t)
            e = (rel_l2(yn_c.cpu().numpy().ravel(), ry), rel_l2(dxn.cpu().numpy().ravel(), rdx),
                 rel_l2(dwn.cpu().numpy().ravel(), rdw))
            assert max(e) <= TOL, (name, t, e)


@pytest.mark.gpu
def test_nhwc_batch_chunks(cct, dev, orc):
    """Chunked passes (workspace limit) in NHWC: image offsets of y / dy are the same per image."""
    import torch
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 13, 3, 16, 32, 6, 1, 1
    x, w = orc.random_problem(41, b, n, d, k, o)
    dy = orc.uniform(42, b * o * n * n)
    dn = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    xt = torch.from_numpy(x).to(dev).view(b, n, n, d)
    wt = torch.from_numpy(w).to(dev).view(o, k, k, d)
    dyn = torch.from_numpy(dy).to(dev).view(b, o, n, n).permute(0, 2, 3, 1).contiguous()
    L = cct.lib()
    old = L.cct_get_workspace_limit()
    try:
        for t in (1, 2, 3):
            L.cct_set_workspace_limit(1 << 16)  # forces several chunks
            y = conv.conv_fwd(xt, wt, dn, t).permute(0, 3, 1, 2).contiguous()
            dx = conv.conv_bwd_data(dyn, wt, dn, t)
            dw = conv.conv_bwd_weight(xt, dyn, dn, t)
            L.cct_set_workspace_limit(old)
            assert rel_l2(y.cpu().numpy().ravel(), orc.conv_fwd(x, w, b, n, d, k, o, s, p)) <= TOL
            assert rel_l2(dx.cpu().numpy().ravel(), orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p)) <= TOL
            assert rel_l2(dw.cpu().numpy().ravel(), orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p)) <= TOL
    finally:
        L.cct_set_workspace_limit(old)


@pytest.mark.gpu
def test_nhwc_ex_is_unsupported(cct, dev):
    import torch
    from paper_1504_04343_b200 import conv
    dn = cct.ConvDesc(13, 3, 16, 32, 2, 1, 1, cct.NHWC)
    x = torch.zeros((2, 13, 13, 16), device=dev)
    w = torch.zeros((32, 3, 3, 16), device=dev)
    with pytest.raises(cct.ConfigError, match="NCHW"):
        conv.conv_fwd_ex(x, w, dn, 1, groups=1)
    assert np.isfinite(0.0)
