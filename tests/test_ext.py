"""Layer extension: grouped convolution (bvlc_reference_caffenet
group = 2 on conv2/4/5) and the bias + ReLU epilogue, through cct_conv_fwd_ex /
cct_conv_bwd_ex, against the oracle (per-group restatement, oracle_py.grouped_*) and
fp64 torch at CaffeNet sizes.  Tolerance: relative L2 <= 1e-4 per tensor."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle_py import grouped_bwd, grouped_fwd, rel_l2

TOL = 1e-4


def T(a, dev, *shape):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).view(*shape)


def test_bad_groups_are_config_errors(cct):
    """CPU: groups must divide d and o; relu is 0/1 (no device needed to reject)."""
    desc = cct.ConvDesc(13, 3, 96, 256, 2, 1, 1)
    out = C.c_size_t()
    for ext in (cct.ConvExt(5, None, 0), cct.ConvExt(0, None, 0), cct.ConvExt(2, None, 3)):
        rc = cct.lib().cct_workspace_size_ex(C.byref(desc.c()), 1, C.byref(ext), 0, C.byref(out))
        assert rc == 1, rc  # CCT_ERR_CONFIG
    ok = cct.lib().cct_workspace_size_ex(C.byref(desc.c()), 1, C.byref(cct.ConvExt(2, None, 1)), 3, C.byref(out))
    assert ok == 0 and out.value > 0


CASES = [  # (name, n, k, d, o, s, p, groups)
    ("g2_implicit", 13, 3, 64, 48, 1, 1, 2),      # d/G = 32: direct implicit groups
    ("g2_conv2like", 15, 5, 96, 64, 1, 2, 2),     # d/G = 48: dk-padded implicit wgrad
    ("g4_small", 11, 3, 16, 32, 1, 1, 4),         # d/G = 4: gathered groups
    ("g2_strided", 23, 5, 8, 16, 2, 1, 2),        # strided, gathered
    ("g1_bias_relu", 12, 3, 16, 24, 1, 1, 1),
]


@pytest.mark.gpu
@pytest.mark.parametrize("t", [1, 2, 3])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_grouped_bias_relu_vs_oracle(cct, dev, orc, case, t):
    from paper_1504_04343_b200 import conv
    _, n, k, d, o, s, p, G = case
    b = 3
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    m = desc.m
    x_np = orc.uniform(41, b * n * n * d)
    w_np = orc.uniform(42, o * k * k * (d // G))
    bias_np = orc.uniform(43, o)
    dy_np = orc.uniform(44, b * o * m * m)
    x, w = T(x_np, dev, b, n, n, d), T(w_np, dev, o, k, k, d // G)
    bias, dy = T(bias_np, dev, o), T(dy_np, dev, b, o, m, m)
    y = conv.conv_fwd_ex(x, w, desc, t, groups=G, bias=bias, relu=True)
    ry = grouped_fwd(orc, x_np, w_np, b, n, d, k, o, s, p, G, bias_np, relu=True)
    assert rel_l2(y.cpu().numpy().ravel(), ry.ravel()) <= TOL
    dx, dw, db = conv.conv_bwd_ex(dy, w, desc, t, groups=G, relu=True, x=x, y=y, need_db=True)
    dz = dy_np.reshape(b, o, m, m) * (y.cpu().numpy() > 0)          # mask of the device y
    rdx, rdw, rdb = grouped_bwd(orc, dz, x_np, w_np, b, n, d, k, o, s, p, G)
    errs = (rel_l2(dx.cpu().numpy().ravel(), rdx.ravel()), rel_l2(dw.cpu().numpy().ravel(), rdw.ravel()),
            rel_l2(db.cpu().numpy().astype(np.float64), rdb))
    assert max(errs) <= TOL, errs
    # determinism
    dx2, dw2, db2 = conv.conv_bwd_ex(dy, w, desc, t, groups=G, relu=True, x=x, y=y, need_db=True)
    assert torch.equal(dx, dx2) and torch.equal(dw, dw2) and torch.equal(db, db2)


@pytest.mark.gpu
def test_no_bias_no_relu_equals_plain_conv(cct, dev, orc):
    """groups = 1, no epilogue: the extension is exactly cct_conv_fwd / bwd."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 13, 3, 32, 32, 2, 1, 1
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
    assert torch.equal(conv.conv_fwd_ex(x, w, desc, 1), conv.conv_fwd(x, w, desc, 1))
    dx, dw, _ = conv.conv_bwd_ex(dy, w, desc, 1, x=x)
    assert torch.equal(dx, conv.conv_bwd_data(dy, w, desc, 1)) and torch.equal(dw, conv.conv_bwd_weight(x, dy, desc, 1))


@pytest.mark.gpu
@pytest.mark.parametrize("layer", [("conv2", 27, 5, 96, 256, 1, 2), ("conv4", 13, 3, 384, 384, 1, 1),
                                   ("conv5", 13, 3, 384, 256, 1, 1)], ids=lambda l: l[0])
def test_caffenet_grouped_layers_vs_fp64_torch(cct, dev, layer):
    """bvlc_reference_caffenet's grouped layers (group = 2) with bias + ReLU at b = 64 (auto
    lowering) against fp64 torch (checker only): y, dx, dw, db."""
    import torch.nn.functional as F
    from paper_1504_04343_b200 import conv
    _, n, k, d, o, s, p = layer
    G, b = 2, 64
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    g = torch.Generator(device=dev).manual_seed(23)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d // G), generator=g, device=dev) * 2 - 1
    bias = torch.rand((o,), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
    y = conv.conv_fwd_ex(x, w, desc, groups=G, bias=bias, relu=True)
    dx, dw, db = conv.conv_bwd_ex(dy, w, desc, groups=G, relu=True, x=x, y=y, need_db=True)
    xd = x.double().permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    wd = w.double().permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    bd = bias.double().requires_grad_(True)
    z = F.conv2d(xd, wd, bd, stride=s, padding=p, groups=G)
    mask = (y > 0).double()                       # the device output's mask (ties at 0 are measure-zero)
    ry = torch.relu(z)
    (z * mask * dy.double()).sum().backward()

    def rel(a, r):
        return float(torch.linalg.norm(a.double() - r) / torch.linalg.norm(r))
    errs = (rel(y, ry.detach()), rel(dx, xd.grad.permute(0, 2, 3, 1)), rel(dw, wd.grad.permute(0, 2, 3, 1)),
            rel(db, bd.grad))
    assert max(errs) <= TOL, errs
