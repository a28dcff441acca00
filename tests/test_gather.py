"""Fused small-channel Type 1 (csrc/gather.cu): the lowered matrix is gathered from staged
input rows inside the tcgen05 GEMM (CaffeNet conv1 class: d * stride % 4 == 0).

Parity against the oracle (direct_convolve restatement, tensor.cpp:77-106) at rel-L2
<= 1e-4, the fused path proven to have run (no lowering phase recorded), and agreement
with the materialised Type 1 path it replaces (CCT_TUNE_GATHER = 0).
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle_py import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-4

# (n, k, d, o, b, stride, pad): conv1, torchvision AlexNet conv1, and geometries that
# exercise padding, o not a multiple of 16, every tile width (32 / 64 / 96 / 128 / 192),
# d = 1 / 2 / 4 / 6, tiles spanning up to 4 output rows, ragged last tiles
GEOMS = [
    (227, 11, 3, 96, 2, 4, 0),
    (224, 11, 3, 64, 2, 4, 2),
    (31, 5, 2, 96, 3, 2, 1),
    (20, 3, 4, 128, 2, 1, 1),
    (17, 7, 1, 40, 3, 4, 3),
    (40, 4, 6, 192, 2, 2, 0),
    (9, 9, 3, 16, 2, 4, 4),
    (63, 11, 3, 96, 1, 4, 5),
]


def _phases(cct, fn):
    L = cct.lib()
    P = C.c_double * 7
    ms, fl, by = P(), P(), P()
    n = (C.c_uint64 * 7)()
    L.cct_profile_read(None, None, None, None, 1)
    L.cct_profile_enable(1)
    out = fn()
    L.cct_profile_enable(0)
    L.cct_profile_read(ms, fl, by, n, 1)
    return out, list(n)


@pytest.mark.parametrize("geom", GEOMS, ids=[f"n{g[0]}k{g[1]}d{g[2]}o{g[3]}s{g[5]}p{g[6]}" for g in GEOMS])
def test_gather_fwd_vs_oracle(cct, dev, orc, geom):
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = geom
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x, w = orc.random_problem(7 + n, b, n, d, k, o)
    ref = orc.conv_fwd(x, w, b, n, d, k, o, s, p)
    xt = torch.from_numpy(x).to(dev).view(b, n, n, d)
    wt = torch.from_numpy(w).to(dev).view(o, k, k, d)
    y, launches = _phases(cct, lambda: conv.conv_fwd(xt, wt, desc, cct.LOWER_T1))
    assert launches[0] == 0, "the fused path must not run a lowering kernel"
    err = rel_l2(y.cpu().numpy().ravel(), ref)
    assert err <= TOL, f"rel-L2 {err:.3e}"
    with cct.tuning(gather=0):
        y0 = conv.conv_fwd(xt, wt, desc, cct.LOWER_T1)
    assert rel_l2(y.cpu().numpy().ravel(), y0.cpu().numpy().ravel()) <= TOL


def test_gather_fwd_nhwc_and_repeatable(cct, dev, orc):
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 227, 11, 3, 96, 3, 4, 0
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    dn = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    y = conv.conv_fwd(x, w, desc, cct.LOWER_T1)
    yn = conv.conv_fwd(x, w, dn, cct.LOWER_T1)
    assert torch.equal(yn.view(b, desc.m, desc.m, o).permute(0, 3, 1, 2).contiguous(), y.view(b, o, desc.m, desc.m))
    for _ in range(3):
        assert torch.equal(conv.conv_fwd(x, w, desc, cct.LOWER_T1), y)


def test_gather_fwd_full_batch_slices(cct, dev, orc):
    """conv1 at b = 256 (BASELINE configs[2]): image slices against the oracle."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 227, 11, 3, 96, 256, 4, 0
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    g = torch.Generator(device=dev).manual_seed(11)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    y = conv.conv_fwd(x, w, desc, cct.LOWER_T1).cpu().numpy()
    wn = w.cpu().numpy().ravel()
    for q in (0, 1, 127, 255):
        ref = orc.conv_fwd(x[q].cpu().numpy().ravel(), wn, 1, n, d, k, o, s, p)
        assert rel_l2(y[q].ravel(), ref) <= TOL


def test_gather_fwd_bias_relu(cct, dev, orc):
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 227, 11, 3, 96, 2, 4, 0
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x, w = orc.random_problem(5, b, n, d, k, o)
    bias = orc.uniform(6, o)
    ref = orc.conv_fwd(x, w, b, n, d, k, o, s, p).reshape(b, o, -1) + bias[None, :, None]
    ref = np.maximum(ref, 0).ravel()
    xt = torch.from_numpy(x).to(dev).view(b, n, n, d)
    wt = torch.from_numpy(w).to(dev).view(o, k, k, d)
    y = conv.conv_fwd_ex(xt, wt, desc, cct.LOWER_T1, bias=torch.from_numpy(bias).to(dev), relu=True)
    assert rel_l2(y.cpu().numpy().ravel(), ref) <= TOL


# ---------------------------------------------------------------------------
# fused backward-weight (conv_wgrad_gather_kernel): dW^T = lowered(x)^T dy with the
# lowered columns gathered into TMEM; o % 4 == 0, o <= 128, k k d <= 384, m >= 16
WGEOMS = [g for g in GEOMS if g[3] % 4 == 0 and g[3] <= 128 and g[1] * g[1] * g[2] <= 384 and
          (g[0] + 2 * g[6] - g[1]) // g[5] + 1 >= 16]


@pytest.mark.parametrize("layout", [0, 1], ids=["nchw", "nhwc"])
@pytest.mark.parametrize("geom", WGEOMS, ids=[f"n{g[0]}k{g[1]}d{g[2]}o{g[3]}s{g[5]}p{g[6]}" for g in WGEOMS])
def test_gather_wgrad_vs_oracle(cct, dev, orc, geom, layout):
    """dW against the oracle's backward-weight (tensor.cpp:77-106 adjoint) at rel-L2 <= 1e-4,
    no lowering kernel launched, and agreement with the materialised Type 1 path."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = geom
    desc = cct.ConvDesc(n, k, d, o, b, s, p, layout)
    x, _ = orc.random_problem(17 + n, b, n, d, k, o)
    m = desc.m
    dy = orc.uniform(18 + n, b * o * m * m)  # NCHW order
    ref = orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p)
    xt = torch.from_numpy(x).to(dev).view(b, n, n, d)
    dyt = torch.from_numpy(dy).to(dev).view(b, o, m, m)
    if layout:
        dyt = dyt.permute(0, 2, 3, 1).contiguous()
    dw, launches = _phases(cct, lambda: conv.conv_bwd_weight(xt, dyt, desc, cct.LOWER_T1))
    assert launches[0] == 0, "the fused path must not run a lowering kernel"
    err = rel_l2(dw.cpu().numpy().ravel(), ref)
    assert err <= TOL, f"rel-L2 {err:.3e}"
    with cct.tuning(gather=0):
        dw0 = conv.conv_bwd_weight(xt, dyt, desc, cct.LOWER_T1)
    assert rel_l2(dw.cpu().numpy().ravel(), dw0.cpu().numpy().ravel()) <= TOL
    # deterministic: fixed chains, fixed-order reduction
    assert torch.equal(conv.conv_bwd_weight(xt, dyt, desc, cct.LOWER_T1), dw)


def test_gather_wgrad_full_batch(cct, dev):
    """conv1 at b = 256 (BASELINE configs[2]; 296 chains): against an fp64 torch reference
    of the same lowered product, and the combined backward (dx + dW in one call)."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 227, 11, 3, 96, 256, 4, 0
    desc = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    g = torch.Generator(device=dev).manual_seed(21)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    m = desc.m
    dy = torch.rand((b, m, m, o), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dw = conv.conv_bwd_weight(x, dy, desc, cct.LOWER_T1)
    # fp64 reference: unfold x (NCHW view) into the lowered matrix, one image chunk at a time
    ref = torch.zeros((o, d * k * k), dtype=torch.float64, device=dev)
    for q0 in range(0, b, 32):
        xc = x[q0:q0 + 32].permute(0, 3, 1, 2).double()
        cols = torch.nn.functional.unfold(xc, k, stride=s, padding=p)          # (bq, d k k, m m)
        dyc = dy[q0:q0 + 32].reshape(-1, m * m, o).double()                    # (bq, m m, o)
        ref += torch.einsum("bcp,bpo->oc", cols, dyc)
    ref = ref.view(o, d, k, k).permute(0, 2, 3, 1).reshape(o, k, k, d)
    err = (torch.linalg.norm(dw.double() - ref) / torch.linalg.norm(ref)).item()
    assert err <= TOL, f"rel-L2 {err:.3e}"
    dx, dw2 = conv.conv_bwd(dy, w, desc, cct.LOWER_T1, x=x)
    assert torch.equal(dw2, dw)


# ---------------------------------------------------------------------------
# fused backward-data (conv_dgrad_hfold_kernel + vfold_kernel): dDhat never reaches HBM,
# the horizontal overlap is folded in the GEMM epilogue, the vertical one by a streaming pass.
# Instantiated fold geometries (k d, s d): (33, 12) conv1 / AlexNet conv1, (20, 8), (28, 16).
DGEOMS = [
    (227, 11, 3, 96, 2, 4, 0),   # CaffeNet conv1
    (224, 11, 3, 64, 2, 4, 2),   # torchvision AlexNet conv1 (pad 2)
    (63, 11, 3, 96, 1, 4, 5),    # pad > k / 2, m = 16
    (31, 5, 4, 32, 2, 2, 1),     # k d = 20, s d = 8, ragged right edge
    (40, 7, 4, 48, 3, 4, 3),     # k d = 28, s d = 16
    (531, 11, 3, 16, 1, 4, 0),   # m = 131 > 128: an output row spans tiles
    (15, 11, 3, 8, 5, 4, 2),     # m = 2: tiles span many images
]


@pytest.mark.parametrize("layout", [0, 1], ids=["nchw", "nhwc"])
@pytest.mark.parametrize("geom", DGEOMS, ids=[f"n{g[0]}k{g[1]}d{g[2]}o{g[3]}s{g[5]}p{g[6]}" for g in DGEOMS])
def test_hfold_dgrad_vs_oracle(cct, dev, orc, geom, layout):
    """dx against the oracle's backward-data (the adjoint of tensor.cpp:77-106) at rel-L2 <=
    1e-4, bitwise repeatable, and in agreement with the materialised Type 1 path."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = geom
    desc = cct.ConvDesc(n, k, d, o, b, s, p, layout)
    _, w = orc.random_problem(23 + n, b, n, d, k, o)
    m = desc.m
    dy = orc.uniform(24 + n, b * o * m * m)  # NCHW order
    ref = orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p)
    wt = torch.from_numpy(w).to(dev).view(o, k, k, d)
    dyt = torch.from_numpy(dy).to(dev).view(b, o, m, m)
    if layout:
        dyt = dyt.permute(0, 2, 3, 1).contiguous()
    dx = conv.conv_bwd_data(dyt, wt, desc, cct.LOWER_T1)
    err = rel_l2(dx.cpu().numpy().ravel(), ref)
    assert err <= TOL, f"rel-L2 {err:.3e}"
    assert torch.equal(conv.conv_bwd_data(dyt, wt, desc, cct.LOWER_T1), dx)
    with cct.tuning(gather=0):
        dx0 = conv.conv_bwd_data(dyt, wt, desc, cct.LOWER_T1)
    assert rel_l2(dx.cpu().numpy().ravel(), dx0.cpu().numpy().ravel()) <= TOL


def test_hfold_dgrad_full_batch(cct, dev):
    """conv1 at b = 256 (BASELINE configs[2]): dx against an fp64 torch reference (fold of the
    fp64 lowered product), and the combined backward (dx + dW in one call)."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 227, 11, 3, 96, 256, 4, 0
    desc = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    g = torch.Generator(device=dev).manual_seed(31)
    m = desc.m
    dy = torch.rand((b, m, m, o), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    dx = conv.conv_bwd_data(dy, w, desc, cct.LOWER_T1)
    wm = w.permute(0, 3, 1, 2).reshape(o, d * k * k).double()                  # (o, d k k) unfold order
    num = den = 0.0
    for q0 in range(0, b, 32):
        cols = torch.einsum("bpo,oc->bcp", dy[q0:q0 + 32].reshape(-1, m * m, o).double(), wm)
        ref = torch.nn.functional.fold(cols, (n, n), k, stride=s, padding=p)  # (bq, d, n, n)
        got = dx[q0:q0 + 32].permute(0, 3, 1, 2).double()
        num += float(((got - ref) ** 2).sum())
        den += float((ref ** 2).sum())
    err = (num / den) ** 0.5
    assert err <= TOL, f"rel-L2 {err:.3e}"
    dx2, dw2 = conv.conv_bwd(dy, w, desc, cct.LOWER_T1, x=x)
    assert torch.equal(dx2, dx)
    # CCT_TUNE_OVERLAP: the backward-weight on the side stream beside the vertical fold, joined
    # back into the call's stream -- same bits as one stream, and ordered for the caller
    with cct.tuning(overlap=0):
        dx3, dw3 = conv.conv_bwd(dy, w, desc, cct.LOWER_T1, x=x)
    assert torch.equal(dx3, dx) and torch.equal(dw3, dw2)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dx4, dw4 = conv.conv_bwd(dy, w, desc, cct.LOWER_T1, x=x, stream=s)
        dw5 = dw4.clone()  # consumer on the caller's stream right after the call
    s.synchronize()
    assert torch.equal(dx4, dx) and torch.equal(dw5, dw2)


def test_fused_conv1_under_workspace_limit(cct, dev):
    """The fused conv1 passes under a workspace limit that forces batch chunks (SPEC batching
    module): forward, backward-data and backward-weight agree with the unchunked call."""
    from paper_1504_04343_b200 import conv
    L = cct.lib()
    n, k, d, o, b, s, p = 227, 11, 3, 96, 12, 4, 0
    desc = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    g = torch.Generator(device=dev).manual_seed(41)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, desc.m, desc.m, o), generator=g, device=dev) * 2 - 1
    full = (conv.conv_fwd(x, w, desc, 1), conv.conv_bwd_data(dy, w, desc, 1), conv.conv_bwd_weight(x, dy, desc, 1))
    old = L.cct_get_workspace_limit()
    unlimited = cct.workspace_size(desc, 1, cct.PASS_BWD)
    try:
        L.cct_set_workspace_limit(8 << 20)
        assert cct.workspace_size(desc, 1, cct.PASS_BWD) < unlimited  # the batch is chunked
        ch = (conv.conv_fwd(x, w, desc, 1), conv.conv_bwd_data(dy, w, desc, 1), conv.conv_bwd_weight(x, dy, desc, 1))
        dx2, dw2 = conv.conv_bwd(dy, w, desc, 1, x=x)
    finally:
        L.cct_set_workspace_limit(old)

    def close(a, ref):
        return float(torch.linalg.norm(a - ref) / torch.linalg.norm(ref)) < 1e-5
    assert torch.equal(ch[0], full[0]) and torch.equal(ch[1], full[1])  # per-image passes: same bits
    assert close(ch[2], full[2]) and close(dw2, full[2]) and torch.equal(dx2, full[1])
