"""GPU parity: the B200 path (libcct.so through the C ABI) against the oracle.

Tolerance (north_star): relative L2 <= 1e-4 per output / gradient tensor, for
every lowering type.  Pure data-movement phases (lower, Khat) are bit-exact.
Sizes: small batches against the oracle and the reference golden vectors;
BASELINE sizes (b = 256) through size-independent properties (linearity,
the fwd/bwd adjoint identity, determinism) plus an image-slice oracle check.
"""
import glob
import os

import numpy as np
import pytest
import torch

from oracle_py import rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-4
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CONV_CASES = sorted(glob.glob(os.path.join(GOLD, "c*.npz")))
CAFFENET = [("conv1", 227, 11, 3, 96, 4, 0), ("conv2", 27, 5, 96, 256, 1, 2), ("conv3", 13, 3, 256, 384, 1, 1),
            ("conv4", 13, 3, 384, 384, 1, 1), ("conv5", 13, 3, 384, 256, 1, 1)]


def T(a, dev, *shape):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).view(*shape)


def run3(cct, dev, x, w, dy, n, k, d, o, b, s, p, t):
    from paper_1504_04343_b200 import conv
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    m = desc.m
    xt, wt, dyt = T(x, dev, b, n, n, d), T(w, dev, o, k, k, d), T(dy, dev, b, o, m, m)
    y = conv.conv_fwd(xt, wt, desc, t)
    dx = conv.conv_bwd_data(dyt, wt, desc, t)
    dw = conv.conv_bwd_weight(xt, dyt, desc, t)
    return y.cpu().numpy().ravel(), dx.cpu().numpy().ravel(), dw.cpu().numpy().ravel()


# ------------------------------------------------------------------- GEMM
def test_gemm_kat(cct, dev):
    from paper_1504_04343_b200 import conv
    a = torch.tensor([[1., 2.], [3., 4.]], device=dev)
    b = torch.tensor([[5., 6.], [7., 8.]], device=dev)
    assert conv.multiply(a, b).cpu().tolist() == [[19, 22], [43, 50]]
    e = torch.eye(5, device=dev)
    bb = torch.rand(5, 7, device=dev)
    # identity: the small half is itself read as tf32, so 3xTF32 is
    # exact to ~2^-22 relative, not bit-exact
    assert float(((conv.multiply(e, bb) - bb).abs() / bb.abs()).max()) < 2.0 ** -20


def test_tf32_operand_truncation(cct, dev):
    """The tensor core reads fp32 operands as tf32 by truncation: raw fp32 is the 'big' half."""
    from paper_1504_04343_b200 import conv
    v = 1.0 + 3 * 2.0 ** -12
    a = torch.zeros((128, 16), device=dev)
    a[:, 0] = v
    b = torch.zeros((16, 128), device=dev)
    b[0, :] = 1.0
    assert conv.multiply_passes(a, b, 1)[0, 0].item() == 1.0
    assert conv.multiply_passes(a, b, 3)[0, 0].item() == v


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "g*.npz"))))
def test_gemm_vs_reference_golden(cct, dev, path):
    from paper_1504_04343_b200 import conv
    z = np.load(path)
    c = conv.multiply(torch.from_numpy(z["A"]).to(dev), torch.from_numpy(z["B"]).to(dev)).cpu().numpy()
    assert rel_l2(c, z["C"]) < 1e-5


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (3, 5, 7), (129, 257, 1000), (1000, 96, 363), (256, 256, 32768)])
def test_gemm_shapes_and_long_k(cct, dev, orc, M, N, K):
    from paper_1504_04343_b200 import conv
    A = orc.uniform(M + 1, M * K).reshape(M, K)
    B = orc.uniform(N + 2, K * N).reshape(K, N)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    c = conv.multiply(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)).cpu().numpy()
    assert rel_l2(c, ref) < 1e-5  # long K is chain-split (truncating accumulator)


def test_gemm_deterministic(cct, dev):
    from paper_1504_04343_b200 import conv
    a = torch.rand(300, 5000, device=dev)
    b = torch.rand(5000, 200, device=dev)
    c1 = conv.multiply(a, b)
    c2 = conv.multiply(a, b)
    assert torch.equal(c1, c2)


# ---------------------------------------------------------- lowering phases
@pytest.mark.parametrize("t", [1, 2, 3])
def test_lower_spec_bit_exact(cct, dev, orc, t):
    from paper_1504_04343_b200 import conv
    b, n, d, k, o = 2, 7, 3, 3, 4
    x, w = orc.random_problem(31, b, n, d, k, o)
    desc = cct.ConvDesc(n, k, d, o, b)
    dh_ref, kh_ref = orc.lower(t, x, w, b, n, d, k, o)
    dh = conv.lower(T(x, dev, b, n, n, d), desc, t, cct.ROWS_SPEC).cpu().numpy()
    kh = conv.lower_khat(T(w, dev, o, k, k, d), desc, t).cpu().numpy()
    assert np.array_equal(dh, dh_ref) and np.array_equal(kh, kh_ref)
    # lift(Rhat) in the SPEC row order vs the oracle lift
    rh = orc.multiply(dh_ref, kh_ref)
    y = conv.lift(torch.from_numpy(rh).to(dev), desc, t, cct.ROWS_SPEC).cpu().numpy().ravel()
    assert rel_l2(y, orc.lift(t, rh, b, n, d, k, o)) < 1e-6


@pytest.mark.parametrize("t", [1, 2, 3])
@pytest.mark.parametrize("geom", [(9, 3, 4, 1, 0), (11, 3, 8, 1, 1), (13, 5, 4, 2, 2), (23, 11, 3, 4, 0)])
def test_lower_internal_bit_exact(cct, dev, orc, t, geom):
    from paper_1504_04343_b200 import conv
    n, k, d, s, p = geom
    b = 2
    x = orc.uniform(41, b * n * n * d)
    desc = cct.ConvDesc(n, k, d, 5, b, s, p)
    dh = conv.lower(T(x, dev, b, n, n, d), desc, t, cct.ROWS_INTERNAL).cpu().numpy()
    assert np.array_equal(dh, orc.lower_internal(t, x, b, n, d, k, s, p))


@pytest.mark.parametrize("geom", [(23, 11, 3, 4, 4), (19, 5, 3, 2, 4), (21, 7, 3, 1, 8), (227, 11, 3, 4, 4)],
                         ids=["s4", "s2", "s1", "conv1"])
def test_lower_small_channel_float4_staging_bit_exact(cct, dev, orc, geom):
    """Unpadded small-channel Type 1 with b n^2 d % 4 == 0 takes lower_t1_vec_kernel (rows staged
    from the float4 boundary below each row start: every misalignment 0..3 occurs, since n d is
    odd here) -- bit-exact against the oracle in both row orders."""
    from paper_1504_04343_b200 import conv
    n, k, d, s, b = geom
    assert (b * n * n * d) % 4 == 0 and (n * d) % 2 == 1
    x = orc.uniform(43, b * n * n * d)
    desc = cct.ConvDesc(n, k, d, 5, b, s, 0)
    dh = conv.lower(T(x, dev, b, n, n, d), desc, 1, cct.ROWS_INTERNAL).cpu().numpy()
    assert np.array_equal(dh, orc.lower_internal(1, x, b, n, d, k, s, 0))
    if s == 1:
        xs, w = orc.random_problem(47, b, n, d, k, 4)
        dh_ref, _ = orc.lower(1, xs, w, b, n, d, k, 4)
        dh = conv.lower(T(xs, dev, b, n, n, d), cct.ConvDesc(n, k, d, 4, b), 1, cct.ROWS_SPEC).cpu().numpy()
        assert np.array_equal(dh, dh_ref)


# --------------------------------------------------------- full conv passes
@pytest.mark.parametrize("t", [1, 2, 3])
@pytest.mark.parametrize("path", CONV_CASES, ids=[os.path.basename(p)[:-4] for p in CONV_CASES])
def test_conv_vs_reference_golden(cct, dev, path, t):
    z = np.load(path)
    n, k, d, o, b, s, p = (int(v) for v in z["shape"])
    y, dx, dw = run3(cct, dev, z["x"], z["w"], z["dy"], n, k, d, o, b, s, p, t)
    errs = rel_l2(y, z["y"]), rel_l2(dx, z["dx"]), rel_l2(dw, z["dw"])
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("t", [1, 2, 3])
@pytest.mark.parametrize("layer", CAFFENET, ids=[l[0] for l in CAFFENET])
def test_caffenet_layers_vs_oracle(cct, dev, orc, layer, t):
    _, n, k, d, o, s, p = layer
    b = 2
    x, w = orc.random_problem(1234, b, n, d, k, o)
    m = (n + 2 * p - k) // s + 1
    dy = orc.uniform(1235, b * o * m * m)
    y, dx, dw = run3(cct, dev, x, w, dy, n, k, d, o, b, s, p, t)
    errs = (rel_l2(y, orc.conv_fwd(x, w, b, n, d, k, o, s, p)),
            rel_l2(dx, orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p)),
            rel_l2(dw, orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p)))
    assert max(errs) <= TOL, errs


@pytest.mark.parametrize("geom", [(5, 5, 2, 3, 1, 1, 0), (1, 1, 4, 4, 3, 1, 0), (6, 3, 5, 7, 1, 3, 2),
                                  (4, 4, 1, 1, 1, 1, 3)])
def test_edge_shapes(cct, dev, orc, geom):
    """n = k (single output pixel), 1x1 images, ragged stride, pad > k/2."""
    n, k, d, o, b, s, p = geom
    x, w = orc.random_problem(7, b, n, d, k, o)
    m = (n + 2 * p - k) // s + 1
    dy = orc.uniform(8, b * o * m * m)
    for t in (1, 2, 3):
        y, dx, dw = run3(cct, dev, x, w, dy, n, k, d, o, b, s, p, t)
        assert rel_l2(y, orc.conv_fwd(x, w, b, n, d, k, o, s, p)) <= TOL
        assert rel_l2(dx, orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p)) <= TOL
        assert rel_l2(dw, orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p)) <= TOL


T23_GEOMS = [(13, 3, 8, 12, 3, 1, 1), (11, 5, 4, 20, 2, 2, 2), (15, 3, 4, 5, 3, 3, 0), (12, 4, 8, 9, 2, 4, 1),
             (9, 1, 4, 7, 3, 2, 0), (27, 5, 4, 10, 1, 1, 2)]


@pytest.mark.parametrize("layout", [0, 1], ids=["nchw", "nhwc"])
@pytest.mark.parametrize("geom", T23_GEOMS, ids=[f"n{g[0]}k{g[1]}s{g[5]}p{g[6]}o{g[3]}" for g in T23_GEOMS])
def test_t23_streaming_kernels(cct, dev, orc, geom, layout):
    """The Type 2 / 3 streaming kernels -- lift from bulk-copied (double-buffered, 16-byte aligned
    down / up) tap-plane runs, expand as shifted copies of the dilated padded dy plane -- over
    strides 1-4, k = 1..5, partial channel groups (o not a multiple of the 8-channel block) and
    runs that start at every float phase (odd plane sizes): fwd, bwd-data, bwd-weight against the
    oracle, repeatable bit for bit."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = geom
    desc = cct.ConvDesc(n, k, d, o, b, s, p, layout)
    m = desc.m
    x_np, w_np = orc.random_problem(61 + n, b, n, d, k, o)
    dy_np = orc.uniform(62 + n, b * o * m * m)
    x, w = T(x_np, dev, b, n, n, d), T(w_np, dev, o, k, k, d)
    dy = T(dy_np, dev, b, o, m, m)
    if layout:
        dy = dy.permute(0, 2, 3, 1).contiguous()
    refs = (orc.conv_fwd(x_np, w_np, b, n, d, k, o, s, p), orc.conv_bwd_data(dy_np, w_np, b, n, d, k, o, s, p),
            orc.conv_bwd_weight(x_np, dy_np, b, n, d, k, o, s, p))
    for t in (2, 3):
        y = conv.conv_fwd(x, w, desc, t)
        dx = conv.conv_bwd_data(dy, w, desc, t)
        dw = conv.conv_bwd_weight(x, dy, desc, t)
        yc = y.permute(0, 3, 1, 2) if layout else y
        for got, ref in zip((yc, dx, dw), refs):
            assert rel_l2(got.contiguous().cpu().numpy().ravel(), ref) <= TOL, (t, geom)
        assert torch.equal(conv.conv_fwd(x, w, desc, t), y) and torch.equal(conv.conv_bwd_data(dy, w, desc, t), dx)


def test_auto_lowering_matches_oracle(cct, dev, orc):
    n, k, d, o, b, s, p = 13, 3, 64, 32, 2, 1, 1
    x, w = orc.random_problem(3, b, n, d, k, o)
    m = (n + 2 * p - k) // s + 1
    dy = orc.uniform(4, b * o * m * m)
    y, dx, dw = run3(cct, dev, x, w, dy, n, k, d, o, b, s, p, cct.LOWER_AUTO)
    assert rel_l2(y, orc.conv_fwd(x, w, b, n, d, k, o, s, p)) <= TOL


# ------------------------------------------- BASELINE sizes: properties + slice
@pytest.mark.parametrize("t", [1, 2, 3])
def test_conv2_b256_properties(cct, dev, orc, t):
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 27, 5, 96, 256, 256, 1, 2
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    m = desc.m
    g = torch.Generator(device=dev).manual_seed(5)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, m, m), generator=g, device=dev) * 2 - 1
    y = conv.conv_fwd(x, w, desc, t)
    dx = conv.conv_bwd_data(dy, w, desc, t)
    dw = conv.conv_bwd_weight(x, dy, desc, t)
    # determinism (fixed split-K order) and exact linearity (scaling by 2 commutes with the 3xTF32 split)
    assert torch.equal(conv.conv_fwd(x, w, desc, t), y)
    assert torch.equal(conv.conv_bwd_weight(x, dy, desc, t), dw)
    assert torch.equal(conv.conv_fwd(2 * x, w, desc, t), 2 * y)
    # adjoint identity <conv(x,w),dy> = <x,dgrad(dy,w)> = <w,wgrad(x,dy)>
    a1 = torch.dot(y.double().ravel(), dy.double().ravel())
    a2 = torch.dot(x.double().ravel(), dx.double().ravel())
    a3 = torch.dot(w.double().ravel(), dw.double().ravel())
    assert abs(a1 - a2) <= 1e-4 * abs(a1) and abs(a1 - a3) <= 1e-4 * abs(a1)
    # oracle on an image slice of the full-batch outputs (images are independent in fwd / dgrad)
    q = 2
    xs, ws, dys = x[:q].cpu().numpy().ravel(), w.cpu().numpy().ravel(), dy[:q].cpu().numpy().ravel()
    assert rel_l2(y[:q].cpu().numpy().ravel(), orc.conv_fwd(xs, ws, q, n, d, k, o, s, p)) <= TOL
    assert rel_l2(dx[:q].cpu().numpy().ravel(), orc.conv_bwd_data(dys, ws, q, n, d, k, o, s, p)) <= TOL


def test_wgrad_full_batch_vs_fp64_gemm(cct, dev):
    """conv2 b=256 backward-weight (K = 186,624 reduction terms) against an fp64 GEMM of
    the same lowered matrices computed by torch on the GPU (checker only)."""
    from paper_1504_04343_b200 import conv
    n, k, d, o, b, s, p = 27, 5, 96, 256, 256, 1, 2
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    g = torch.Generator(device=dev).manual_seed(9)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
    dw = conv.conv_bwd_weight(x, dy, desc, 1).double()
    dh = conv.lower(x, desc, 1, cct.ROWS_INTERNAL).double()                # (b m^2, k^2 d)
    dr = dy.double().permute(0, 2, 3, 1).reshape(-1, o)                     # (b m^2, o)
    ref = (dr.t() @ dh).reshape(o, k, k, d)
    err = float(torch.linalg.norm(dw - ref) / torch.linalg.norm(ref))
    assert err <= TOL, err


@pytest.mark.parametrize("layer", [("conv3", 13, 3, 256, 384, 1, 1), ("conv4", 13, 3, 384, 384, 1, 1),
                                   ("conv5", 13, 3, 384, 256, 1, 1), ("conv2", 27, 5, 96, 256, 1, 2),
                                   ("conv1", 227, 11, 3, 96, 4, 0)], ids=lambda l: l[0])
def test_caffenet_b256_vs_fp64(cct, dev, layer):
    """Full-batch (b = 256) training step of CaffeNet layers exactly as the bench runs it
    (auto lowering: implicit Type 1 incl. implicit backward-data, stream-K GEMMs for the
    ragged last wave, A-in-TMEM narrow tiles, slab-major col2im) against fp64 torch
    convolutions on the GPU (checker only)."""
    import torch.nn.functional as F
    from paper_1504_04343_b200 import conv
    _, n, k, d, o, s, p = layer
    b = 256  # every layer at the bench's batch (conv1: K = 774,400 backward-weight terms)
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    t = cct.select_lowering(desc, 3)[0]
    g = torch.Generator(device=dev).manual_seed(17)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
    cache = conv.alloc_cache(desc, t, dev)
    y = conv.conv_fwd_cached(x, w, desc, t, cache=cache)
    dx, dw = conv.conv_bwd(dy, w, desc, t, x=x, cache=cache)
    xd = x.double().permute(0, 3, 1, 2).contiguous()
    wd = w.double().permute(0, 3, 1, 2).contiguous()
    dyd = dy.double()
    ry = F.conv2d(xd, wd, stride=s, padding=p)
    rdx = torch.nn.grad.conv2d_input(xd.shape, wd, dyd, stride=s, padding=p).permute(0, 2, 3, 1)
    rdw = torch.nn.grad.conv2d_weight(xd, wd.shape, dyd, stride=s, padding=p).permute(0, 2, 3, 1)

    def rel(a, r):
        return float(torch.linalg.norm(a.double() - r) / torch.linalg.norm(r))
    assert rel(y, ry) <= TOL and rel(dx, rdx) <= TOL and rel(dw, rdw) <= TOL, (rel(y, ry), rel(dx, rdx), rel(dw, rdw))


# ------------------------------------------------------------- error behaviour
def test_misaligned_pointer_is_config_error(cct, dev):
    from paper_1504_04343_b200 import conv
    desc = cct.ConvDesc(9, 3, 4, 8, 2)
    buf = torch.zeros(2 * 9 * 9 * 4 + 1, device=dev)
    x = buf[1:].view(2, 9, 9, 4)
    w = torch.zeros(8, 3, 3, 4, device=dev)
    with pytest.raises(cct.ConfigError):
        conv.conv_fwd(x, w, desc, 1)


def test_small_workspace_is_resource_error(cct, dev):
    import ctypes as C
    desc = cct.ConvDesc(9, 3, 4, 8, 2)
    x = torch.zeros(2, 9, 9, 4, device=dev)
    w = torch.zeros(8, 3, 3, 4, device=dev)
    y = torch.zeros(2, 8, 7, 7, device=dev)
    ws = torch.zeros(16, dtype=torch.uint8, device=dev)
    st = cct.lib().cct_conv_fwd(C.byref(desc.c()), 1, C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()),
                                C.c_void_p(y.data_ptr()), C.c_void_p(ws.data_ptr()), 16, None)
    assert st == 2 and b"workspace too small" in cct.lib().cct_last_error()


def test_phase_timings(cct, dev):
    """PhaseTimings: lower / multiply / lift recorded separately."""
    import ctypes as C
    from paper_1504_04343_b200 import conv
    L = cct.lib()
    desc = cct.ConvDesc(13, 3, 64, 64, 8, 1, 1)
    x = torch.rand(8, 13, 13, 64, device=dev)
    w = torch.rand(64, 3, 3, 64, device=dev)
    P = C.c_double * 7
    ms, fl, by = P(), P(), P()
    n = (C.c_uint64 * 7)()
    L.cct_profile_read(None, None, None, None, 1)
    L.cct_profile_enable(1)
    conv.conv_fwd(x, w, desc, 2)
    L.cct_profile_enable(0)
    L.cct_profile_read(ms, fl, by, n, 1)
    assert n[0] == 1 and n[1] >= 1 and n[2] == 1  # lower, gemm, lift
    assert ms[1] > 0 and fl[1] > 0


@pytest.mark.parametrize("t", [1, 2, 3])
@pytest.mark.parametrize("layer", CAFFENET[:3], ids=[l[0] for l in CAFFENET[:3]])
def test_cached_training_step_matches_separate_passes(cct, dev, orc, layer, t):
    """cct_conv_fwd_cached + cct_conv_bwd (Dhat lowered once, dy expanded once)
    give the same tensors as the three separate entry points, bit for bit -- except the
    stand-alone passes of a strided Type 1 layer, which the cost model may run in
    space-to-depth form (a different K order: equal to fp32 rounding)."""
    from paper_1504_04343_b200 import conv
    _, n, k, d, o, s, p = layer
    b = 3
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    g = torch.Generator(device=dev).manual_seed(t)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
    cache = conv.alloc_cache(desc, t, dev)
    y = conv.conv_fwd_cached(x, w, desc, t, cache=cache)
    dx, dw = conv.conv_bwd(dy, w, desc, t, x=x, cache=cache)
    yf, dxf, dwf = conv.conv_fwd(x, w, desc, t), conv.conv_bwd_data(dy, w, desc, t), conv.conv_bwd_weight(x, dy, desc, t)
    for a_, b_ in ((y, yf), (dx, dxf), (dw, dwf)):
        if s > 1 and t == 1:
            assert float(torch.linalg.norm(a_ - b_) / torch.linalg.norm(b_)) < 1e-5
        else:
            assert torch.equal(a_, b_)
    _, dw2 = conv.conv_bwd(dy, w, desc, t, x=None if cache is not None else x, cache=cache, want_dx=False)
    assert torch.equal(dw2, dw)


@pytest.mark.parametrize("t", [1, 2, 3])
def test_batch_chunking_under_workspace_limit(cct, dev, t):
    """A small workspace limit splits the batch into chunks (SPEC batching module):
    every output agrees with the unchunked pass to fp32 rounding."""
    from paper_1504_04343_b200 import conv
    L = cct.lib()
    n, k, d, o, b, s, p = 27, 5, 32, 48, 12, 1, 2
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
    full = (conv.conv_fwd(x, w, desc, t), conv.conv_bwd_data(dy, w, desc, t), conv.conv_bwd_weight(x, dy, desc, t))
    old = L.cct_get_workspace_limit()
    try:
        L.cct_set_workspace_limit(8 << 20)
        small = cct.workspace_size(desc, t, cct.PASS_FWD)
        assert small <= (8 << 20) or t == 3
        ch = (conv.conv_fwd(x, w, desc, t), conv.conv_bwd_data(dy, w, desc, t), conv.conv_bwd_weight(x, dy, desc, t))
        cache = conv.alloc_cache(desc, t, dev)
        y2 = conv.conv_fwd_cached(x, w, desc, t, cache=cache)
        dx2, dw2 = conv.conv_bwd(dy, w, desc, t, x=x, cache=cache)
    finally:
        L.cct_set_workspace_limit(old)
    # chunks change the GEMM's N extent, hence possibly its tile width and the
    # number of TMEM sub-accumulators: equal to fp32 rounding, not bit for bit
    def close(a, ref):
        return float(torch.linalg.norm(a - ref) / torch.linalg.norm(ref)) < 1e-5
    assert close(ch[0], full[0]) and close(ch[1], full[1]) and close(y2, full[0])
    assert close(dx2, full[1])
    for dwc in (ch[2], dw2):
        assert close(dwc, full[2])


@pytest.mark.parametrize("layer", [("conv2s", 27, 5, 96, 64, 1, 2), ("conv3", 13, 3, 256, 384, 1, 1),
                                   ("d16", 11, 3, 16, 40, 1, 1), ("d48", 12, 5, 48, 64, 1, 2)],
                         ids=lambda l: l[0])
def test_implicit_lowering_matches_materialised(cct, dev, orc, layer):
    """Implicit Type 1 (TMA im2col operands, no Dhat in HBM) == materialised Type 1:
    forward bit for bit (same K order, same GEMM); both match the oracle."""
    from paper_1504_04343_b200 import conv
    L = cct.lib()
    _, n, k, d, o, s, p = layer
    b = 3
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x_np, w_np = orc.random_problem(77, b, n, d, k, o)
    dy_np = orc.uniform(78, b * o * desc.m * desc.m)
    x = T(x_np, dev, b, n, n, d)
    w = T(w_np, dev, o, k, k, d)
    dy = T(dy_np, dev, b, o, desc.m, desc.m)
    old = L.cct_get_implicit_lowering()
    try:
        L.cct_set_implicit_lowering(1)
        assert cct.lowered_cache_size(desc, 1) == 0
        yi, dwi = conv.conv_fwd(x, w, desc, 1), conv.conv_bwd_weight(x, dy, desc, 1)
        cache = conv.alloc_cache(desc, 1, dev)
        yc = conv.conv_fwd_cached(x, w, desc, 1, cache=cache)
        _, dwc = conv.conv_bwd(dy, w, desc, 1, x=x, cache=cache)
        L.cct_set_implicit_lowering(0)
        ym, dwm = conv.conv_fwd(x, w, desc, 1), conv.conv_bwd_weight(x, dy, desc, 1)
    finally:
        L.cct_set_implicit_lowering(old)
    assert torch.equal(yi, ym) and torch.equal(yc, ym)
    assert torch.equal(dwc, dwi)
    # materialised bwd-weight of a narrow bank (o < 128) runs in the swapped
    # orientation (dW = dRhat^T Dhat): same products, different rounding
    assert float(torch.linalg.norm(dwi - dwm) / torch.linalg.norm(dwm)) < 2e-5
    assert rel_l2(yi.cpu().numpy().ravel(), orc.conv_fwd(x_np, w_np, b, n, d, k, o, s, p)) <= TOL
    assert rel_l2(dwi.cpu().numpy().ravel(), orc.conv_bwd_weight(x_np, dy_np, b, n, d, k, o, s, p)) <= TOL


@pytest.mark.parametrize("layer", [("conv2s", 27, 5, 96, 64, 1, 2), ("conv3", 13, 3, 256, 384, 1, 1),
                                   ("pad0_d20", 12, 3, 20, 32, 1, 0), ("padk-1", 10, 3, 8, 16, 1, 2),
                                   ("k1", 9, 1, 16, 16, 1, 0), ("d3", 11, 4, 3, 16, 1, 1),
                                   ("longK", 9, 5, 8, 176, 1, 2), ("stride2", 15, 3, 32, 48, 2, 1),
                                   ("d48", 12, 5, 48, 64, 1, 2)],
                         ids=lambda l: l[0])
def test_implicit_dgrad(cct, dev, orc, layer):
    """Implicit stride-1 backward-data (dy -> NHWC, forward convolution with the rotated
    kernel bank straight into dx; implicit mode 2 forces it) matches the oracle and the
    materialised path; backward-weight with the NHWC dy as B operand too.  Stride 2 runs
    as the stride-1 backward of its space-to-depth form."""
    from paper_1504_04343_b200 import conv
    L = cct.lib()
    _, n, k, d, o, s, p = layer
    b = 3
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x_np, w_np = orc.random_problem(91, b, n, d, k, o)
    dy_np = orc.uniform(92, b * o * desc.m * desc.m)
    x = T(x_np, dev, b, n, n, d)
    w = T(w_np, dev, o, k, k, d)
    dy = T(dy_np, dev, b, o, desc.m, desc.m)
    old = L.cct_get_implicit_lowering()
    try:
        L.cct_set_implicit_lowering(2)
        dxi, dwi = conv.conv_bwd_data(dy, w, desc, 1), conv.conv_bwd_weight(x, dy, desc, 1)
        cache = conv.alloc_cache(desc, 1, dev)
        conv.conv_fwd_cached(x, w, desc, 1, cache=cache)
        dxc, dwc = conv.conv_bwd(dy, w, desc, 1, x=x, cache=cache)
        L.cct_set_implicit_lowering(0)
        dxm, dwm = conv.conv_bwd_data(dy, w, desc, 1), conv.conv_bwd_weight(x, dy, desc, 1)
    finally:
        L.cct_set_implicit_lowering(old)
    assert torch.equal(dxc, dxi) and torch.equal(dwc, dwi)
    ref_dx = orc.conv_bwd_data(dy_np, w_np, b, n, d, k, o, s, p)
    ref_dw = orc.conv_bwd_weight(x_np, dy_np, b, n, d, k, o, s, p)
    for got in (dxi, dxm):
        assert rel_l2(got.cpu().numpy().ravel(), ref_dx) <= TOL
    for got in (dwi, dwm):
        assert rel_l2(got.cpu().numpy().ravel(), ref_dw) <= TOL
    assert float(torch.linalg.norm(dxi - dxm) / torch.linalg.norm(dxm)) < 5e-5  # two ~1e-5 paths


S2D_LAYERS = [("conv1", 227, 11, 3, 96, 4, 0), ("conv1s", 35, 11, 3, 96, 4, 0), ("s2p1", 15, 3, 32, 40, 2, 1),
              ("ragged", 14, 4, 64, 48, 3, 2), ("s2d16", 23, 5, 4, 16, 2, 1), ("k_lt_s", 20, 3, 4, 8, 4, 1),
              ("pad_gt", 17, 6, 16, 32, 2, 4), ("no_s2d", 19, 7, 12, 32, 3, 3)]


@pytest.mark.parametrize("layer", S2D_LAYERS, ids=lambda l: l[0])
def test_space_to_depth(cct, dev, orc, layer):
    """Strided Type 1 layers run as the stride-1 convolution of the space-to-depth
    blocked input (k' = ceil(k/s) taps of depth s^2 d; s2d.cuh): forward, backward-data,
    backward-weight and the cached training step against the oracle, and against the
    materialised path.  s^2 d % 16 != 0 (no_s2d) stays materialised.  Implicit mode 2
    forces the blocked form; by default the cost model picks it per pass (prefer_s2d)."""
    from paper_1504_04343_b200 import conv
    L = cct.lib()
    _, n, k, d, o, s, p = layer
    b = 2
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x_np, w_np = orc.random_problem(31, b, n, d, k, o)
    dy_np = orc.uniform(32, b * o * desc.m * desc.m)
    x = T(x_np, dev, b, n, n, d)
    w = T(w_np, dev, o, k, k, d)
    dy = T(dy_np, dev, b, o, desc.m, desc.m)
    blocked = (s * s * d) % 16 == 0
    old = L.cct_get_implicit_lowering()
    gather_off = cct.tuning(gather=0)  # the fused gather form would take conv1-class layers
    gather_off.__enter__()
    try:
        L.cct_set_implicit_lowering(2)  # forces the blocked form (else the cost model picks per pass)
        ks, ns = -(-k // s), desc.m + -(-k // s) - 1
        assert cct.lowered_cache_size(desc, 1) == (b * ns * ns * s * s * d * 4 if blocked else
                                                    b * desc.m * desc.m * ((k * k * d + 3) // 4 * 4) * 4)
        y, dx, dw = (conv.conv_fwd(x, w, desc, 1), conv.conv_bwd_data(dy, w, desc, 1),
                     conv.conv_bwd_weight(x, dy, desc, 1))
        cache = conv.alloc_cache(desc, 1, dev)
        yc = conv.conv_fwd_cached(x, w, desc, 1, cache=cache)
        dxc, dwc = conv.conv_bwd(dy, w, desc, 1, x=x, cache=cache)
        L.cct_set_implicit_lowering(0)
        ym, dxm, dwm = (conv.conv_fwd(x, w, desc, 1), conv.conv_bwd_data(dy, w, desc, 1),
                        conv.conv_bwd_weight(x, dy, desc, 1))
    finally:
        L.cct_set_implicit_lowering(old)
        gather_off.__exit__(None, None, None)
    assert torch.equal(yc, y) and torch.equal(dxc, dx) and torch.equal(dwc, dw)
    refs = (orc.conv_fwd(x_np, w_np, b, n, d, k, o, s, p), orc.conv_bwd_data(dy_np, w_np, b, n, d, k, o, s, p),
            orc.conv_bwd_weight(x_np, dy_np, b, n, d, k, o, s, p))
    for got, ref in zip((y, dx, dw), refs):
        assert rel_l2(got.cpu().numpy().ravel(), ref) <= TOL
    for got, ref in zip((ym, dxm, dwm), refs):
        assert rel_l2(got.cpu().numpy().ravel(), ref) <= TOL
    if not blocked:
        assert torch.equal(y, ym) and torch.equal(dx, dxm)


@pytest.mark.parametrize("t", [2, 3])
@pytest.mark.parametrize("layer", [CAFFENET[1], CAFFENET[2], ("d3", 11, 4, 3, 16, 1, 1)], ids=lambda l: l[0])
def test_fused_types_2_3(cct, dev, orc, layer, t):
    """CCT_TUNE_FUSED_T23: a Type 2 / 3 request on a layer with the implicit form (d % 16 == 0)
    runs fused -- the k^2 (Type 3) or k (Type 2) shifted products accumulated in TMEM, one
    im2col box per tap, no Rhat and no lift pass: bit for bit the implicit Type 1 result, and
    within the oracle tolerance.  Without the implicit form (d = 3) the request stays the
    materialised Type 2 / 3 path (lift phase recorded)."""
    import ctypes as C
    from paper_1504_04343_b200 import conv
    L = cct.lib()
    _, n, k, d, o, s, p = layer
    b = 4
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    m = desc.m
    x_np, w_np = orc.random_problem(91, b, n, d, k, o)
    dy_np = orc.uniform(92, b * o * m * m)
    x, w, dy = T(x_np, dev, b, n, n, d), T(w_np, dev, o, k, k, d), T(dy_np, dev, b, o, m, m)
    P = C.c_double * 7
    ms, fl, by = P(), P(), P()
    cnt = (C.c_uint64 * 7)()
    with cct.tuning(fused_t23=1):
        L.cct_profile_read(None, None, None, None, 1)
        L.cct_profile_enable(1)
        yf = conv.conv_fwd(x, w, desc, t)
        dxf = conv.conv_bwd_data(dy, w, desc, t)
        dwf = conv.conv_bwd_weight(x, dy, desc, t)
        torch.cuda.synchronize()
        L.cct_profile_enable(0)
        L.cct_profile_read(ms, fl, by, cnt, 1)
    fused = d % 16 == 0
    assert (cnt[2] == 0) == fused  # lift phase only on the materialised Type 2 / 3 path
    y1, dx1, dw1 = (conv.conv_fwd(x, w, desc, 1), conv.conv_bwd_data(dy, w, desc, 1),
                    conv.conv_bwd_weight(x, dy, desc, 1))
    if fused:
        assert torch.equal(yf, y1) and torch.equal(dxf, dx1) and torch.equal(dwf, dw1)
    refs = (orc.conv_fwd(x_np, w_np, b, n, d, k, o, s, p), orc.conv_bwd_data(dy_np, w_np, b, n, d, k, o, s, p),
            orc.conv_bwd_weight(x_np, dy_np, b, n, d, k, o, s, p))
    for got, ref in zip((yf, dxf, dwf), refs):
        assert rel_l2(got.cpu().numpy().ravel(), ref) <= TOL


SWAP_SCRIPT = r"""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "oracle"))
import paper_1504_04343_b200 as cct
from paper_1504_04343_b200 import conv
from oracle_py import Oracle, rel_l2, grouped_fwd
cct.set_tuning("fwd_swap", 1)
orc = Oracle(); dev = torch.device("cuda")
out = {}
for name, (n, k, d, o, s, p, G, mode) in {"conv1": (227, 11, 3, 96, 4, 0, 1, 1), "conv1_s2d": (227, 11, 3, 96, 4, 0, 1, 2),
                                           "implicit": (13, 3, 32, 48, 1, 1, 1, 1),
                                           "grouped_bias": (13, 3, 64, 64, 1, 1, 2, 1)}.items():
    b = 2
    cct.lib().cct_set_implicit_lowering(mode)
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x = orc.uniform(5, b * n * n * d); w = orc.uniform(6, o * k * k * (d // G)); bias = orc.uniform(7, o)
    xt = torch.from_numpy(x).to(dev).view(b, n, n, d); wt = torch.from_numpy(w).to(dev).view(o, k, k, d // G)
    bt = torch.from_numpy(bias).to(dev)
    y = conv.conv_fwd_ex(xt, wt, desc, 1, groups=G, bias=bt, relu=True)
    ref = grouped_fwd(orc, x, w, b, n, d, k, o, s, p, G, bias, relu=True)
    out[name] = rel_l2(y.cpu().numpy().ravel(), ref.ravel())
print(json.dumps(out))
"""


def test_swapped_forward_opt_in(cct, dev):
    """CCT_TUNE_FWD_SWAP = 1: narrow banks (o < 128) run the forward swapped -- channels on the
    128-row side, pixels 256 wide (materialised Dhat or TMA-im2col B operand), NCHW rows
    through the transposing epilogue with a per-row bias + ReLU.  Off by default (slower
    on conv1); kept correct here."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, ROOT=root)
    r = subprocess.run([sys.executable, "-c", SWAP_SCRIPT], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(errs) == 4 and max(errs.values()) <= TOL, errs


@pytest.mark.parametrize("M,N,K", [(100, 384, 40), (300, 384, 3000), (5000, 768, 1000), (40000, 384, 3456),
                                   (700, 1152, 17)])
def test_composite_384_tile(cct, dev, M, N, K):
    """N a multiple of 384 with K-major operands runs the 256 + 128 composite tile
    (single-buffered, 64-row B boxes), CTA pairs or not, stream-K when ragged: against
    an fp64 GEMM (checker only)."""
    import ctypes as C
    L = cct.lib()
    L.cct_debug_gemm.argtypes = [C.c_int64] * 3 + [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_int,
                                                   C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p]
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    ld = (K + 3) // 4 * 4
    A = torch.rand((M, ld), generator=g, device=dev) * 2 - 1
    B = torch.rand((N, ld), generator=g, device=dev) * 2 - 1
    Cm = torch.empty((M, N), device=dev)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = L.cct_debug_gemm(M, N, K, A.data_ptr(), ld, 0, B.data_ptr(), ld, 0, Cm.data_ptr(), N, 1, 3, 0, st)
    assert rc == 0, L.cct_last_error()
    ref = A[:, :K].double() @ B[:, :K].double().t()
    err = float(torch.linalg.norm(Cm.double() - ref) / torch.linalg.norm(ref))
    assert err <= TOL, err


@pytest.mark.parametrize("split_k", [7, 96, 300])
def test_split_k_with_empty_trailing_splits(cct, dev, split_k):
    """Requested split counts the kernel trims (no empty split) reduce over exactly the
    slices that were written: regression for a stale slice summed into the result."""
    from paper_1504_04343_b200 import conv
    g = torch.Generator(device=dev).manual_seed(split_k)
    a = torch.rand((96, 6050 * 16), generator=g, device=dev) * 2 - 1
    b = torch.rand((6050 * 16, 40), generator=g, device=dev) * 2 - 1
    ws = conv.Workspace(dev)
    ws.get(512 << 20).fill_(255)  # stale garbage (NaN bytes) in the scratch
    c = conv.multiply(a, b, split_k=split_k, ws=ws)
    ref = a.double() @ b.double()
    assert float(torch.linalg.norm(c.double() - ref) / torch.linalg.norm(ref)) <= TOL
