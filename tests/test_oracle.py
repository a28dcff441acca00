"""CPU: pin the oracle (oracle/cct_oracle.c) before trusting it.

(1) SPEC known-answer examples.
(2) Golden vectors produced by the reference's own tensor.cpp / gemm.cpp
    (tests/golden/make_golden.py) -- bit-exact for direct convolution and GEMM.
(3) Live comparison with the reference build when oracle/_ref is present.
(4) Properties: linearity, kernel additivity, the lower/multiply/lift diagram,
    and the adjoint identity that ties fwd, bwd-data and bwd-weight together.
"""
import glob
import os

import numpy as np
import pytest

from oracle_py import rel_l2

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CONV_CASES = sorted(glob.glob(os.path.join(GOLD, "c*.npz")))
GEMM_CASES = sorted(glob.glob(os.path.join(GOLD, "g*.npz")))


# ---------------------------------------------------------------- SPEC KATs
def test_kat_direct_convolve_fixture(orc):
    # D = [[1,2,3],[4,5,6],[7,8,9]], K = [[1,0],[0,1]] -> [[6,8],[12,14]]
    x = np.arange(1, 10, dtype=np.float32)
    w = np.array([1, 0, 0, 1], np.float32)
    y = orc.direct_convolve_batch(x, 1, 3, 1, w, 2, 1)
    assert y.tolist() == [6, 8, 12, 14]


def test_kat_identity_and_zero_kernel(orc):
    x = orc.uniform(5, 4 * 4)
    assert np.array_equal(orc.direct_convolve_batch(x, 1, 4, 1, np.ones(1, np.float32), 1, 1), x)
    assert not orc.direct_convolve_batch(x, 1, 4, 1, np.zeros(1, np.float32), 1, 1).any()


def test_kat_batch_is_independent_calls(orc):
    # SPEC.md:68 / tensor.cpp:108-118: b=3, o=2 equals 6 independent convolutions
    b, n, d, k, o = 3, 6, 2, 3, 2
    x, w = orc.random_problem(11, b, n, d, k, o)
    y = orc.direct_convolve_batch(x, b, n, d, w, k, o).reshape(b, o, -1)
    for q in range(b):
        for j in range(o):
            single = orc.direct_convolve_batch(x[q * n * n * d:(q + 1) * n * n * d], 1, n, d,
                                               w[j * k * k * d:(j + 1) * k * k * d], k, 1)
            assert np.array_equal(y[q, j], single)


def test_kat_multiply(orc):
    # SPEC.md:185
    c = orc.multiply(np.array([[1, 2], [3, 4]], np.float32), np.array([[5, 6], [7, 8]], np.float32))
    assert c.tolist() == [[19, 22], [43, 50]]
    b = orc.uniform(3, 12).reshape(3, 4)
    assert np.array_equal(orc.multiply(np.eye(3, dtype=np.float32), b), b)


@pytest.mark.parametrize("args,shape", [
    ((1, 1, 3, 2, 3, 1), (1, 18, 1)),     # n = k -> 1 x k^2 d
    ((1, 1, 5, 2, 3, 1), (9, 18, 1)),     # T1 n=5,k=3,d=2,o=1 -> 9x18, 18x1
    ((3, 2, 5, 2, 3, 4), (50, 2, 36)),    # T3 n=5,k=3,d=2,o=4,b=2 -> 50x2, 2x36
])
def test_kat_lowered_shapes(orc, args, shape):
    t, b, n, d, k, o = args
    assert orc.lowered_shape(t, b, n, d, k, o) == shape


def test_kat_lift_type3_fixture(orc):
    # Type 3 on the 3x3 / 2x2 fixture -> [[6,8],[12,14]]
    x = np.arange(1, 10, dtype=np.float32)
    w = np.array([1, 0, 0, 1], np.float32)
    for t in (1, 2, 3):
        assert orc.convolve_lowered(t, x, w, 1, 3, 1, 2, 1).tolist() == [6, 8, 12, 14]
    rows, cols, kc = orc.lowered_shape(3, 1, 3, 1, 2, 1)
    assert not orc.lift(3, np.zeros((rows, kc), np.float32), 1, 3, 1, 2, 1).any()


def test_kat_type1_lift_is_reshape(orc):
    # Type 1, o = b = 1: R[r, c] = Rhat[c m + r]
    n, k = 5, 3
    m = n - k + 1
    rh = np.arange(m * m, dtype=np.float32).reshape(m * m, 1)
    y = orc.lift(1, rh, 1, n, 1, k, 1).reshape(m, m)
    for r in range(m):
        for c in range(m):
            assert y[r, c] == rh[c * m + r, 0]


def test_kat_estimate(orc):
    # n=5,k=3,d=2,o=1,b=1,T1 -> 162 lowered elements, 324 flops
    low, fl, lift = orc.estimate(1, 1, 5, 2, 3, 1)
    assert (low, fl, lift) == (162, 324, 0)
    # k = 1 -> identical counts for all types
    assert len({orc.estimate(t, 2, 7, 3, 1, 4) for t in (1, 2, 3)}) == 1
    # T1 / T3 flop ratio = (m/n)^2
    n, k = 13, 3
    m = n - k + 1
    r = orc.estimate(1, 4, n, 8, k, 8)[1] / orc.estimate(3, 4, n, 8, k, 8)[1]
    assert abs(r - (m / n) ** 2) < 1e-12
    # lift adds per output are 0 / k-1 / k^2-1
    for t, per in ((1, 0), (2, k - 1), (3, k * k - 1)):
        assert orc.estimate(t, 2, n, 4, k, 5)[2] == 2 * m * m * 5 * per


# ----------------------------------------------------------- golden vectors
def _case(path):
    z = np.load(path)
    n, k, d, o, b, s, p = (int(v) for v in z["shape"])
    return z, (n, k, d, o, b, s, p)


@pytest.mark.parametrize("path", CONV_CASES, ids=[os.path.basename(p)[:-4] for p in CONV_CASES])
def test_oracle_matches_reference_golden_bit_exact(orc, path):
    z, (n, k, d, o, b, s, p) = _case(path)
    x2, w2 = orc.random_problem(int(z["seed"][0]), b, n, d, k, o)
    assert np.array_equal(x2, z["x"]) and np.array_equal(w2, z["w"]), "RNG stream differs from the reference"
    assert np.array_equal(orc.conv_fwd(z["x"], z["w"], b, n, d, k, o, s, p), z["y"])
    assert np.array_equal(orc.conv_bwd_data(z["dy"], z["w"], b, n, d, k, o, s, p), z["dx"])
    assert np.array_equal(orc.conv_bwd_weight(z["x"], z["dy"], b, n, d, k, o, s, p), z["dw"])
    if "y_direct" in z:
        assert np.array_equal(orc.direct_convolve_batch(z["x"], b, n, d, z["w"], k, o), z["y_direct"])


@pytest.mark.parametrize("path", CONV_CASES, ids=[os.path.basename(p)[:-4] for p in CONV_CASES])
@pytest.mark.parametrize("t", [1, 2, 3])
def test_lowered_restatement_matches_golden(orc, path, t):
    """Appendix A lowered paths (fwd/dgrad/wgrad, every type) vs the reference outputs."""
    z, (n, k, d, o, b, s, p) = _case(path)
    assert rel_l2(orc.lowered("fwd", t, z["x"], z["w"], b, n, d, k, o, s, p), z["y"]) < 1e-6
    assert rel_l2(orc.lowered("bwd_data", t, z["dy"], z["w"], b, n, d, k, o, s, p), z["dx"]) < 1e-6
    assert rel_l2(orc.lowered("bwd_weight", t, z["x"], z["dy"], b, n, d, k, o, s, p), z["dw"]) < 1e-6


@pytest.mark.parametrize("path", GEMM_CASES, ids=[os.path.basename(p)[:-4] for p in GEMM_CASES])
def test_oracle_gemm_matches_reference_golden(orc, path):
    z = np.load(path)
    assert np.array_equal(orc.multiply(z["A"], z["B"]), z["C"])
    assert np.array_equal(z["C_threads3"], z["C"])  # thread-count invariance


def test_rng_matches_reference_stream(orc):
    gold = np.load(os.path.join(GOLD, "rng_seed1234_first4096.npy"))
    assert np.array_equal(orc.uniform(1234, gold.size), gold)


# ----------------------------------------------------------- live reference
def test_live_reference_adapters(orc, ref):
    for (n, k, d, o, b, s, p) in [(12, 3, 3, 5, 2, 2, 1), (9, 4, 2, 3, 1, 1, 2)]:
        x, w = ref.random_problem(77, b, n, d, k, o)
        m = (n + 2 * p - k) // s + 1
        dy = orc.uniform(78, b * o * m * m)
        assert np.array_equal(orc.conv_fwd(x, w, b, n, d, k, o, s, p), ref.conv_fwd(x, w, b, n, d, k, o, s, p))
        assert np.array_equal(orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p),
                              ref.conv_bwd_data(dy, w, b, n, d, k, o, s, p))
        assert np.array_equal(orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p),
                              ref.conv_bwd_weight(x, dy, b, n, d, k, o, s, p))


def test_live_reference_multiply_thread_invariance(ref):
    a = ref.random_mat(1, 64, 64)
    b = ref.random_mat(2, 64, 64)
    c1 = ref.multiply(a, b, 1)
    for t in (2, 4, 8):
        assert np.array_equal(ref.multiply(a, b, t), c1)
    with pytest.raises(ValueError):
        ref.multiply(a, b, 0)  # config_error: threads out of [1, 256] (gemm.cpp:26-30)


# ----------------------------------------------------------------- properties
def test_linearity_and_additivity(orc):
    # SPEC.md:71-72
    b, n, d, k, o = 2, 8, 3, 3, 2
    x, w = orc.random_problem(5, b, n, d, k, o)
    w2 = orc.uniform(6, w.size)
    y = orc.direct_convolve_batch(x, b, n, d, w, k, o)
    assert np.array_equal(orc.direct_convolve_batch(2 * x, b, n, d, w, k, o), 2 * y)
    lhs = orc.direct_convolve_batch(x, b, n, d, w + w2, k, o)
    rhs = y + orc.direct_convolve_batch(x, b, n, d, w2, k, o)
    assert rel_l2(lhs, rhs) < 1e-6


@pytest.mark.parametrize("t", [1, 2, 3])
def test_commutative_diagram(orc, t):
    # lift(multiply(lower)) == direct_convolve_batch
    b, n, d, k, o = 2, 9, 4, 3, 5
    x, w = orc.random_problem(9, b, n, d, k, o)
    assert rel_l2(orc.convolve_lowered(t, x, w, b, n, d, k, o), orc.direct_convolve_batch(x, b, n, d, w, k, o)) < 1e-6


def test_adjoint_identity(orc):
    # <conv(x,w), dy> = <x, dgrad(dy,w)> = <w, wgrad(x,dy)>
    b, n, d, k, o, s, p = 2, 11, 3, 3, 4, 2, 1
    x, w = orc.random_problem(21, b, n, d, k, o)
    m = (n + 2 * p - k) // s + 1
    dy = orc.uniform(22, b * o * m * m)
    a = float(np.dot(orc.conv_fwd(x, w, b, n, d, k, o, s, p).astype(np.float64), dy))
    bb = float(np.dot(x.astype(np.float64), orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p)))
    c = float(np.dot(w.astype(np.float64), orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p)))
    assert abs(a - bb) < 1e-5 * abs(a) and abs(a - c) < 1e-5 * abs(a)


def test_internal_lowering_element_counts(orc):
    # each D element appears at most k^2 / k / 1 times in Dhat
    b, n, d, k = 1, 7, 2, 3
    x = np.arange(1, b * n * n * d + 1, dtype=np.float32)
    for t, cap in ((1, k * k), (2, k), (3, 1)):
        dh = orc.lower_internal(t, x, b, n, d, k, 1, 0)
        counts = np.bincount(dh.ravel().astype(np.int64), minlength=x.size + 1)[1:]
        assert counts.max() <= cap and counts.min() >= 1
