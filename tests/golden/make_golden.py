"""Generate golden vectors from the REFERENCE's own code (oracle/_ref/libcctref.so:
/root/reference/proj/src/{tensor,gemm}.cpp compiled unmodified + oracle/ref_shim.cpp).

    make -C oracle && python tests/golden/make_golden.py

Each case stores the reference-generated inputs (DataBatch::random then
KernelBank::random from std::mt19937_64(seed), tensor.cpp:39-64; dy from
Mat::random, gemm.cpp:82-87) and the reference outputs:
  * y  = direct_convolve_batch on the zero-embedded input, subsampled
  * dx = direct_convolve on the dilated dy with rotated kernels
  * dw = direct_convolve of the batch-as-depth data with dilated dy
  * y_direct (stride 1, pad 0 cases only) = direct_convolve_batch itself.
GEMM cases store multiply_reference (gemm.cpp:124) and multiply with 3 threads.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle_py import Reference  # noqa: E402

# (name, n, k, d, o, b, stride, pad)
CASES = [
    ("c1_s1p0", 9, 3, 4, 8, 2, 1, 0),
    ("c2_s1p1", 11, 3, 8, 16, 2, 1, 1),
    ("c3_s2p2", 13, 5, 4, 12, 2, 2, 2),
    ("c4_conv1like", 23, 11, 3, 8, 2, 4, 0),
    ("c5_conv2like", 15, 5, 16, 32, 2, 1, 2),
    ("c6_conv3like", 13, 3, 32, 48, 1, 1, 1),
    ("c7_ragged", 10, 4, 5, 6, 3, 3, 1),
]
GEMMS = [("g1", 16, 24, 8), ("g2", 33, 65, 17), ("g3", 64, 300, 96)]


def main():
    ref = Reference()
    for i, (name, n, k, d, o, b, s, p) in enumerate(CASES):
        seed = 1234 + i
        x, w = ref.random_problem(seed, b, n, d, k, o)
        m = (n + 2 * p - k) // s + 1
        dy = ref.random_mat(seed + 1000, 1, b * o * m * m).ravel()
        out = dict(x=x, w=w, dy=dy, shape=np.array([n, k, d, o, b, s, p], np.int64), seed=np.array([seed]),
                   y=ref.conv_fwd(x, w, b, n, d, k, o, s, p),
                   dx=ref.conv_bwd_data(dy, w, b, n, d, k, o, s, p),
                   dw=ref.conv_bwd_weight(x, dy, b, n, d, k, o, s, p))
        if s == 1 and p == 0:
            out["y_direct"] = ref.direct_convolve_batch(x, b, n, d, w, k, o)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    for j, (name, M, K, N) in enumerate(GEMMS):
        A = ref.random_mat(99 + j, M, K)
        B = ref.random_mat(199 + j, K, N)
        import ctypes as C  # noqa: F401
        Cr = np.empty((M, N), np.float32)
        ref.lib.ref_multiply_reference(A, B, Cr, M, K, N)
        Ct = ref.multiply(A, B, threads=3)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), A=A, B=B, C=Cr, C_threads3=Ct)
    # the reference RNG stream (rng(1234): DataBatch::random(1, 16, 16) first)
    x, _ = ref.random_problem(1234, 1, 16, 16, 1, 1)
    np.save(os.path.join(HERE, "rng_seed1234_first4096.npy"), x[:4096])
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
