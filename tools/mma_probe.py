"""Per-k-block cost of the tcgen05 GEMM vs tile width, passes and CTA-pair mode, with the
A operand L2-resident (M*K*4 = 64 MB) so HBM does not bound it.
Run with CCT_GEMM_CG=1 or 2 to force the CTA mode.  Prints ns per (tile, k-block) per SM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_bench import run  # noqa: E402

M, K = 16384, 1024
for N in (32, 64, 96, 128, 192, 256):
    for passes in (1, 3):
        ms, tf = run(M, N, K, 0, 0, passes, 0, 20, cmaj=1)
        cg = int(os.environ.get("CCT_GEMM_CG", "2"))
        tiles = (M // 128) * ((N + N - 1) // N)
        kb = K // 16
        per = ms * 1e6 / (tiles * kb / 148.0)
        print(f"CG={cg} N={N:4d} passes={passes}: {ms*1e3:8.1f} us  {tf:6.1f} TF/s  {per:6.1f} ns per tile-kblock per SM",
              flush=True)
