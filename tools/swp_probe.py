"""Swapped narrow-bank forward shapes: transposing epilogue vs output row stride (diagnostic)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, "tools")
from gemm_bench import L  # noqa: E402

M, N, K = 96, 774400, int(sys.argv[1]) if len(sys.argv) > 1 else 368
LDA, LDB = (K + 3) // 4 * 4, (K + 3) // 4 * 4
dev = torch.device("cuda")
A = torch.rand((M, LDA), device=dev)
B = torch.rand((N, LDB), device=dev)
Cm = torch.empty((M * N + 8,), device=dev)
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for ldm, tag in ((3025, f"K={K} rows 12 KB apart (overlapping, timing only)"),):
    for passes in (3, 3 | 0x100):
        def go():
            rc = L.cct_debug_gemm(M, N, K, A.data_ptr(), LDA, 0, B.data_ptr(), LDB, 0, Cm.data_ptr(), ldm, 1, passes, 256, st)
            assert rc == 0, L.cct_last_error()
        for _ in range(2):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            go()
        e1.record()
        torch.cuda.synchronize()
        print(f"{tag:45s} {'TRO' if passes & 0x100 else 'reg'}: {e0.elapsed_time(e1) / 5 * 1e3:8.1f} us", flush=True)
