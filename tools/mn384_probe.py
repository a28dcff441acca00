"""Diagnostic: composite 384 tile with an MN-major B (debug GEMM vs fp64)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, "tools")
from gemm_bench import L  # noqa: E402

dev = torch.device("cuda")
for (M, N, K, amaj, bmaj) in ((96, 384, 2000, 0, 1), (96, 363, 2000, 0, 1), (300, 384, 2000, 0, 1),
                              (96, 384, 2000, 1, 1), (96, 256, 2000, 0, 1), (96, 192, 2000, 0, 1)):
    g = torch.Generator(device=dev).manual_seed(1)
    ldn = (N + 3) // 4 * 4
    A = torch.rand((K, M) if amaj else (M, K), generator=g, device=dev) * 2 - 1
    B = torch.rand((K, ldn) if bmaj else (N, K), generator=g, device=dev) * 2 - 1
    Cm = torch.zeros((M, N), device=dev)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = L.cct_debug_gemm(M, N, K, A.data_ptr(), A.shape[1], amaj, B.data_ptr(), B.shape[1], bmaj, Cm.data_ptr(),
                          N, 1, 3, 0, st)
    torch.cuda.synchronize()
    Ad = A.double().t() if amaj else A.double()
    Bd = B[:, :N].double() if bmaj else B.double().t()
    ref = Ad @ Bd
    err = float(torch.linalg.norm(Cm.double() - ref) / torch.linalg.norm(ref))
    colerr = ((Cm.double() - ref).abs().amax(0) / ref.abs().amax()).cpu()
    bad = (colerr > 1e-3).nonzero().ravel().tolist()
    print(f"M={M} N={N} K={K} A={'MN' if amaj else 'K'} B={'MN' if bmaj else 'K'} rc={rc} rel={err:.2e} bad cols {bad[:8]}..{bad[-4:] if bad else ''} n={len(bad)}", flush=True)
