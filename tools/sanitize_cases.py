"""Small problems that reach every GEMM template instance the library dispatches,
for compute-sanitizer (memcheck / racecheck / synccheck) runs:

    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Each case is checked against an fp64 torch reference (rel-L2 <= 1e-4), so a run
under the sanitizer is also a correctness run.  Sizes are tiny (the sanitizers
slow kernels down by 10-1000x); stream-K and the 384-wide tiles need a few
hundred tiles, so those cases use K = 32.  Prints one line per case and
"SANITIZE_CASES_OK <n>" at the end.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402

dev = torch.device("cuda")
TOL = 1e-4


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-300))


def ref_conv(x, w, s, p):
    # x (b,n,n,d) NHWC, w (o,k,k,d) -> y (b,o,m,m)
    return torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(0, 3, 1, 2), stride=s,
                                      padding=p)


def conv_case(name, n, k, d, o, b, s, p, types=(1, 2, 3), **tune):
    g = torch.Generator(device=dev).manual_seed(n * 1000 + d + o)
    x = torch.rand((b, n, n, d), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    dy = torch.rand((b, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
    xr = x.double().permute(0, 3, 1, 2).requires_grad_(True)
    wr = w.double().permute(0, 3, 1, 2).requires_grad_(True)
    yr = torch.nn.functional.conv2d(xr, wr, stride=s, padding=p)
    yr.backward(dy.double())
    ry, rdx, rdw = yr.detach(), xr.grad.permute(0, 2, 3, 1), wr.grad.permute(0, 2, 3, 1)
    with cct.tuning(**tune):
        for t in types:
            y = conv.conv_fwd(x, w, desc, t)
            dx = conv.conv_bwd_data(dy, w, desc, t)
            dw = conv.conv_bwd_weight(x, dy, desc, t)
            # the combined backward (one call: shared expand; fused small-channel layers fork the
            # backward-weight onto the side stream, CCT_TUNE_OVERLAP)
            dx2, dw2 = conv.conv_bwd(dy, w, desc, t, x=x)
            torch.cuda.synchronize()
            e = (rel(y, ry), rel(dx, rdx), rel(dw, rdw), rel(dx2, rdx), rel(dw2, rdw))
            print(f"{name} T{t} {tune}: fwd {e[0]:.1e} dgrad {e[1]:.1e} wgrad {e[2]:.1e} "
                  f"combined {e[3]:.1e} / {e[4]:.1e}", flush=True)
            assert max(e) <= TOL, (name, t, e)


def gemm_case(M, N, K, a_mn, b_mn, bn):
    import ctypes as C
    L = cct.lib()
    L.cct_debug_gemm.argtypes = [C.c_int64] * 3 + [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_int,
                                                   C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p]
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    A = torch.rand((K, M) if a_mn else (M, K), generator=g, device=dev) * 2 - 1
    B = torch.rand((K, N) if b_mn else (N, K), generator=g, device=dev) * 2 - 1
    Cm = torch.zeros((M, N), device=dev)
    st = torch.cuda.current_stream().cuda_stream
    cct.check(L.cct_debug_gemm(M, N, K, A.data_ptr(), A.shape[1], a_mn, B.data_ptr(), B.shape[1], b_mn,
                               Cm.data_ptr(), N, 1, 3, bn, st))
    torch.cuda.synchronize()
    Ad = A.double().t() if a_mn else A.double()
    Bd = B.double() if b_mn else B.double().t()
    e = rel(Cm, Ad @ Bd)
    print(f"gemm M{M} N{N} K{K} A{'MN' if a_mn else 'K'} B{'MN' if b_mn else 'K'} bn{bn}: {e:.1e}", flush=True)
    assert e <= TOL


def main():
    n = 0
    # every tile width, both operand majors, single CTAs and CTA pairs (M > 128)
    for bn in (64, 96, 128, 192, 256, 384):
        for a_mn, b_mn in ((0, 0), (1, 0), (0, 1), (1, 1)):
            for M in (100, 300):
                gemm_case(M, bn, 48, a_mn, b_mn, bn)
                n += 1
    # stream-K (>= one wave of tiles, ragged) and the composite 384 tile
    gemm_case(19200 + 64, 64, 32, 0, 0, 64); n += 1
    gemm_case(148 * 128 + 200, 384, 32, 0, 0, 384); n += 1
    # conv passes: materialised T1/T2/T3, implicit (fwd im2col, wgrad MN-major im2col incl. padded
    # taps, swapped wgrad / dgrad), space-to-depth, CH2 chains (K > 4096), split-K
    conv_case("small", 9, 3, 16, 32, 2, 1, 1); n += 3
    conv_case("imp48", 9, 3, 48, 64, 2, 1, 1, implicit_bwd=2); n += 3
    conv_case("imp_wide", 9, 3, 32, 256, 2, 1, 1, implicit_bwd=2); n += 3
    conv_case("imp384", 7, 3, 64, 384, 2, 1, 1, types=(1,), implicit_bwd=2); n += 1
    conv_case("dgrad_swap", 9, 3, 96, 64, 3, 1, 1, types=(1,), implicit_bwd=2, dgrad_swap=2); n += 1
    conv_case("s2d", 23, 11, 3, 96, 2, 4, 0, types=(1,), s2d=2); n += 1
    conv_case("conv1like", 23, 11, 3, 96, 2, 4, 0); n += 3
    conv_case("chain2", 7, 3, 512, 256, 2, 1, 1, types=(1,)); n += 1
    conv_case("nopairs", 9, 3, 32, 96, 2, 1, 1, types=(1,), cta_pairs=1); n += 1
    conv_case("single_producer", 9, 3, 32, 96, 2, 1, 1, types=(1,), split_producer=0); n += 1
    conv_case("a_smem", 9, 3, 32, 64, 2, 1, 1, types=(1,), a_tmem=0, a_tmem_wide=0); n += 1
    conv_case("a_ring", 9, 3, 32, 64, 2, 1, 1, types=(1,), a_tmem=2); n += 1
    conv_case("fwd_swap", 19, 3, 16, 64, 4, 1, 1, types=(1,), fwd_swap=1); n += 1
    # fused small-channel Type 1 (gather forward / backward-weight, hfold backward-data) at a
    # batch whose tiles wrap every ring (> 148 tiles: CTAs with several tiles and chains)
    conv_case("gather_conv1", 227, 11, 3, 96, 8, 4, 0, types=(1,)); n += 1
    conv_case("gather_6mma", 227, 11, 3, 96, 8, 4, 0, types=(1,), gather=2); n += 1
    conv_case("gather_pad", 71, 11, 3, 64, 3, 4, 2, types=(1,)); n += 1
    conv_case("gather_no_overlap", 71, 11, 3, 64, 3, 4, 2, types=(1,), overlap=0); n += 1
    # Types 2 / 3 streaming kernels (bulk-copy lift, shift-copy expand): strides 2 and 3, odd plane
    # sizes (runs at every 16-byte phase), partial channel groups
    conv_case("t23_s2", 11, 5, 4, 20, 3, 2, 2, types=(2, 3)); n += 2
    conv_case("t23_s3", 15, 3, 4, 13, 3, 3, 0, types=(2, 3)); n += 2
    conv_case("t23_k1", 9, 1, 4, 7, 3, 2, 0, types=(2, 3)); n += 2
    print(f"SANITIZE_CASES_OK {n}", flush=True)


if __name__ == "__main__":
    main()
