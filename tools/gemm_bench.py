"""Per-layout microbenchmark of the tcgen05 GEMM kernel (cct_debug_gemm).

Usage: python tools/gemm_bench.py [--only NAME] [--reps R]
Prints TF/s (algorithmic 2MNK) for each operand-storage combination with 1
(plain TF32) and 3 (3xTF32) tensor-core passes.
"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402

L = cct.lib()
L.cct_debug_gemm.argtypes = [C.c_int64] * 3 + [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_int,
                                               C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p]
L.cct_debug_gemm.restype = C.c_int

SHAPES = {
    # name: (M, N, K) -- conv2 b=256 shapes (K capped at the 4096 chain limit)
    "fwd_like": (186624, 256, 2400),
    "dgrad_like": (2400, 186624, 256),
    "wgrad_like": (2400, 256, 4096),
    "square": (8192, 8192, 2048),
    "narrow96": (65536, 96, 4096),
    "narrow64": (65536, 64, 4096),
    "conv1fwd": (774400, 96, 432),
    "conv1dgrad": (831744, 48, 864),
    "mid192": (65536, 192, 4096),
}


def run(M, N, K, amaj, bmaj, passes, bn=0, reps=10, cmaj=0):
    dev = torch.device("cuda")
    A = torch.rand((K, M) if amaj else (M, K), device=dev)
    B = torch.rand((K, N) if bmaj else (N, K), device=dev)
    Cm = torch.empty((M, N), device=dev)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def go():
        # cmaj = 1: column-major C (lanes = rows contiguous), as the conv passes store
        ldm, ldn = (1, M) if cmaj else (N, 1)
        rc = L.cct_debug_gemm(M, N, K, A.data_ptr(), A.shape[1], amaj, B.data_ptr(), B.shape[1], bmaj,
                              Cm.data_ptr(), ldm, ldn, passes, bn, st)
        assert rc == 0, L.cct_last_error()

    for _ in range(3):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 2.0 * M * N * K / ms / 1e9


def rate_table(reps=5):
    """Steady-state GEMM rate vs tile width N and reduction length K (cost-model
    calibration): M large enough for >= 16 tiles per CTA pair, so pipeline fill and
    the last wave are a small part of the time (the model adds those separately)."""
    out = {}
    for N in (64, 96, 128, 192, 256, 384, 1024):
        for K in (64, 256, 1024, 4096):
            M = 524288 if N < 1024 else 131072
            if K == 4096:
                M //= 4
            ms, tf = run(M, N, K, 0, 0, 3, 0, reps, cmaj=1)
            out[f"{N},{K}"] = tf
            print(f"rate N={N:5d} K={K:5d}: {tf:6.1f} TF/s", flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--bn", type=int, default=0)
    ap.add_argument("--layouts", default="kk,mm,mk,km")
    ap.add_argument("--passes", default="1,3")
    ap.add_argument("--rate-table", action="store_true")
    a = ap.parse_args()
    if a.rate_table:
        import json
        print(json.dumps(rate_table()))
        raise SystemExit(0)
    for name, (M, N, K) in SHAPES.items():
        if a.only and a.only != name:
            continue
        lay = {"kk": (0, 0), "mm": (1, 1), "mk": (1, 0), "km": (0, 1)}
        for amaj, bmaj in (lay[x] for x in a.layouts.split(",")):
            res = []
            for passes in (int(x) for x in a.passes.split(",")):
                ms, tf = run(M, N, K, amaj, bmaj, passes, a.bn, a.reps, cmaj=1)
                res.append(f"p{passes}: {ms:7.3f} ms {tf:6.1f} TF/s")
            print(f"{name:11s} M={M} N={N} K={K} A={'MN' if amaj else 'K '} B={'MN' if bmaj else 'K '} | "
                  + " | ".join(res), flush=True)

