"""First-light diagnostics on the B200 (run under gpurun with a timeout).

Prints one line per check and keeps going after failures so one GPU call
yields as much information as possible.  Uses the oracle only as the checker.
"""
import os
import sys
import time
import traceback

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402
from oracle_py import Oracle, rel_l2  # noqa: E402

dev = torch.device("cuda:0")
orc = Oracle()


def step(name, fn):
    t0 = time.time()
    try:
        msg = fn()
        torch.cuda.synchronize()
        print(f"[ok  ] {name}: {msg} ({time.time() - t0:.1f}s)", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"[FAIL] {name}: {e!r}", flush=True)
        traceback.print_exc()


def tf32_semantics():
    v = 1.0 + 3 * 2.0 ** -12  # trunc -> 1.0 ; RN -> 1 + 2^-10
    a = torch.full((128, 16), 0.0, device=dev)
    a[:, 0] = v
    b = torch.zeros((16, 128), device=dev)
    b[0, :] = 1.0
    c1 = conv.multiply_passes(a, b, 1)
    c3 = conv.multiply_passes(a, b, 3)
    return f"1-pass={c1[0, 0].item()!r} (trunc=1.0, rn={1 + 2 ** -10}), 3-pass={c3[0, 0].item()!r} exact={v!r}"


def gemm_check(M, N, K, split=1):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    c = conv.multiply(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), split_k=split).cpu().numpy()
    c1 = conv.multiply_passes(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), 1).cpu().numpy()
    return f"3xTF32 relL2={rel_l2(c, ref):.2e}  1xTF32 relL2={rel_l2(c1, ref):.2e}"


def conv_check(n, k, d, o, b, s, p, t):
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x, w = orc.random_problem(1234, b, n, d, k, o)
    m = desc.m
    dy = orc.uniform(99, b * o * m * m)
    xt = torch.from_numpy(x).to(dev).view(b, n, n, d)
    wt = torch.from_numpy(w).to(dev).view(o, k, k, d)
    dyt = torch.from_numpy(dy).to(dev).view(b, o, m, m)
    y = conv.conv_fwd(xt, wt, desc, t).cpu().numpy().ravel()
    dx = conv.conv_bwd_data(dyt, wt, desc, t).cpu().numpy().ravel()
    dw = conv.conv_bwd_weight(xt, dyt, desc, t).cpu().numpy().ravel()
    ry = orc.conv_fwd(x, w, b, n, d, k, o, s, p)
    rdx = orc.conv_bwd_data(dy, w, b, n, d, k, o, s, p)
    rdw = orc.conv_bwd_weight(x, dy, b, n, d, k, o, s, p)
    return f"T{t} fwd={rel_l2(y, ry):.2e} dgrad={rel_l2(dx, rdx):.2e} wgrad={rel_l2(dw, rdw):.2e}"


def timing(n, k, d, o, b, s, p, t, reps=5):
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    m = desc.m
    x = torch.rand((b, n, n, d), device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), device=dev) * 2 - 1
    dy = torch.rand((b, o, m, m), device=dev) * 2 - 1
    out = []
    for name, f in (("fwd", lambda: conv.conv_fwd(x, w, desc, t)),
                    ("dgrad", lambda: conv.conv_bwd_data(dy, w, desc, t)),
                    ("wgrad", lambda: conv.conv_bwd_weight(x, dy, desc, t))):
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out.append(f"{name} {ms:.3f} ms {desc.flops_per_pass() / ms / 1e9:.1f} TF/s")
    return " | ".join(out)


def lower_bw(n, k, d, o, b, s, p, t, reps=5):
    desc = cct.ConvDesc(n, k, d, o, b, s, p)
    x = torch.rand((b, n, n, d), device=dev)
    f = lambda: conv.lower(x, desc, t, cct.ROWS_INTERNAL)  # noqa: E731
    dh = f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byts = dh.numel() * 4 + x.numel() * 4
    return f"{ms:.3f} ms (incl. alloc) {byts / ms / 1e6:.0f} GB/s alg"


if __name__ == "__main__":
    print(torch.cuda.get_device_name(0), torch.cuda.get_device_capability(0), flush=True)
    step("tf32 semantics", tf32_semantics)
    for shp in [(128, 128, 16), (256, 256, 256), (300, 200, 100), (1000, 96, 363), (129, 257, 1000)]:
        step(f"gemm {shp}", lambda shp=shp: gemm_check(*shp))
    step("gemm split-K (64,64,40000) s=8", lambda: gemm_check(64, 64, 40000, split=8))
    for K in (512, 2048, 8192, 32768):
        step(f"gemm chain K={K} split=1", lambda K=K: gemm_check(256, 256, K, split=1))
        step(f"gemm chain K={K} auto", lambda K=K: gemm_check(256, 256, K, split=0))
    cfgs = [(9, 3, 4, 8, 2, 1, 0), (11, 3, 8, 16, 2, 1, 1), (13, 5, 4, 12, 2, 2, 2), (23, 11, 3, 8, 2, 4, 0),
            (27, 5, 96, 256, 2, 1, 2), (13, 3, 256, 384, 2, 1, 1)]
    for cfg in cfgs:
        for t in (1, 2, 3):
            step(f"conv {cfg}", lambda cfg=cfg, t=t: conv_check(*cfg, t))
    step("timing conv2 b256 T1", lambda: timing(27, 5, 96, 256, 256, 1, 2, 1))
    step("timing conv3 b256 T1", lambda: timing(13, 3, 256, 384, 256, 1, 1, 1))
    step("lower bw conv2 T1", lambda: lower_bw(27, 5, 96, 256, 256, 1, 2, 1))
    step("lower bw conv1 T1", lambda: lower_bw(227, 11, 3, 96, 256, 4, 0, 1))
    step("timing conv1 b256 T1", lambda: timing(227, 11, 3, 96, 256, 4, 0, 1))
    step("timing conv5 b256 T3", lambda: timing(13, 3, 384, 256, 256, 1, 1, 3))
    step("launch count", lambda: str(cct.launch_count()))
