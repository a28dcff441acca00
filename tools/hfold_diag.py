"""Diagnostic: fused backward-data (hfold) vs the materialised path by batch size, image and row."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402

n, k, d, o, s, p = 227, 11, 3, 96, 4, 0
dev = torch.device("cuda")
for b in [int(v) for v in sys.argv[1:]] or [8, 64, 149, 256]:
    desc = cct.ConvDesc(n, k, d, o, b, s, p, cct.NHWC)
    g = torch.Generator(device=dev).manual_seed(31)
    m = desc.m
    dy = torch.rand((b, m, m, o), generator=g, device=dev) * 2 - 1
    w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
    dx = conv.conv_bwd_data(dy, w, desc, cct.LOWER_T1)
    with cct.tuning(gather=0):
        dx0 = conv.conv_bwd_data(dy, w, desc, cct.LOWER_T1)
    err = ((dx - dx0).norm() / dx0.norm()).item()
    bad = ((dx - dx0).abs() > 1e-3 * dx0.abs().max()).nonzero()
    print(f"b={b}: rel-L2 {err:.3e}, bad elements {bad.shape[0]}", flush=True)
    if bad.shape[0]:
        imgs = bad[:, 0].unique()
        print("  images:", imgs[:20].tolist(), "count", imgs.numel())
        rows = bad[:, 1].unique()
        print("  rows:", rows[:40].tolist(), "count", rows.numel())
        cols = bad[:, 2].unique()
        print("  cols:", cols[:40].tolist(), "count", cols.numel())
