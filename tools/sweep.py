"""BASELINE configs[1]: lowering-type sweep over input/output channel ratios.

n=13, k=3, pad 1, stride 1, batch 256; d*o fixed at 2^16 and 2^17, d/o from 1/16 to 16
(SURVEY 8(a) a12).  For every point and every lowering type: one training step of the layer
(fwd with the lowered cache + combined bwd) timed with CUDA events, the per-phase device
counters (cct_profile_*), and the cost model's prediction / choice.  Writes one JSON object
per point to --out and prints a table.

Also used to calibrate the cost model: `--calibrate` fits the per-phase rates from the
measured counters and prints a cct_calibration.
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1504_04343_b200 as cct  # noqa: E402
from paper_1504_04343_b200 import conv  # noqa: E402

PHASES = ["lower", "gemm", "lift", "expand", "col2im", "reduce", "other"]
POINTS = [(64, 1024), (128, 512), (256, 256), (512, 128), (1024, 64),
          (128, 1024), (256, 512), (512, 256), (1024, 128)]


def step_time(desc, t, x, w, dy, reps):
    dev = x.device
    cache = conv.alloc_cache(desc, t, dev)
    ws = conv.Workspace(dev)
    ws.get(max(cct.workspace_size(desc, t, cct.PASS_FWD), cct.workspace_size(desc, t, cct.PASS_BWD)))
    y = torch.empty(desc.y_shape(), device=dev)
    dx = torch.empty_like(x)
    dw = torch.empty_like(w)

    def one():
        conv.conv_fwd_cached(x, w, desc, t, cache=cache, out=y, ws=ws)
        conv.conv_bwd(dy, w, desc, t, x=x, cache=cache, dx=dx, dw=dw, ws=ws)

    one()
    torch.cuda.synchronize()
    L = cct.lib()
    P = C.c_double * 7
    ms, fl, by = P(), P(), P()
    n = (C.c_uint64 * 7)()
    L.cct_profile_read.argtypes = [P, P, P, C.c_uint64 * 7, C.c_int]
    L.cct_profile_read(ms, fl, by, n, 1)
    L.cct_profile_enable(1)
    one()
    L.cct_profile_enable(0)
    L.cct_profile_read(ms, fl, by, n, 1)
    phases = {PHASES[i]: {"ms": ms[i], "flops": fl[i], "bytes": by[i], "launches": int(n[i])}
              for i in range(7) if n[i]}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(reps):
        e0.record()
        one()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    times.sort()
    return times[len(times) // 2], phases


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    ap.add_argument("--extra", default="", help="extra n,k,d,o,s,p points separated by ';'")
    a = ap.parse_args()
    dev = torch.device("cuda")
    pts = [(13, 3, d, o, 1, 1) for d, o in POINTS]
    if a.extra:
        pts += [tuple(int(v) for v in p.split(",")) for p in a.extra.split(";")]
    rows = []
    for (n, k, d, o, s, p) in pts:
        desc = cct.ConvDesc(n, k, d, o, a.batch, s, p)
        g = torch.Generator(device=dev).manual_seed(d * 7 + o)
        x = torch.rand((a.batch, n, n, d), generator=g, device=dev) * 2 - 1
        w = torch.rand((o, k, k, d), generator=g, device=dev) * 2 - 1
        dy = torch.rand((a.batch, o, desc.m, desc.m), generator=g, device=dev) * 2 - 1
        choice, est = cct.select_lowering(desc, 3)
        rec = {"n": n, "k": k, "d": d, "o": o, "stride": s, "pad": p, "b": a.batch, "ratio": d / o,
               "alg_gflop_step": 3 * desc.flops_per_pass() / 1e9, "model_choice": choice, "types": {}}
        for t in (1, 2, 3):
            ms, ph = step_time(desc, t, x, w, dy, a.reps)
            rec["types"][t] = {"ms": ms, "model_ms": est[t - 1].model_seconds * 1e3,
                               "alg_tflops": 3 * desc.flops_per_pass() / (ms * 1e-3) / 1e12, "phases": ph}
        meas = min(rec["types"], key=lambda t: rec["types"][t]["ms"])
        rec["measured_best"] = meas
        rows.append(rec)
        tt = rec["types"]
        print(f"d={d:5d} o={o:5d} d/o={d / o:7.4f} | T1 {tt[1]['ms']:7.3f} ms | T2 {tt[2]['ms']:7.3f} ms | "
              f"T3 {tt[3]['ms']:7.3f} ms | best T{meas} | model T{choice} "
              f"(model ms {tt[1]['model_ms']:.3f}/{tt[2]['model_ms']:.3f}/{tt[3]['model_ms']:.3f})", flush=True)
        for t in (2, 3):
            ph = tt[t]["phases"]
            print("      T%d phases: " % t + "  ".join(
                f"{nm} {v['ms'] * 1e3:6.0f} us {v['bytes'] / (v['ms'] * 1e-3) / 1e12 if v['ms'] else 0:4.2f} TB/s"
                for nm, v in ph.items() if nm != "gemm") + f"  gemm {ph['gemm']['ms'] * 1e3:6.0f} us", flush=True)
        del x, w, dy
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")
    # calibration: aggregate measured rates per phase class
    agg = {}
    for r in rows:
        for t in r["types"].values():
            for nm, v in t["phases"].items():
                A = agg.setdefault(nm, [0.0, 0.0, 0.0, 0])
                A[0] += v["ms"]
                A[1] += v["bytes"]
                A[2] += v["flops"]
                A[3] += v["launches"]
    print("measured phase rates:")
    for nm, (ms, by, fl, nl) in agg.items():
        print(f"  {nm:7s} {by / (ms * 1e-3) / 1e12 if ms else 0:6.2f} TB/s  {fl / (ms * 1e-3) / 1e12 if ms else 0:7.1f} "
              f"TF/s  {ms / nl * 1e3 if nl else 0:8.1f} us/launch")
    hits = sum(1 for r in rows if r["model_choice"] == r["measured_best"])
    print(f"model choice == measured best on {hits}/{len(rows)} points")


if __name__ == "__main__":
    main()
