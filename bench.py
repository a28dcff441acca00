"""Benchmark: CaffeNet conv1-conv5 fwd + bwd-data + bwd-weight on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N > 1: torchrun --nproc-per-node N ... bench.py --gpus N ...)

Workload (BASELINE.json configs[3], and configs[4] at N = 8): the conv1-5
stack with the cost model choosing each layer's lowering, 256 images per GPU
(weak scaling; 8 GPUs = the 2048-image global batch of configs[4]).  A step =
fwd conv1..5, then bwd-data + bwd-weight conv5..1, plus the NCCL sum
all-reduce of every layer's weight gradient when N > 1.  Inputs are U(-1,1)
synthetic tensors of the CaffeNet shapes; the step's working set (> 2 GB)
exceeds the 126 MB L2, so no flush is needed between steps.

value  = images/s over all ranks, inputs resident in HBM, CUDA-event timed on
         the compute stream, max over ranks.
e2e    = the same step through the C ABI fed from pinned HOST buffers: per step
         H2D of every layer's x and dy, D2H of every layer's dW (the result).
roofline = the dominant kernel (the tcgen05 3xTF32 GEMM), timed live with CUDA
         events around every GEMM launch inside the timed region.
cpu_baseline = the reference's own CPU path (oracle/_ref: its multiply,
         gemm.cpp:93, around the restated lowering) on a bounded sample, rank 0, N = 1.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import shutil
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv fwd+bwd images/s and TFLOPS vs B200 peak at 1/2/4/8 GPUs vs CPU ref"
UNIT = "images/s"
PHASES = ["lower", "gemm", "lift", "expand", "col2im", "reduce", "other"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256, help="images per GPU")
    ap.add_argument("--lowering", default="auto", help="auto | 1 | 2 | 3 | comma list per layer")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="images in the CPU sample (0 = auto)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None
        self.path = f"/tmp/cct_clocks_{os.getpid()}.csv"

    def start(self):
        if shutil.which("nvidia-smi") is None:
            return
        self.f = open(self.path, "w")
        self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                   "-i", str(self.idx), "-lms", "200"], stdout=self.f,
                                  stderr=subprocess.DEVNULL)

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref), used by --impl reference and cpu_baseline
# ---------------------------------------------------------------------------
def cpu_reference_stack(images: int, types, threads: int):
    """Time the reference CPU path on `images` images of the conv1-5 stack.
    Returns (seconds, images, kind, threads)."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_py import REF_SO, Oracle, Reference  # noqa: E402
    from paper_1504_04343_b200.stack import CAFFENET
    kind = "reference" if os.path.exists(REF_SO) else "port"
    impl = Reference() if kind == "reference" else Oracle()
    orc = Oracle()
    rng = np.random.default_rng(7)
    t = 0.0
    for li, l in enumerate(CAFFENET):
        m = (l.n + 2 * l.pad - l.k) // l.stride + 1
        x = rng.uniform(-1, 1, images * l.n * l.n * l.d).astype(np.float32)
        w = rng.uniform(-1, 1, l.o * l.k * l.k * l.d).astype(np.float32)
        dy = rng.uniform(-1, 1, images * l.o * m * m).astype(np.float32)
        args = (images, l.n, l.d, l.k, l.o, l.stride, l.pad)
        tp = types[li]
        t0 = time.perf_counter()
        if kind == "reference":
            impl.lowered("fwd", tp, x, w, *args, threads=threads)
            impl.lowered("bwd_data", tp, dy, w, *args, threads=threads)
            impl.lowered("bwd_weight", tp, x, dy, *args, threads=threads)
        else:
            orc.lowered("fwd", tp, x, w, *args)
            orc.lowered("bwd_data", tp, dy, w, *args)
            orc.lowered("bwd_weight", tp, x, dy, *args)
        t += time.perf_counter() - t0
    return t, images, kind, (threads if kind == "reference" else 1)


def run_reference(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import paper_1504_04343_b200 as cct
    from paper_1504_04343_b200.stack import CAFFENET
    types = [cct.select_lowering(l.desc(a.batch), 3)[0] for l in CAFFENET]
    threads = min(os.cpu_count() or 1, 256)
    sample = a.cpu_sample or 1
    for _ in range(a.warmup):
        cpu_reference_stack(sample, types, threads)
    tot, imgs = 0.0, 0
    for _ in range(a.steps):
        t, n, kind, thr = cpu_reference_stack(sample, types, threads)
        tot += t
        imgs += n
    v = imgs / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp64 accumulate)", "data": "synthetic U(-1,1)",
        "config": {"workload": "caffenet conv1-5 fwd+bwd_data+bwd_weight, per-layer lowering as the B200 arm",
                   "images_per_step": sample, "lowering": types},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": kind,
                         "sample": f"{sample} image(s) of the conv1-5 stack per step, fwd+bwd, reference "
                                   f"multiply (gemm.cpp:93) with {thr} threads around the restated lowering"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "tflops": v * 6.4598e9 / 1e12,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)), "measured"
        except ValueError:
            pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def gemm_traffic():
    """DRAM bytes per GEMM launch from the committed ncu launch list of this
    command (profiles/r01/gemm_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "r01", "gemm_traffic.json")
    try:
        return json.load(open(p))["avg_dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


def tf32_cublas_probe(torch):
    """cuBLAS dense TF32 throughput on this box (context for the roofline)."""
    n = 8192
    a = torch.rand((n, n), device="cuda")
    b = torch.rand((n, n), device="cuda")
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    torch.backends.cuda.matmul.allow_tf32 = prev
    return 2.0 * n ** 3 / (e0.elapsed_time(e1) / 5 * 1e-3) / 1e12


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_1504_04343_b200 as cct
    from paper_1504_04343_b200.stack import CAFFENET, ConvStack

    world, rank, local = dist_env()
    if world != a.gpus:
        a.gpus = world if world > 1 else a.gpus
    # CCT_BENCH_BACKEND=gloo lets several ranks share one GPU to exercise the
    # multi-rank path where only one device is available (validation only).
    backend = os.environ.get("CCT_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    L = cct.lib()
    if a.lowering == "auto":
        lowering = cct.LOWER_AUTO
    elif "," in a.lowering:
        lowering = [int(t) for t in a.lowering.split(",")]
    else:
        lowering = int(a.lowering)
    st = ConvStack(a.batch, dev, CAFFENET, lowering, group=group, seed=1234 + rank)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(a.warmup):
        st.step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    if rank == 0:
        clocks.start()
        time.sleep(0.3)
    cct.reset_launch_count()
    L.cct_profile_read(None, None, None, None, 1)
    L.cct_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        st.step()
    e1.record(stream)
    torch.cuda.synchronize()
    L.cct_profile_enable(0)
    launches = cct.launch_count()
    barrier()
    clk = clocks.stop() if rank == 0 else None
    ms = e0.elapsed_time(e1) / a.steps
    ms_max = ms
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    P = C.c_double * 7
    pms, pfl, pby = P(), P(), P()
    pn = (C.c_uint64 * 7)()
    L.cct_profile_read.argtypes = [P, P, P, C.c_uint64 * 7, C.c_int]
    L.cct_profile_read(pms, pfl, pby, pn, 1)
    phase = {PHASES[i]: {"ms_per_step": pms[i] / a.steps, "launches_per_step": pn[i] / a.steps}
             for i in range(7) if pn[i]}

    images = a.batch * world
    value = images / (ms_max * 1e-3)
    flops_step = st.flops_per_step() * world
    tflops = flops_step / (ms_max * 1e-3) / 1e12

    # ---- e2e: host-fed step through the C ABI -------------------------------
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, st, torch, world, group, dev)

    peaks, peak_src = measured_peaks()
    tf32_meas = tf32_cublas_probe(torch) if rank == 0 else None
    # dominant kernel: the GEMM.  achieved = algorithmic conv flops / GEMM device time.
    gemm_ms = pms[1] / a.steps
    alg_per_rank = st.flops_per_step()
    achieved = alg_per_rank / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    # The GEMMs run at max SM clock inside this step (clocks below), so the ceiling is
    # the burst tensor rate: measured dense bf16 / 2 (TF32) / 3 (three products).  The
    # sustained figure (power-capped 4 s matmul at ~1.3 GHz) is kept for reference.
    peak = peaks.get("bf16_tflops") / 2.0 / 3.0
    peak_sus = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) / 2.0 / 3.0
    roofline = {
        "bound": "tensor", "kernel": "gemm3xtf32_kernel (tcgen05 kind::tf32, 3 products per K step)",
        "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": (achieved / peak) if achieved else None,
        "peak_source": f"{peak_src} bf16_tflops (burst) / 2 (TF32 rate) / 3 (3xTF32 products)",
        "peak_sustained": peak_sus,
        "tf32_cublas_tflops_measured": tf32_meas,
        "frac_of_burst_ceiling": (achieved / (tf32_meas / 3.0)) if (achieved and tf32_meas) else None,
        "step_frac": (flops_step / world / (ms_max * 1e-3) / 1e12) / peak,
        "traffic": gemm_traffic(),
        "gemm_share_of_step": (gemm_ms / ms) if ms else None,
    }

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        try:
            thr = min(os.cpu_count() or 1, 256)
            sample = a.cpu_sample or 1
            t, n, kind, used = cpu_reference_stack(sample, st.types, thr)
            cpu = {"value": n / t, "unit": UNIT, "cores": used, "kind": kind,
                   "sample": f"{n} image(s) of the conv1-5 stack fwd+bwd ({t:.1f} s), lowering {st.types}"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "unavailable", "sample": repr(exc)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (3xTF32 tensor-core GEMMs, fp32 accumulate)",
            "data": "synthetic U(-1,1), CaffeNet conv1-5 shapes",
            "config": {"workload": "caffenet conv1-5 fwd+bwd_data+bwd_weight, auto lowering per layer",
                       "images_per_gpu": a.batch, "global_batch": images,
                       "lowering": {l.name: t for l, t in zip(st.layers, st.types)},
                       "parallelism": f"dp{world} (batch split, NCCL all-reduce of dW)" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (step working set > 2 GB)"},
            "tflops": tflops, "tflops_per_gpu": tflops / world,
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clk, "phases": phase,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(a, st, torch, world, group, dev):
    """K steps fed from pinned host memory: H2D x/dy of every layer on a copy
    stream (overlapping the previous layer's compute), D2H of every dW.  The device
    inputs are double-buffered, so step k+1's copies start while step k computes
    (the copy stream waits only for the step that last read the same buffer set)."""
    import torch.distributed as dist
    hx = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in st.x]
    hdy = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in st.dy]
    hdw = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in st.dw]
    for h, t in zip(hx + hdy, st.x + st.dy):
        h.copy_(t.cpu())
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream(device=dev)
    nl = len(st.layers)
    h2d = sum(t.numel() * 4 for t in hx + hdy)
    d2h = sum(t.numel() * 4 for t in hdw)
    bufs = [(st.x, st.dy), ([torch.empty_like(t) for t in st.x], [torch.empty_like(t) for t in st.dy])]
    done = [None, None]  # comp-stream event: the last step that read buffer set s finished
    step = [0]

    def one():
        s = step[0] & 1
        step[0] += 1
        xs, dys = bufs[s]
        evx, evdy = [], []
        with torch.cuda.stream(copy):
            if done[s] is not None:
                copy.wait_event(done[s])
            for i in range(nl):
                xs[i].copy_(hx[i], non_blocking=True)
                e = torch.cuda.Event()
                e.record(copy)
                evx.append(e)
            for i in reversed(range(nl)):
                dys[i].copy_(hdy[i], non_blocking=True)
                e = torch.cuda.Event()
                e.record(copy)
                evdy.append(e)
        evdy = evdy[::-1]
        from paper_1504_04343_b200.conv import conv_bwd, conv_fwd_cached
        for i, d in enumerate(st.descs):
            comp.wait_event(evx[i])
            conv_fwd_cached(xs[i], st.w[i], d, st.types[i], cache=st.cache[i], out=st.y[i], ws=st.ws)
        handles = []
        for i in reversed(range(nl)):
            d, t = st.descs[i], st.types[i]
            comp.wait_event(evdy[i])
            conv_bwd(dys[i], st.w[i], d, t, x=xs[i], cache=st.cache[i], dx=st.dx[i], dw=st.dw[i], ws=st.ws)
            if group is not None:
                handles.append((i, dist.all_reduce(st.dw[i], group=group, async_op=True)))
            else:
                hdw[i].copy_(st.dw[i], non_blocking=True)
        for i, h in handles:
            h.wait()
            hdw[i].copy_(st.dw[i], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(comp)
        done[s] = ev

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(a.steps):
        one()
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": a.batch * world / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "h2d_gb_per_s": h2d / (ms * 1e-3) / 1e9,
            "path": "C ABI (cct_conv_*) on double-buffered device inputs fed by pinned-host H2D copies on a side stream"}


if __name__ == "__main__":
    if os.environ.get("CCT_BENCH_WATCHDOG"):  # diagnostics: dump the Python stacks after N s
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["CCT_BENCH_WATCHDOG"]), repeat=True)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
