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
e2e    = the same step through the C ABI fed from and returned to pinned HOST
         buffers: per step H2D of every layer's x and dy, D2H of every layer's
         y, dx and dW (the results the reference API returns on the host).
configs = device-timed configs[0] (conv2 b=256 T1), configs[2] (conv1 b=256) and
         the configs[1] ratio sweep, plus configs[0] on the reference CPU path.
--global-batch G = strong scaling (configs[4]: 2048 split over the ranks).
roofline = the dominant kernel (the tcgen05 3xTF32 GEMM), timed live with CUDA
         events around every GEMM launch inside the timed region.
cpu_baseline = the reference's own CPU path (oracle/_ref: its multiply,
         gemm.cpp:93, around the restated lowering) on a bounded sample (32 images of
         the stack), rank 0, N = 1.
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
WORKLOAD = "caffenet conv1-5 fwd+bwd_data+bwd_weight, auto lowering per layer"
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
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling (configs[4]): split this many images over the ranks "
                         "(0 = weak scaling, --batch images per GPU)")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs[0..2] device / CPU lines")
    ap.add_argument("--layout", default="nhwc", choices=["nchw", "nhwc"],
                    help="y / dy layout of every layer (NHWC = the next layer's input order)")
    ap.add_argument("--h2d-wc", type=int, default=0, help="e2e: write-combined pinned H2D source buffers (1)")
    ap.add_argument("--copy-streams", type=int, default=1,
                    help="e2e: copy streams per direction (measured: 2-3 no faster than 1)")
    ap.add_argument("--tune", default="", help="A/B runs: comma list key=value of cct_set_tuning switches")
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
# reference CPU path (oracle/_ref), used by --impl reference and cpu_baseline.
# This half of the file never imports the package or loads libcct.so: the
# reference arm is the reference's own code only.
# ---------------------------------------------------------------------------
# (name, n, k, d, o, stride, pad) -- BASELINE.json configs: conv1 227x227x3 -> 96 k11 s4;
# conv2 27x27x96 -> 256 k5 p2; conv3-5 13x13, k3, p1 (= stack.CAFFENET, tests/test_bench_contract.py)
CAFFENET_GEOM = (("conv1", 227, 11, 3, 96, 4, 0), ("conv2", 27, 5, 96, 256, 1, 2),
                 ("conv3", 13, 3, 256, 384, 1, 1), ("conv4", 13, 3, 384, 384, 1, 1),
                 ("conv5", 13, 3, 384, 256, 1, 1))
# the lowering the B200 arm's cost model picks for the stack at b = 256 (checked against
# cct_select_lowering by tests/test_bench_contract.py), so both arms run the same types
REF_TYPES = (1, 1, 1, 1, 1)
STACK_GFLOP_PER_IMAGE = 6.4598  # 3 passes x sum 2 m^2 k^2 d o
CPU_STACK_SAMPLE = 32           # images per CPU step (b = 32 for the stack)


def _reference_impl():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle_py import REF_SO, Oracle, Reference  # noqa: E402
    if os.path.exists(REF_SO):
        return Reference(), "reference"
    return Oracle(), "port"


def cpu_reference_layer(impl, kind, geom, images, tp, threads, seed=7):
    """One layer's fwd + bwd-data + bwd-weight on the reference CPU path; seconds."""
    import numpy as np
    _, n, k, d, o, s, p = geom
    m = (n + 2 * p - k) // s + 1
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, images * n * n * d).astype(np.float32)
    w = rng.uniform(-1, 1, o * k * k * d).astype(np.float32)
    dy = rng.uniform(-1, 1, images * o * m * m).astype(np.float32)
    args = (images, n, d, k, o, s, p)
    kw = {"threads": threads} if kind == "reference" else {}
    t0 = time.perf_counter()
    impl.lowered("fwd", tp, x, w, *args, **kw)
    impl.lowered("bwd_data", tp, dy, w, *args, **kw)
    impl.lowered("bwd_weight", tp, x, dy, *args, **kw)
    return time.perf_counter() - t0


def cpu_reference_stack(images: int, types, threads: int):
    """Time the reference CPU path (its multiply, gemm.cpp:93-122, threaded, around the
    restated lowering / lifting) on `images` images of the conv1-5 stack.
    Returns (seconds, images, kind, threads)."""
    impl, kind = _reference_impl()
    t = sum(cpu_reference_layer(impl, kind, g, images, types[li], threads, seed=7 + li)
            for li, g in enumerate(CAFFENET_GEOM))
    return t, images, kind, (threads if kind == "reference" else 1)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def ref_types(a):
    if a.lowering in ("auto", ""):
        return list(REF_TYPES)
    if "," in a.lowering:
        return [int(t) for t in a.lowering.split(",")]
    return [int(a.lowering)] * len(CAFFENET_GEOM)


def workload_config(a, world, per_gpu, global_images, types):
    """The `config` both arms print for the same command line (same workload, so the driver's
    same-config check holds); the reference arm's bounded sample is in its cpu_baseline."""
    return {"workload": WORKLOAD,
            "images_per_gpu": per_gpu, "global_batch": global_images,
            "lowering": {g[0]: t for g, t in zip(CAFFENET_GEOM, types)},
            "parallelism": f"dp{world} (batch split, NCCL all-reduce of dW)" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (step working set > 2 GB)",
            "layout": a.layout,
            **({"tune": a.tune} if a.tune else {})}


def run_reference(a):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    types = ref_types(a)
    # the GPU arm's per-rank batch for the same flags (equal split of --global-batch, rank 0's share)
    per_gpu = -(-a.global_batch // world) if a.global_batch else a.batch
    threads = min(os.cpu_count() or 1, 256)
    sample = a.cpu_sample or CPU_STACK_SAMPLE
    for _ in range(a.warmup):
        cpu_reference_stack(sample, types, threads)
    times = []
    kind, thr = "port", 1
    for _ in range(a.steps):
        t, n, kind, thr = cpu_reference_stack(sample, types, threads)
        times.append(t)
    tot = sum(times)
    v = sample * a.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * tot / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp64 accumulate)", "data": "synthetic U(-1,1), CaffeNet conv1-5 shapes",
        "config": workload_config(a, world, per_gpu, per_gpu * world if not a.global_batch else a.global_batch,
                                  types),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{sample} of the workload's images of the conv1-5 stack per step (BASELINE.md section 3), "
                                   f"fwd+bwd_data+bwd_weight, the reference's multiply (gemm.cpp:93) with {thr} "
                                   f"threads around the restated lowering; median step {1e3 * statistics.median(times):.0f} ms"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "tflops": v * STACK_GFLOP_PER_IMAGE / 1e3,
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
    """DRAM bytes per GEMM-phase launch from the committed ncu launch list of this
    command (profiles/r02/gemm_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "r02", "gemm_traffic.json")
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


def time_layer_step(torch, desc, tp, steps=5, warmup=2):
    """Device ms of one layer's training step (fwd with the lowered cache, then bwd-data +
    bwd-weight) through the C ABI, CUDA events on the current stream."""
    from paper_1504_04343_b200 import PASS_BWD, PASS_FWD, workspace_size
    from paper_1504_04343_b200.conv import Workspace, alloc_cache, conv_bwd, conv_fwd_cached
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(11)

    def u(*shape):
        return torch.rand(shape, generator=g, device=dev).mul_(2).sub_(1)

    x, w = u(desc.b, desc.n, desc.n, desc.d), u(desc.o, desc.k, desc.k, desc.d)
    dy = u(desc.b, desc.o, desc.m, desc.m)
    y, dx, dw = torch.empty_like(dy), torch.empty_like(x), torch.empty_like(w)
    cache = alloc_cache(desc, tp, dev)
    ws = Workspace(dev)
    ws.get(max(workspace_size(desc, tp, PASS_FWD), workspace_size(desc, tp, PASS_BWD)))

    def one():
        conv_fwd_cached(x, w, desc, tp, cache=cache, out=y, ws=ws)
        conv_bwd(dy, w, desc, tp, x=x, cache=cache, dx=dx, dw=dw, ws=ws)

    for _ in range(warmup):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run_configs(torch, ceiling):
    """Device-timed numbers for the other BASELINE.json configs on this GPU: configs[0]
    (conv2, b = 256, Type 1), configs[2] (conv1, b = 256, cost-model lowering) and the
    configs[1] ratio sweep (n = 13, k = 3, p = 1, b = 256; every type at every point)."""
    import paper_1504_04343_b200 as cct
    out = {}

    def rec(desc, tp):
        ms = time_layer_step(torch, desc, tp)
        fl = 3 * desc.flops_per_pass()
        return {"lowering": tp, "ms_per_step": ms, "images_per_s": desc.b / (ms * 1e-3),
                "tflops": fl / (ms * 1e-3) / 1e12, "frac_of_3xtf32_ceiling": fl / (ms * 1e-3) / 1e12 / ceiling}

    out["configs[0] conv2 b256 T1 fwd+bwd"] = rec(cct.ConvDesc(27, 5, 96, 256, 256, 1, 2), 1)
    c1 = cct.ConvDesc(227, 11, 3, 96, 256, 4, 0)
    out["configs[2] conv1 b256 auto fwd+bwd"] = rec(c1, cct.select_lowering(c1, 3)[0])
    sweep = []
    for d, o in ((64, 1024), (128, 512), (256, 256), (512, 128), (1024, 64),
                 (128, 1024), (256, 512), (512, 256), (1024, 128)):
        desc = cct.ConvDesc(13, 3, d, o, 256, 1, 1)
        row = {"d": d, "o": o, "d_over_o": d / o, "model_choice": cct.select_lowering(desc, 3)[0]}
        for tp in (1, 2, 3):
            r = rec(desc, tp)
            row[f"T{tp}_ms"] = r["ms_per_step"]
            row[f"T{tp}_tflops"] = r["tflops"]
        row["measured_best"] = min((1, 2, 3), key=lambda t: row[f"T{t}_ms"])
        sweep.append(row)
    out["configs[1] ratio sweep n13 k3 p1 b256 fwd+bwd"] = sweep
    return out


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
            # NCCL's own log (stderr) records the communicator's rank count and transport
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
        print(f"cct-bench rank {rank}/{world} on cuda:{local} backend {backend}", file=sys.stderr, flush=True)
    L = cct.lib()
    for kv in filter(None, a.tune.split(",")):
        k_, v_ = kv.split("=")
        cct.set_tuning(k_, int(v_))
    if a.lowering == "auto":
        lowering = cct.LOWER_AUTO
    elif "," in a.lowering:
        lowering = [int(t) for t in a.lowering.split(",")]
    else:
        lowering = int(a.lowering)
    strong = a.global_batch > 0
    st = ConvStack(a.batch, dev, CAFFENET, lowering, group=group, seed=1234, layout=int(a.layout == "nhwc"),
                   global_batch=a.global_batch if strong else None)
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

    images = st.global_batch
    value = images / (ms_max * 1e-3)
    flops_step = stack_flops(CAFFENET) * images
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
        "bound": "tensor", "kernel": "gemm3xtf32_kernel + the fused conv1 gather / hfold GEMMs (tcgen05 kind::tf32, 3 products per K step)",
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
    cfg = None
    if rank == 0 and world == 1 and not a.no_cpu:
        try:
            thr = min(os.cpu_count() or 1, 256)
            sample = a.cpu_sample or CPU_STACK_SAMPLE
            t, n, kind, used = cpu_reference_stack(sample, st.types, thr)
            cpu = {"value": n / t, "unit": UNIT, "cores": used, "kind": kind, "cpu_model": cpu_model(),
                   "sample": f"{n} images of the conv1-5 stack fwd+bwd_data+bwd_weight ({t:.1f} s; BASELINE.md "
                             f"section 3), lowering {st.types}, the reference's multiply with {used} threads"}
            if not a.no_configs:
                # configs[0] on the CPU at its full batch: conv2, b = 256, Type 1
                impl, kind1 = _reference_impl()
                t1 = cpu_reference_layer(impl, kind1, CAFFENET_GEOM[1], 256, 1, thr)
                cpu["configs[0] conv2 b256 T1 fwd+bwd"] = {
                    "images_per_s": 256 / t1, "seconds": t1, "tflops": 3 * 2 * 27 ** 2 * 25 * 96 * 256 * 256 / t1 / 1e12,
                    "cores": thr if kind1 == "reference" else 1, "kind": kind1}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "unavailable", "sample": repr(exc)}
    if rank == 0 and world == 1 and not a.no_configs:
        cfg = run_configs(torch, peak)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f32 (3xTF32 tensor-core GEMMs, fp32 accumulate)",
            "data": "synthetic U(-1,1), CaffeNet conv1-5 shapes",
            "config": workload_config(a, world, st.batch, images, list(st.types)),
            "tflops": tflops, "tflops_per_gpu": tflops / world,
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clk, "phases": phase, "configs": cfg,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def stack_flops(layers):
    return float(sum(3 * l.desc(1).flops_per_pass() for l in layers))


def run_e2e(a, st, torch, world, group, dev):
    """K steps through the C ABI fed from, and returning to, pinned HOST memory.
    Per step: H2D of every layer's x and dy (copy stream 1), D2H of every layer's
    y, dx and dW (copy stream 2) -- the reference API returns OutputBatch and the
    gradients on the host.  Inputs and outputs are double-buffered on
    the device, so step k+1's uploads and step k's downloads overlap compute."""
    import torch.distributed as dist

    from paper_1504_04343_b200.conv import conv_bwd, conv_fwd_cached
    nl = len(st.layers)
    pin = lambda ts: [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in ts]  # noqa: E731
    keep = []

    def pin_wc(ts):
        """Page-locked write-combined host buffers (cudaHostAllocWriteCombined) for the H2D
        sources: the DMA engine reads them without snooping the CPU caches."""
        import ctypes
        from cuda.bindings import runtime as cudart
        out = []
        for t in ts:
            nbytes = t.numel() * t.element_size()
            err, ptr = cudart.cudaHostAlloc(nbytes, cudart.cudaHostAllocWriteCombined)
            if int(err) != 0:
                return pin(ts)
            buf = (ctypes.c_char * nbytes).from_address(int(ptr))
            keep.append((ptr, buf))
            out.append(torch.frombuffer(buf, dtype=t.dtype).view(t.shape))
        return out

    hx, hdy = (pin_wc(st.x), pin_wc(st.dy)) if a.h2d_wc else (pin(st.x), pin(st.dy))
    hy, hdx, hdw = pin(st.y), pin(st.dx), pin(st.dw)
    for h, t in zip(hx + hdy, st.x + st.dy):
        h.copy_(t.cpu())
    comp = torch.cuda.current_stream()
    # several copy streams per direction: independent DMA queues keep both PCIe directions
    # busier than one stream each
    ncs = max(1, a.copy_streams)
    ups = [torch.cuda.Stream(device=dev) for _ in range(ncs)]
    downs = [torch.cuda.Stream(device=dev) for _ in range(ncs)]
    h2d = sum(t.numel() * 4 for t in hx + hdy)
    d2h = sum(t.numel() * 4 for t in hy + hdx + hdw)
    ins = [(st.x, st.dy), ([torch.empty_like(t) for t in st.x], [torch.empty_like(t) for t in st.dy])]
    outs = [(st.y, st.dx, st.dw), ([torch.empty_like(t) for t in st.y], [torch.empty_like(t) for t in st.dx],
                                   [torch.empty_like(t) for t in st.dw])]
    in_free = [None, None]   # comp event: the last step that read input set s is done
    out_free = [None, None]  # down events: the downloads of output set s are done
    step = [0]

    def ev(s):
        e = torch.cuda.Event()
        e.record(s)
        return e

    def one():
        s = step[0] & 1
        step[0] += 1
        xs, dys = ins[s]
        ys, dxs, dws = outs[s]
        evx, evdy = [None] * nl, [None] * nl
        if in_free[s] is not None:
            for u in ups:
                u.wait_event(in_free[s])
        for i in range(nl):
            u = ups[i % ncs]
            with torch.cuda.stream(u):
                xs[i].copy_(hx[i], non_blocking=True)
                evx[i] = ev(u)
        for i in reversed(range(nl)):
            u = ups[(i + 1) % ncs]
            with torch.cuda.stream(u):
                dys[i].copy_(hdy[i], non_blocking=True)
                evdy[i] = ev(u)
        if out_free[s] is not None:
            for e in out_free[s]:
                comp.wait_event(e)

        def download(j, host, dev_t):
            e = ev(comp)
            dn = downs[j % ncs]
            with torch.cuda.stream(dn):
                dn.wait_event(e)
                host.copy_(dev_t, non_blocking=True)

        for i, d in enumerate(st.descs):
            comp.wait_event(evx[i])
            conv_fwd_cached(xs[i], st.w[i], d, st.types[i], cache=st.cache[i], out=ys[i], ws=st.ws)
            download(i, hy[i], ys[i])
        handles = []
        for i in reversed(range(nl)):
            d, t = st.descs[i], st.types[i]
            comp.wait_event(evdy[i])
            conv_bwd(dys[i], st.w[i], d, t, x=xs[i], cache=st.cache[i], dx=dxs[i], dw=dws[i], ws=st.ws)
            download(i + 1, hdx[i], dxs[i])
            if group is not None:
                handles.append((i, dist.all_reduce(dws[i], group=group, async_op=True)))
            else:
                download(i, hdw[i], dws[i])
        for i, h in handles:
            h.wait()
            download(i, hdw[i], dws[i])
        in_free[s] = ev(comp)
        out_free[s] = [ev(dn) for dn in downs]

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for _ in range(a.steps):
        one()
    for dn in downs:
        comp.wait_stream(dn)  # the last step's results are on the host
    e1.record(comp)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": st.global_batch / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "h2d_gb_per_s": h2d / (ms * 1e-3) / 1e9, "d2h_gb_per_s": d2h / (ms * 1e-3) / 1e9,
            "path": "C ABI (cct_conv_fwd_cached / cct_conv_bwd) on double-buffered device buffers: pinned-host "
                    f"H2D of x, dy{' (write-combined)' if a.h2d_wc else ''} and D2H of y, dx, dW on {ncs} + {ncs} "
                    "copy streams overlapping compute"}


if __name__ == "__main__":
    if os.environ.get("CCT_BENCH_WATCHDOG"):  # diagnostics: dump the Python stacks after N s
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["CCT_BENCH_WATCHDOG"]), repeat=True)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
