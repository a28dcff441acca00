"""PCIe copy-rate probe for the e2e leg: H2D alone, D2H alone and both directions at once from
pinned host buffers allocated while the process is bound to each NUMA node in turn (page-locked
pages are placed on the allocating thread's node), so the e2e host buffers can be put on the
node the GPU hangs off.  Prints one JSON line per (node, mode).

    gpurun -- 'python tools/pcie_probe.py'
"""
import glob
import json
import os
import subprocess

import torch


def nodes():
    out = {}
    for d in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        cpus = []
        for part in open(os.path.join(d, "cpulist")).read().strip().split(","):
            if not part:
                continue
            a, _, b = part.partition("-")
            cpus += list(range(int(a), int(b or a) + 1))
        if cpus:
            out[int(d.rsplit("node", 1)[1])] = cpus
    return out


def gpu_node():
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(
        torch.cuda.get_device_properties(0), "pci_bus_id") else None
    try:
        q = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                           capture_output=True, text=True).stdout.split()[0]
        dom, rest = q.lower().split(":", 1)
        path = f"/sys/bus/pci/devices/{dom[-4:]}:{rest}/numa_node"
        return int(open(path).read()), q
    except Exception as e:  # noqa: BLE001
        return None, f"{bus} {e}"


def rate(mode, host_src, host_dst, dev_src, dev_dst, iters=5):
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    for it in range(iters + 1):
        if it == 1:
            ev[0].record()
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1):
                dev_dst.copy_(host_src, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2):
                host_dst.copy_(dev_src, non_blocking=True)
    cur = torch.cuda.current_stream()
    cur.wait_stream(s1)
    cur.wait_stream(s2)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    return host_src.numel() * 4 * iters / (ms * 1e-3) / 1e9


def main():
    nb = 256 << 20  # floats: 1 GiB per buffer
    dev_src = torch.empty(nb, device="cuda")
    dev_dst = torch.empty(nb, device="cuda")
    gn, bus = gpu_node()
    print(json.dumps({"gpu_bus": bus, "gpu_numa_node": gn, "nodes": {k: f"{v[0]}-{v[-1]} ({len(v)})"
                                                                     for k, v in nodes().items()}}), flush=True)
    allc = sorted(os.sched_getaffinity(0))
    for node, cpus in list(nodes().items()) + [("all", allc)]:
        os.sched_setaffinity(0, set(cpus) & set(allc) or set(allc))
        hs = torch.empty(nb, pin_memory=True)
        hd = torch.empty(nb, pin_memory=True)
        hs.uniform_()
        hd.zero_()
        r = {m: round(rate(m, hs, hd, dev_src, dev_dst), 2) for m in ("h2d", "d2h", "both")}
        print(json.dumps({"node": node, "gb_per_s_each": r}), flush=True)
        del hs, hd
        torch.cuda.synchronize()
    os.sched_setaffinity(0, set(allc))


if __name__ == "__main__":
    main()
