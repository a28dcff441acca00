"""CPU: the bench's reference arm is independent of the product.

``bench.py --impl reference`` times the reference's own CPU path on the same
workload as the B200 arm; it must not import the package or map libcct.so
(the driver records which shared objects each arm loaded), and its per-layer
geometry / lowering list must be the ones the B200 arm runs.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_geometry_and_types_match_the_b200_arm():
    import bench
    from paper_1504_04343_b200 import select_lowering
    from paper_1504_04343_b200.stack import CAFFENET
    assert tuple((l.name, l.n, l.k, l.d, l.o, l.stride, l.pad) for l in CAFFENET) == bench.CAFFENET_GEOM
    assert tuple(select_lowering(l.desc(256), 3)[0] for l in CAFFENET) == bench.REF_TYPES
    gflop = sum(3 * l.desc(1).flops_per_pass() for l in CAFFENET) / 1e9
    assert abs(gflop - bench.STACK_GFLOP_PER_IMAGE) < 1e-3


PROBE = r"""
import os, sys, json
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-sample", "1"]
sys.path.insert(0, os.environ["ROOT"])
import bench
bench.run_reference(bench.parse())
maps = open("/proc/self/maps").read()
print(json.dumps({"pkg": any(m.startswith("paper_1504_04343_b200") for m in sys.modules),
                  "libcct": "libcct.so" in maps, "torch": "torch" in sys.modules}))
"""


def test_reference_arm_never_loads_the_product():
    r = subprocess.run([sys.executable, "-c", PROBE], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, ROOT=ROOT), cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.strip().splitlines()]
    bench_line, probe = lines[0], lines[-1]
    assert bench_line["impl"] == "reference" and bench_line["value"] > 0
    assert bench_line["cpu_baseline"]["kind"] in ("reference", "port")
    assert bench_line["config"]["workload"].startswith("caffenet conv1-5")
    assert probe == {"pkg": False, "libcct": False, "torch": False}
    # the same config the B200 arm prints for the same flags (the driver's same-config check);
    # the bounded CPU sample is described in cpu_baseline, not in config
    import argparse
    import bench
    a = argparse.Namespace(layout="nhwc", tune="")
    assert bench_line["config"] == json.loads(json.dumps(bench.workload_config(a, 1, 256, 256, list(bench.REF_TYPES))))
    assert "1 of the workload's images" in bench_line["cpu_baseline"]["sample"]
