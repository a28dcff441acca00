"""convbench -- the SPEC's bench-cli harness (acceptance 7 and 9).

CPU tests: the planning / simulation commands (schedule, estimate), the record
formats (CSV / JSON schema twins), the exit-code contract and the line-numbered
configuration errors.  GPU tests: verify / sweeps on the device path.
"""
import csv
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1504_04343_b200", "_lib", "convbench")
DATA = os.path.join(ROOT, "paper_1504_04343_b200", "data")
LAYERS = os.path.join(DATA, "caffenet.layers")
DEVICES = os.path.join(DATA, "hybrid.devices")


def run(*args, check_rc=None):
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    if check_rc is not None:
        assert p.returncode == check_rc, (p.returncode, p.stderr[-2000:])
    return p


def records(fmt, *args):
    out = run(*args, "--format", fmt, check_rc=0).stdout
    if fmt == "json":
        return json.loads(out)
    return list(csv.DictReader(io.StringIO(out)))


def test_help_lists_every_command():
    out = run("--help", check_rc=0).stdout
    for cmd in ("verify", "sweep-ratio", "sweep-batch", "sweep-partitions", "schedule", "estimate"):
        assert cmd in out


def test_schedule_proportional_third(tmp_path):
    """CPU 1 TFLOPS + GPU 2 TFLOPS -> 1/3 of the input to the CPU (section 2.3)."""
    recs = records("json", "schedule", "--devices", DEVICES, "--layers", LAYERS, "--layer", "conv2",
                   "--granularity", "30")
    prop = {r["device"]: r for r in recs if r["kind"] == "proportional"}
    assert abs(prop["cpu"]["fraction"] - 1 / 3) < 1e-9 and abs(prop["gpu"]["fraction"] - 2 / 3) < 1e-9
    assert prop["cpu"]["p"] + prop["gpu"]["p"] == 8
    opt = [r for r in recs if r["kind"] == "sweep-optimum"][0]
    assert 1.0 <= opt["gap"] <= 1.01  # zero overheads: proportional is optimal
    curve = [r for r in recs if r["kind"] == "curve"]
    assert len(curve) == 31
    spans = [r["makespan_s"] for r in curve]
    i = spans.index(min(spans))
    assert all(spans[j] >= spans[j + 1] for j in range(i)) and all(spans[j] <= spans[j + 1] for j in range(i, 30))


def test_schedule_single_device_degenerate(tmp_path):
    f = tmp_path / "one.devices"
    f.write_text("gpu 2.0e15 0\n")
    recs = records("json", "schedule", "--devices", str(f), "--template", "13 3 256 384 64 1 1")
    assert recs[0]["fraction"] == 1 and recs[0]["p"] == 64
    assert [r for r in recs if r["kind"] == "gap"][0]["gap"] == 1


def test_schedule_gap_audit_1000():
    """SPEC acceptance 7: 1000 seeded 2-device profiles, overheads <= 5% of the work
    time: the proportional heuristic stays within 5% of the optimum."""
    recs = records("json", "schedule", "--devices", DEVICES, "--layers", LAYERS, "--layer", "conv3",
                   "--granularity", "100", "--audit", "1000")
    audit = [r for r in recs if r["kind"] == "audit"][0]
    assert audit["passed"] == "true" and 1.0 <= audit["gap"] <= 1.05 and audit["reps"] == 1000


def test_csv_json_schema_twins():
    """CSV and JSON emissions carry identical data and field names."""
    args = ("schedule", "--devices", DEVICES, "--layers", LAYERS, "--layer", "conv1", "--granularity", "10")
    rj = records("json", *args)
    rc = records("csv", *args)
    assert len(rj) == len(rc) and list(rj[0].keys()) == list(rc[0].keys())
    for a, b in zip(rj, rc):
        for k, v in a.items():
            if v is None:
                assert b[k] == ""
            elif isinstance(v, str):
                assert b[k] == v
            else:
                assert float(b[k]) == pytest.approx(float(v), rel=1e-12, abs=0)


def test_estimate_records_every_strategy():
    recs = records("json", "estimate", "--layers", LAYERS)
    assert len(recs) == 15
    conv2 = [r for r in recs if r["layer"] == "conv2"]
    assert {r["strategy"] for r in conv2} == {1, 2, 3}
    # SPEC footprints: Type3 < Type2 < Type1 lowered bytes for k >= 2
    fp = {r["strategy"]: r["footprint_bytes"] for r in conv2}
    assert fp[3] < fp[2] < fp[1]


@pytest.mark.parametrize("content,line", [("conv1 227 11 3 96 8 4 0\nbad 13 3 x 4 1\n", 2),
                                          ("# c\n\na 5 3 2 1\n", 3),
                                          ("a 5 3 2 1 1\na 5 3 2 1 1\n", 2),
                                          ("a 5 9 2 1 1\n", 1)])
def test_malformed_layer_file_is_config_error_with_line(tmp_path, content, line):
    f = tmp_path / "bad.layers"
    f.write_text(content)
    p = run("estimate", "--layers", str(f), check_rc=2)
    assert f"bad.layers:{line}" in p.stderr


def test_malformed_device_file_is_config_error_with_line(tmp_path):
    f = tmp_path / "bad.devices"
    f.write_text("cpu 1e12 0\ngpu fast 0\n")
    p = run("schedule", "--devices", str(f), "--template", "13 3 8 8 4", check_rc=2)
    assert "bad.devices:2" in p.stderr


def test_bad_flags_are_config_errors():
    run("estimate", "--layers", LAYERS, "--bogus", "1", check_rc=2)
    run("estimate", "--layers", LAYERS, "--format", "xml", check_rc=2)
    run("frobnicate", check_rc=2)
    run("estimate", "--layers", "/nonexistent.layers", check_rc=2)


# ----------------------------------------------------------------- GPU path
@pytest.mark.gpu
def test_verify_default_layer_file_passes():
    """SPEC acceptance 9: verify exits 0 on the shipped layer file (all strategies,
    forward vs the exact fp64 oracle, backward through the adjoint identity)."""
    recs = records("json", "verify", "--layers", LAYERS)
    assert len(recs) == 15 and all(r["passed"] == "true" for r in recs)
    assert max(r["rel_l2"] for r in recs) <= 1e-4 and max(r["adjoint_err"] for r in recs) <= 1e-4


@pytest.mark.gpu
def test_verify_tolerance_zero_fails_k1_passes_tight(tmp_path):
    p = run("verify", "--layers", LAYERS, "--batch", "2", "--strategy", "1", "--tolerance", "0")
    assert p.returncode == 1
    f = tmp_path / "k1.layers"
    f.write_text("pointwise 12 1 8 16 2\n")
    recs = records("json", "verify", "--layers", str(f), "--tolerance", "1e-6")
    assert all(r["passed"] == "true" for r in recs)


@pytest.mark.gpu
def test_sweep_ratio_single_step_one_record_per_strategy():
    recs = records("json", "sweep-ratio", "--template", "13 3 64 64 8 1 1", "--ratio-range", "1:1:1", "--reps", "2")
    assert sorted(r["strategy"] for r in recs) == [1, 2, 3]
    assert len({r["measured_winner"] for r in recs}) == 1 and len({r["model_winner"] for r in recs}) == 1
    assert all(r["total_s"] > 0 and r["images_per_s"] > 0 for r in recs)


@pytest.mark.gpu
def test_sweep_batch_direction():
    """Fig. 2(b) direction: batched lowering beats per-image lowering in throughput."""
    recs = records("json", "sweep-batch", "--layers", LAYERS, "--layer", "conv2", "--batch", "1,64",
                   "--strategy", "1", "--reps", "3")
    tp = {r["b"]: r["images_per_s"] for r in recs}
    assert tp[64] >= 1.5 * tp[1]


@pytest.mark.gpu
def test_sweep_partitions_none_and_p():
    recs = records("json", "sweep-partitions", "--layers", LAYERS, "--layer", "conv3", "--partitions",
                   "none,1,2,4", "--strategy", "1", "--reps", "2", "--threads", "4")
    kinds = [(r["kind"], r["p"]) for r in recs]
    assert kinds == [("none", 8), ("partitioned", 1), ("partitioned", 2), ("partitioned", 4)]
    # footprint: p partitions of b/p images -> the same total lowered bytes
    fps = [r["footprint_bytes"] for r in recs[1:]]
    assert fps[0] == fps[1] == fps[2]
