"""CPU: the automatic lowering optimizer against measured B200 data.

profiles/r02/sweep_lowering_types_b256_r2final.jsonl holds one training step (fwd + bwd)
per lowering type, measured on a B200 for BASELINE configs[1] (n=13, k=3, pad 1,
b=256, d*o = 2^16 / 2^17, d/o in [1/16, 16]) plus the CaffeNet conv2-5 shapes
(tools/sweep.py).  SPEC.md:499 (acceptance 3): the model's winner must match the
measured winner at the extreme ratios; here it must match everywhere within 5%.
"""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SWEEP = os.path.join(ROOT, "profiles", "r02", "sweep_lowering_types_b256_r2final.jsonl")


def rows():
    return [json.loads(l) for l in open(SWEEP)]


@pytest.mark.parametrize("r", rows(), ids=lambda r: f"d{r['d']}_o{r['o']}_n{r['n']}")
def test_model_picks_measured_winner(cct, r):
    desc = cct.ConvDesc(r["n"], r["k"], r["d"], r["o"], r["b"], r["stride"], r["pad"])
    choice, est = cct.select_lowering(desc, 3)
    meas = {int(t): v["ms"] for t, v in r["types"].items()}
    best = min(meas, key=meas.get)
    assert meas[choice] <= 1.05 * meas[best], (choice, best, meas)
    if r["d"] / r["o"] >= 8 or r["d"] / r["o"] <= 1 / 8:
        # the winner must match at the extreme ratios -- unless the measured
        # runner-up is within 3% of the winner, i.e. a tie at run-to-run noise (~1.5%)
        runner_up = sorted(meas.values())[1]
        assert choice == best or runner_up <= 1.03 * meas[best], (choice, best, meas)


def test_model_time_calibrated(cct):
    ratios = []
    for r in rows():
        desc = cct.ConvDesc(r["n"], r["k"], r["d"], r["o"], r["b"], r["stride"], r["pad"])
        _, est = cct.select_lowering(desc, 3)
        for t in (1, 2, 3):
            ratios.append(est[t - 1].model_seconds * 1e3 / r["types"][str(t)]["ms"])
    ratios.sort()
    assert 0.8 < ratios[len(ratios) // 2] < 1.25
    assert ratios[0] > 0.6 and ratios[-1] < 1.6


def test_ratio_crossover_direction(cct):
    """Appendix A's trend: the lifting-heavy types gain on Type 1 as d/o grows.  On B200 with
    the implicit (TMA im2col) Type 1 path, Type 1 still wins at d/o = 16 in the configs[1]
    sweep (measured, profiles/r02) -- the crossover moved past the sweep -- so the model must
    show the trend, not a flip: the best lifting type's time relative to Type 1 falls from
    d/o = 1/16 to d/o = 16."""
    def rel(d, o):
        _, est = cct.select_lowering(cct.ConvDesc(13, 3, d, o, 256, 1, 1), 3)
        return min(est[1].model_seconds, est[2].model_seconds) / est[0].model_seconds
    lo, hi = rel(64, 1024), rel(1024, 64)
    assert lo > 1.3 and hi < 1.15 and hi < lo  # measured (r2final sweep): 1.56 and 1.05


def test_fused_conv1_passes_modelled(cct):
    """CaffeNet conv1 (b = 256) runs the fused small-channel kernels (gather forward /
    backward-weight, hfold backward-data); the model prices those passes within 25 % of
    their B200 times (profiles/r02: forward 0.33, backward-data 0.45, backward-weight
    0.31 ms) and picks Type 1."""
    desc = cct.ConvDesc(227, 11, 3, 96, 256, 4, 0)
    for p, ms in ((0, 0.33), (1, 0.45), (2, 0.31)):
        choice, est = cct.select_lowering(desc, p)
        assert choice == 1
        assert 0.75 < est[0].model_seconds * 1e3 / ms < 1.25, (p, est[0].model_seconds)
