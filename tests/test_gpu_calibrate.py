"""GPU l-curves of the calibration tool (pasa_budget per step, SURVEY.md §8f
NEXT 2) against the oracle on the same synthetic trajectories: l_t relative
error <= 1e-12 (fixed-grid fp64 tree vs sequential sum), and the resulting table
equals the oracle's table within 1e-12 relative.  Also runs the CLI once."""
import json

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

SHAPE = (4, 5, 12, 16)
T = 50


@pytest.fixture(scope="module")
def cal():
    from paper_2604_12219_b200 import build
    build.build()
    from paper_2604_12219_b200 import calibrate as C
    return C


def _oracle_curve_velocity(seed):
    xs = list(synth.ThreePhase(shape=SHAPE, T=T, seed=seed, device="cuda").trajectory())
    vs = [((xs[t + 1] - xs[t]) * T) for t in range(T)]
    out = np.full(T, np.nan)
    for t in range(1, T):
        out[t] = oracle.l1(vs[t], vs[t - 1], kind=1)
    return out


def _oracle_curve_latent(seed):
    xs = list(synth.ThreePhase(shape=SHAPE, T=T, seed=seed, device="cuda").trajectory())
    out = np.full(T, np.nan)
    for t in range(2, T):
        out[t] = oracle.l1(xs[t], xs[t - 1], xs[t - 2], kind=0, h_t=1.0 / T, h_tm1=1.0 / T)
    return out


@pytest.mark.parametrize("signal", ["velocity", "latent"])
def test_curves_and_table_match_oracle(cal, signal):
    from paper_2604_12219_b200 import Budget
    b = Budget()
    got, want = [], []
    for seed in range(3):
        if signal == "velocity":
            got.append(cal.curve_from_velocities(cal.synthetic_velocities(SHAPE, T, seed, "cuda"),
                                                 T, b))
            want.append(_oracle_curve_velocity(seed))
        else:
            xs = synth.ThreePhase(shape=SHAPE, T=T, seed=seed, device="cuda").trajectory()
            got.append(cal.curve_from_latents(xs, T, b))
            want.append(_oracle_curve_latent(seed))
    got, want = np.stack(got), np.stack(want)
    first = 1 if signal == "velocity" else 2
    assert np.all(np.isnan(got[:, :first]))
    rel = np.abs(got[:, first:] - want[:, first:]) / np.abs(want[:, first:])
    assert rel.max() <= 1e-12, rel.max()
    a = cal.calibrate(got, rho=0.15)
    w = oracle.calibrate(want, rho=0.15)
    assert np.allclose(a["rho_table"], w["rho_table"], rtol=1e-12, atol=0)
    assert a["l1_mean"] == pytest.approx(w["l1_mean"], rel=1e-12)
    # three-phase shape: early and late steps get more budget
    assert a["rho_table"][10] > 0.15 > a["rho_table"][30] and a["rho_table"][47] > 0.15


def test_cli_writes_table(cal, tmp_path):
    out = tmp_path / "calib.json"
    csv = tmp_path / "calib.csv"
    assert cal.main(["--config", "tiny", "--trajectories", "2", "--out", str(out),
                     "--csv", str(csv)]) == 0
    doc = json.loads(out.read_text())
    assert len(doc["rho_table"]) == 50 and doc["n_trajectories"] == 2
    assert doc["sum_rho_sparse"] == pytest.approx(0.15 * doc["n_sparse"], rel=1e-9) or \
        any(doc["clipped"])
    assert csv.read_text().count("\n") == 51
