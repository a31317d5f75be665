"""CPU pins of the oracle's offline calibration, Eqs. 9-11 (
SURVEY.md §8f NEXT 2): per-step l-curves of N trajectories -> pointwise mean
(R-19) -> l-bar over the sparse steps (Eq. 9) -> alpha_t (Eq. 10) -> rho_t with
the clip of R-18 (Eq. 11); dense prefix rho_t = 1 (R-15).

Pins: the SPEC worked schedules (tests/golden/spec_examples.json), Eq. 11's
budget conservation, the constant curve = PISA reduction, scale invariance,
linearity of the trajectory average, and agreement with the per-step budget
oracle run in table-free mode with l-bar taken from the calibration."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
T = 50
D = 10                  # floor(0.2 * 50 + 0.5) dense steps


def _gold():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        return json.load(f)


def _curve(sparse_vals):
    c = np.full(T, np.nan)                       # dense entries are ignored
    c[D:D + len(sparse_vals)] = sparse_vals
    return c


def test_spec_worked_schedules():
    """SPEC.md:406-407 with the sparse steps = the listed l values."""
    for ex in _gold()["schedule"]:
        ls = ex["l"]
        Tn = D + len(ls)
        c = np.full(Tn, np.nan)
        c[D:] = ls
        r = oracle.calibrate(c[None, :], rho=ex["rho"], dense_frac=D / Tn)   # D dense steps
        assert r["l1_mean"] == pytest.approx(sum(ls) / len(ls), rel=1e-15)
        assert np.allclose(r["rho_table"][D:], ex["rho_t"], rtol=1e-15, atol=1e-15), ex["cite"]
        assert r["clipped"][D:].tolist() == ex["clipped"]
        assert np.all(r["rho_table"][:D] == 1.0) and not r["clipped"][:D].any()
        if "alpha" in ex:
            assert np.allclose(r["alpha"][D:], ex["alpha"], rtol=1e-15)


def test_conservation_eq11_and_scale_invariance():
    """sum_{t in T_sparse} rho_t = rho |T_sparse| when nothing clips;
    Eq. 10 is invariant to scaling every curve."""
    rng = np.random.default_rng(0)
    curves = np.stack([_curve(rng.uniform(0.2, 1.0, T - D)) for _ in range(5)])
    a = oracle.calibrate(curves, rho=0.15)
    assert a["rho_table"][D:].sum() == pytest.approx(0.15 * (T - D), rel=1e-12)
    b = oracle.calibrate(curves * 3.25, rho=0.15)
    assert np.allclose(a["rho_table"], b["rho_table"], rtol=1e-13, atol=0)
    assert b["l1_mean"] == pytest.approx(3.25 * a["l1_mean"], rel=1e-13)


def test_constant_curve_is_pisa():
    """a constant l-curve gives alpha = 1 and rho_t = rho."""
    r = oracle.calibrate(_curve(np.full(T - D, 0.375))[None, :], rho=0.15)
    assert np.all(r["alpha"][D:] == 1.0) and np.all(r["rho_table"][D:] == 0.15)


def test_trajectory_average_is_pointwise_mean():
    """R-19: calibrating N curves equals calibrating their pointwise mean."""
    rng = np.random.default_rng(1)
    curves = np.stack([_curve(rng.uniform(0.5, 2.0, T - D)) for _ in range(4)])
    a = oracle.calibrate(curves, rho=0.2)
    b = oracle.calibrate(curves.mean(axis=0)[None, :], rho=0.2)
    assert np.allclose(a["rho_table"], b["rho_table"], rtol=1e-14, atol=0)


def test_clip_and_budget_agree_with_per_step_oracle():
    """The table equals the per-step budget oracle (Eq. 10-11 at step t with
    l1_mean = the calibrated l-bar), including clipped steps (R-18)."""
    rng = np.random.default_rng(2)
    vals = rng.uniform(0.1, 1.0, T - D)
    vals[3] = 25.0                                   # forces a clip at rho = 0.15
    r = oracle.calibrate(_curve(vals)[None, :], rho=0.15)
    assert r["clipped"].sum() == 1
    for t in range(D, T):
        x_t, x_tm1 = np.zeros(8) + vals[t - D], np.zeros(8)
        step = oracle.budget(x_t, x_tm1, kind=1, T=T, step=t, rho=0.15, l1_mean=r["l1_mean"])
        assert step["rho_t"] == pytest.approx(r["rho_table"][t], rel=1e-14)   # l via a mean of 8
        assert step["clipped"] == bool(r["clipped"][t])


def test_rejects_degenerate():
    with pytest.raises(ValueError):
        oracle.calibrate(_curve(np.zeros(T - D))[None, :])       # l-bar = 0
    with pytest.raises(ValueError):
        oracle.calibrate(np.ones((1, 3)), dense_frac=1.0)        # no sparse step
