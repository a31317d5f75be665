"""Offline budget calibration, Eqs. 9-11.

Records the l-curve of N calibration trajectories with ``pasa_budget`` on the
GPU (one reduction per step), then turns the curves into the per-step density
table with ``pasa_calibrate`` (native, include/pasa.h): pointwise mean over
trajectories (R-19), l-bar over the sparse steps (Eq. 9), alpha_t (Eq. 10),
rho_t = min(rho alpha_t, rho_max) (Eq. 11, R-18), dense prefix = 1 (R-15).
The table feeds ``pasa_schedule.rho_table`` (``Budget(..., rho_table=...)``).

Signals:
* ``velocity`` (default, the paper's offline signal):
  l_t = mean |v_t - v_{t-1}| of adjacent velocity predictions;
* ``latent`` (the online reading R-16): l_t from three consecutive latents,
  mean |v_{t-1} - v_{t-2}| with v = (x_{t+1} - x_t) / h.

Trajectories: the seeded three-phase synthetic trajectory (``synth.ThreePhase``,
seeds 0..N-1, at a config's latent shape), or dumped velocity predictions
(``--noise-pred f1.npy f2.npy ...``, each [T, ...]).

    python -m paper_2604_12219_b200.calibrate --config cogvideox5b --trajectories 10 \\
        --out calib.json [--csv calib.csv]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _C
from .api import Budget


def calibrate(curves, *, rho=0.15, dense_frac=0.2, rho_max=1.0) -> dict:
    """pasa_calibrate on l-curves [N, T] (host arrays).  Returns dict(rho_table,
    alpha, clipped, l1_mean)."""
    c = np.ascontiguousarray(np.atleast_2d(np.asarray(curves, dtype=np.float64)))
    N, T = c.shape
    tab, alpha = np.zeros(T), np.zeros(T)
    clipped = np.zeros(T, dtype=np.int32)
    lbar = ctypes.c_double()
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    _C.check(_C.lib().pasa_calibrate(P(c), N, T, rho, dense_frac, rho_max, P(tab), P(alpha),
                                     P(clipped), ctypes.byref(lbar)), "pasa_calibrate")
    return dict(rho_table=tab, alpha=alpha, clipped=clipped.astype(bool), l1_mean=lbar.value)


def _l1(budget: Budget, a, b, c=None, *, T, step, h=1.0):
    kind = "velocity" if c is None else "latent"
    budget(a, b, c, T=T, step=step, h_t=h, h_tm1=h, l1_mean=1.0, kind=kind)
    return budget.read()["l1"]


def curve_from_velocities(vs: Iterable[torch.Tensor], T: int, budget: Budget) -> np.ndarray:
    """l_t = mean |v_t - v_{t-1}| for t >= 1 (l_0 = NaN), v_t on the device."""
    out = np.full(T, np.nan)
    prev = None
    for t, v in enumerate(vs):
        if t >= T:
            break
        v = v.contiguous()
        if prev is not None:
            out[t] = _l1(budget, v, prev, T=T, step=t)
        prev = v
    return out


def curve_from_latents(xs: Iterable[torch.Tensor], T: int, budget: Budget) -> np.ndarray:
    """Online reading R-16: l_t from (x_t, x_{t-1}, x_{t-2}), t >= 2, h = 1/T."""
    out = np.full(T, np.nan)
    hist: list = []
    for t, x in enumerate(xs):
        if t >= T:
            break
        hist = (hist + [x.contiguous()])[-3:]
        if t >= 2:
            out[t] = _l1(budget, hist[2], hist[1], hist[0], T=T, step=t, h=1.0 / T)
    return out


def synthetic_velocities(shape: Sequence[int], T: int, seed: int, device):
    """v_t = (x_{t+1} - x_t) * T of the seeded three-phase trajectory."""
    import synth
    xs = synth.ThreePhase(shape=tuple(shape), T=T, seed=seed, device=device).trajectory()
    prev = next(xs)
    for x in xs:
        yield (x - prev) * T
        prev = x


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--config", default="cogvideox5b")
    ap.add_argument("--trajectories", type=int, default=10)
    ap.add_argument("--T", type=int, default=50)
    ap.add_argument("--rho", type=float, default=0.15)
    ap.add_argument("--dense-frac", type=float, default=0.2)
    ap.add_argument("--rho-max", type=float, default=1.0)
    ap.add_argument("--signal", default="velocity", choices=["velocity", "latent"])
    ap.add_argument("--noise-pred", nargs="*", default=None,
                    help=".npy files of dumped velocity predictions, each [T, ...]")
    ap.add_argument("--out", default=None)
    ap.add_argument("--csv", default=None)
    a = ap.parse_args(argv)
    dev = torch.device("cuda")
    budget = Budget(dev)
    curves = []
    if a.noise_pred:
        for f in a.noise_pred:
            arr = np.load(f)
            vs = (torch.from_numpy(np.ascontiguousarray(arr[t])).float().to(dev)
                  for t in range(arr.shape[0]))
            curves.append(curve_from_velocities(vs, a.T, budget))
        source = {"noise_pred": a.noise_pred}
    else:
        import synth
        shape = synth.CONFIGS[a.config]["latent"]
        for seed in range(a.trajectories):
            if a.signal == "velocity":
                curves.append(curve_from_velocities(synthetic_velocities(shape, a.T, seed, dev),
                                                    a.T, budget))
            else:
                xs = synth.ThreePhase(shape=tuple(shape), T=a.T, seed=seed, device=dev)
                curves.append(curve_from_latents(xs.trajectory(), a.T, budget))
        source = {"synthetic": "three-phase (synth.ThreePhase)", "config": a.config,
                  "latent_shape": list(shape), "seeds": list(range(a.trajectories))}
    curves = np.stack(curves)
    res = calibrate(curves, rho=a.rho, dense_frac=a.dense_frac, rho_max=a.rho_max)
    D = max(int(math.floor(a.dense_frac * a.T + 0.5)), 2)
    doc = {
        "what": "PASA offline budget calibration, Eqs. 9-11 (PAPER.md:276-294)",
        "signal": a.signal, "source": source, "T": a.T, "rho": a.rho,
        "dense_frac": a.dense_frac, "rho_max": a.rho_max, "n_trajectories": int(curves.shape[0]),
        "l1_mean": res["l1_mean"], "rho_table": res["rho_table"].tolist(),
        "alpha": res["alpha"].tolist(), "clipped": res["clipped"].tolist(),
        "sum_rho_sparse": float(res["rho_table"][D:].sum()), "n_sparse": a.T - D,
        "l1_curves": [[None if not np.isfinite(x) else float(x) for x in c] for c in curves],
    }
    text = json.dumps(doc, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        print(text)
    if a.csv:
        with open(a.csv, "w") as f:
            f.write("t,l1_mean_curve,alpha,rho_t,clipped\n")
            fin = np.isfinite(curves)
            lavg = np.where(fin.any(axis=0),
                            np.where(fin, curves, 0.0).sum(axis=0) / np.maximum(fin.sum(axis=0), 1),
                            np.nan)
            for t in range(a.T):
                f.write(f"{t},{lavg[t]},{res['alpha'][t]},{res['rho_table'][t]},"
                        f"{int(res['clipped'][t])}\n")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
