"""Compensation-mode x group-size sweep: fidelity against
dense attention versus B200 throughput of the PASA path.

For G in {1, 8, 16, 32, 64, >= N_K} and comp in {grouped, zeroth, none} the same
route (pasa_route; the routing does not depend on G or comp) drives pasa_attn;
the output is compared with dense attention (torch SDPA in fp32 on the same bf16
inputs: the measurement reference, not part of the product path) by relative
Frobenius error ||O - O_dense||_F / ||O_dense||_F, and the statistics + attention
kernels are timed with CUDA events.  G = 1 is the per-block first-order
expansion (exact Taylor order, Eq. 5), G >= N_K is PISA's global H-bar (Eq. 6),
G = 32 is PASA.  G = 1 runs on the CUDA-core kernel (per-block first
order: one 128x128x128 product per dropped block), so its timing is not comparable.

Generators: ``correlated`` (strength 1: the first-order term
matters) and ``video`` (smooth latent-grid keys, synth.video_qkv).

    python -m paper_2604_12219_b200.sweep --S 16384 --H 4 --D 128 --seeds 4 --out sweep.json
"""
from __future__ import annotations

import argparse
import json

import numpy as np
import torch

from . import Budget, Route, RouteCfg, attn

GROUPS = [1, 8, 16, 32, 64, "global"]
COMPS = ["grouped", "zeroth", "none"]


def dense_reference(q, k, v):
    """Dense softmax attention in fp32 on the device ([B, S, H, D] layout)."""
    qt, kt, vt = (x.float().transpose(1, 2) for x in (q, k, v))
    o = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt)
    return o.transpose(1, 2)


def rel_fro(a, b):
    return float((a.float() - b).norm() / b.norm())


def run(q, k, v, *, rho=0.15, beta=0.1, seed=42, step=25, reps=5, bq256=False):
    B, S, H, D = q.shape
    NK = (S + 63) // 64
    dense = dense_reference(q, k, v)
    budget = Budget()
    z = torch.zeros(64, device=q.device)
    budget(z, z, z, T=50, step=step, rho_table=[rho] * 50)
    rows = []
    for G in GROUPS:
        g = NK if G == "global" else G
        for comp in COMPS:
            if comp != "grouped" and G != 32:
                continue                      # zeroth / none do not depend on G
            route = Route(B, S, H, D, RouteCfg(Bq=128, G=g, comp=comp, beta=beta))
            route(q, k, budget, seed, step)
            out = attn(q, k, v, route)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                attn(q, k, v, route, out)
            e1.record()
            torch.cuda.synchronize()
            rows.append({"G": G, "comp": comp, "rel_frobenius": rel_fro(out, dense),
                         "attn_ms": e0.elapsed_time(e1) / reps,
                         "kernel": "tcgen05" if g in (8, 16, 32, 64) or g % 128 == 0 or g >= NK
                         else "cuda-core"})
    if bq256:
        # routing granularity (NEXT 4 / reading R-29): one kept set per 256 queries
        for comp in COMPS:
            route = Route(B, S, H, D, RouteCfg(Bq=256, G=32, comp=comp, beta=beta))
            route(q, k, budget, seed, step)
            out = attn(q, k, v, route)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                attn(q, k, v, route, out)
            e1.record()
            torch.cuda.synchronize()
            rows.append({"G": 32, "comp": comp, "Bq": 256, "rel_frobenius": rel_fro(out, dense),
                         "attn_ms": e0.elapsed_time(e1) / reps, "kernel": "tcgen05 (Bq 256)"})
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--S", type=int, default=16384)
    ap.add_argument("--H", type=int, default=4)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--rho", type=float, default=0.15)
    ap.add_argument("--seeds", type=int, default=4)
    ap.add_argument("--generator", default="correlated", choices=["correlated", "video"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--bq256", action="store_true",
                    help="also route at Bq = 256 (G = 32, all three modes)")
    a = ap.parse_args(argv)
    import synth
    per_seed = []
    for seed in range(a.seeds):
        if a.generator == "correlated":
            q, k, v = synth.correlated_qkv(1, a.S, a.H, a.D, seed=seed, device="cuda")
        else:
            F = max(1, a.S // (32 * 32))
            q, k, v = synth.video_qkv(1, (F, 32, a.S // (32 * F)), a.H, a.D, seed=seed,
                                      device="cuda")
        per_seed.append(run(q, k, v, rho=a.rho, bq256=a.bq256))
    table = []
    for n, r in enumerate(per_seed[0]):
        errs = [ps[n]["rel_frobenius"] for ps in per_seed]
        ms = [ps[n]["attn_ms"] for ps in per_seed]
        table.append({"G": r["G"], "comp": r["comp"], "Bq": r.get("Bq", 128), "kernel": r["kernel"],
                      "rel_frobenius_mean": float(np.mean(errs)),
                      "rel_frobenius_std": float(np.std(errs)),
                      "attn_ms_median": float(np.median(ms))})
    doc = {"what": "PASA compensation / group-size sweep (SURVEY.md §8f NEXT 3)",
           "generator": a.generator, "S": a.S, "H": a.H, "D": a.D, "rho": a.rho,
           "seeds": a.seeds, "reference": "dense SDPA fp32 on the same bf16 inputs",
           "rows": table}
    text = json.dumps(doc, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    print(text)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
