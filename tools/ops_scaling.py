#!/usr/bin/env python
"""Attention launch time against the number of ops per CTA (budget rho varied): the
intercept of T = a + b * ops estimates the per-CTA fixed cost (COMP=none: kept blocks
only, so the centroid / first-order ops' own costs cannot leak into the intercept) (prologue: op list, barrier
init, TMEM allocation, first loads; epilogue: O read-out and store) that the co-resident
CTA does not hide.  CFG=cogvideox5b python tools/ops_scaling.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402

name = os.environ.get("CFG", "cogvideox5b")
c = synth.CONFIGS[name]
B, S, H, D = c["B"], c["S"], c["H"], c["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
rows = []
for rho in [float(x) for x in os.environ.get("RHOS", "0.02 0.05 0.1 0.15 0.25 0.4").split()]:
    bud = P.Budget()
    z = torch.zeros(64, device="cuda")
    bud(z, z, z, T=50, step=25, rho_table=[rho] * 50)
    comp = os.environ.get("COMP", "grouped")
    r = P.Route(B, S, H, D, P.RouteCfg(Bq=c["Bq"], G=c["G"], comp=comp))
    r(q, k, bud, 1, 25)
    rd = r.read()
    kk = rd["k"]
    NK, W = r.NK, (r.NK + 31) // 32
    # ops per (head, q-block): k kept + centroid chunks with a dropped block + groups with one
    mask = rd["mask"].reshape(-1, W)
    bits = np.unpackbits(mask.view(np.uint8), axis=1, bitorder="little")[:, :NK].astype(bool)
    dropped = ~bits
    nch = (NK + 63) // 64
    c_ops = sum(dropped[:, 64 * j:64 * (j + 1)].any(1) for j in range(nch))
    G = c["G"]
    f_ops = sum(dropped[:, G * g:G * (g + 1)].any(1) for g in range((NK + G - 1) // G))
    if comp == "none":
        c_ops = f_ops = 0
    elif comp == "zeroth":
        f_ops = 0
    ops = float(np.mean(kk + c_ops + f_ops))
    out = P.attn(q, k, v, r, stats_only=True)
    for _ in range(3):
        P.attn(q, k, v, r, out, reuse_stats=True)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            P.attn(q, k, v, r, out, reuse_stats=True)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10)
    rows.append((rho, kk, ops, best))
    print(f"{name} rho {rho:.2f} k {kk} ops/CTA {ops:.1f} attn {best:.4f} ms", flush=True)
x = np.array([r[2] for r in rows]); y = np.array([r[3] for r in rows])
b, a = np.polyfit(x, y, 1)
n_cta = B * H * ((S + c["Bq"] - 1) // c["Bq"])
waves = n_cta / (2 * 148)
print(f"fit: T = {a:.4f} ms + {b * 1e3:.3f} us x ops  ->  fixed {a / waves * 1e3:.2f} us per CTA-pair "
      f"wave ({waves:.1f} waves of 296 CTAs); at the config's rho the fixed share is "
      f"{a / y[np.argmin(abs(np.array([r[0] for r in rows]) - c['rho']))]:.1%}")
