#!/usr/bin/env python
"""Per-rank work of the head-partitioned multi-GPU run, emulated on one GPU: the bench
step (budget + route + statistics + attention) for H/N heads of a config, N = 1, 2, 4,
8, each head keyed by its global index (head_offset) exactly as rank 0 would run it.
Since ranks share nothing on the hot path, the N-GPU step time is max over ranks of
these per-rank times (plus the launch barrier); the printed efficiency t_1 / (N t_N)
is the strong-scaling efficiency this predicts (the driver measures the real one).
    CFG=wan14b_720p python tools/scaling_emulate.py"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402

name = os.environ.get("CFG", "wan14b_720p")
c = synth.CONFIGS[name]
B, S, H, D = c["B"], c["S"], c["H"], c["D"]
tp = synth.ThreePhase(shape=c["latent"], T=50, seed=7, device="cuda")
x_t, x_tm1, x_tm2 = (x.contiguous() for x in tp.latents(25))
res = {}
for N in (1, 2, 4, 8):
    if H % N:
        continue
    Hl = H // N
    q, k, v = synth.iid_qkv(B, S, Hl, D, seed=1000, dtype=torch.bfloat16, device="cuda")
    cfg = P.RouteCfg(Bq=c["Bq"], G=c["G"], H_total=H, head_offset=0)
    bud = P.Budget()
    route = P.Route(B, S, Hl, D, cfg)
    out = torch.empty_like(q)

    def step():
        bud(x_t, x_tm1, x_tm2, T=50, step=25, rho=c["rho"], l1_mean=tp.expected_l1_mean(),
            h_t=1 / 50, h_tm1=1 / 50, rho_table=[c["rho"]] * 50)
        route(q, k, bud, P.layer_seed(42, 0), 25)
        P.attn(q, k, v, route, out)

    for _ in range(3):
        step()
    xs = []
    for _ in range(int(os.environ.get("REPS", "10"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        xs.append(e0.elapsed_time(e1))
    res[N] = statistics.median(xs)
    del q, k, v, out, route
    torch.cuda.empty_cache()
t1 = res[1]
for N, t in res.items():
    print(f"{name} N={N}: {H // N} heads per rank, step {t:.3f} ms, "
          f"{4.0 * S * S * D * B * H / (t * 1e-3) / 1e12:,.0f} TFLOP/s-equiv whole job, "
          f"predicted strong-scaling efficiency {t1 / (N * t):.3f}", flush=True)
