#!/usr/bin/env python
"""Time pasa_route at Wan-14B with and without the Gumbel bias (beta 0.1 / 0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_2604_12219_b200 as P
c = synth.CONFIGS["wan14b_720p"]
q, k, v = synth.iid_qkv(1, c["S"], 40, 128, seed=1, dtype=torch.bfloat16, device="cuda")
b = P.Budget(); z = torch.zeros(64, device="cuda"); b(z, z, z, T=50, step=25, rho_table=[0.15] * 50)
for beta in (0.1, 0.0):
    r = P.Route(1, c["S"], 40, 128, P.RouteCfg(Bq=128, G=32, beta=beta))
    for _ in range(3): r(q, k, b, 7, 25)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): r(q, k, b, 7, 25)
    e1.record(); torch.cuda.synchronize()
    print("beta", beta, "route ms", e0.elapsed_time(e1) / 10)
