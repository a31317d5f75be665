#!/usr/bin/env python
"""Time pasa_route on one config (CFG, default Wan-14B) with and without the Gumbel
bias (beta 0.1 / 0); PASA_LIB selects a library build for A/B runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402

name = os.environ.get("CFG", "wan14b_720p")
c = synth.CONFIGS[name]
B, S, H, D = c["B"], c["S"], c["H"], c["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
b = P.Budget()
z = torch.zeros(64, device="cuda")
b(z, z, z, T=50, step=25, rho_table=[c["rho"]] * 50)
for beta in (0.1, 0.0):
    r = P.Route(B, S, H, D, P.RouteCfg(Bq=c["Bq"], G=c["G"], beta=beta))
    for _ in range(3):
        r(q, k, b, 7, 25)
    best = 1e9
    for _ in range(int(os.environ.get("REPS", "5"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            r(q, k, b, 7, 25)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10)
    print(f"{name} {os.path.basename(os.environ.get('PASA_LIB', 'in-tree'))} chunks {os.environ.get('PASA_ROUTE_CHUNKS', 'auto')} beta {beta} "
          f"route ms (min) {best:.3f}", flush=True)
