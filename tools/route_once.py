#!/usr/bin/env python
"""One pasa_route call at a BASELINE config (CFG, BETA env) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402

c = synth.CONFIGS[os.environ.get("CFG", "wan14b_720p")]
B, S, H, D = c["B"], c["S"], c["H"], c["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
b = P.Budget()
z = torch.zeros(64, device="cuda")
b(z, z, z, T=50, step=25, rho_table=[c["rho"]] * 50)
r = P.Route(B, S, H, D, P.RouteCfg(Bq=c["Bq"], G=c["G"], beta=float(os.environ.get("BETA", "0.1"))))
for _ in range(int(os.environ.get("N", "2"))):
    r(q, k, b, 7, 25)
torch.cuda.synchronize()
