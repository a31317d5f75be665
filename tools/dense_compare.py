#!/usr/bin/env python
"""One launch of either PASA's attention kernel (MODE=pasa, the bench's Wan-14B launch) or
torch's dense SDPA (MODE=dense, DENSE_HEADS heads of the same tensors: 8 heads of Wan-14B
is 23.4 TFLOP, the PASA launch's 23.0) after warm-up, for a side-by-side ncu capture:
    ncu --set full -c 1 -s <warm-up launches> ... python tools/dense_compare.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

cfg = synth.CONFIGS[os.environ.get("CFG", "wan14b_720p")]
B, S, H, D = cfg["B"], cfg["S"], cfg["H"], cfg["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
if os.environ.get("MODE", "dense") == "dense":
    n = int(os.environ.get("DENSE_HEADS", "8"))
    qd, kd, vd = (t[:, :, :n].transpose(1, 2).contiguous() for t in (q, k, v))
    del q, k, v
    for _ in range(3):
        torch.nn.functional.scaled_dot_product_attention(qd, kd, vd)
else:
    import paper_2604_12219_b200 as P
    bud = P.Budget()
    z = torch.zeros(64, device="cuda")
    bud(z, z, z, T=50, step=25, rho_table=[cfg["rho"]] * 50)
    r = P.Route(B, S, H, D, P.RouteCfg(Bq=cfg["Bq"], G=cfg["G"]))
    r(q, k, bud, 1, 25)
    out = P.attn(q, k, v, r, stats_only=True)
    for _ in range(3):
        P.attn(q, k, v, r, out, reuse_stats=True)
torch.cuda.synchronize()
print("done")
