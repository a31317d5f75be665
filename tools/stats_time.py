#!/usr/bin/env python
"""Time the K/V statistics pass (pasa_attn STATS_ONLY) on one config (CFG); reports
ms (min of REPS) and the achieved HBM bandwidth of the algorithmic bytes
(2 S d 2 B per head read)."""
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
r = P.Route(B, S, H, D, P.RouteCfg(Bq=c["Bq"], G=c["G"]))
r(q, k, b, 7, 25)
out = torch.empty_like(q)
best = 1e9
for _ in range(int(os.environ.get("REPS", "8"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        P.attn(q, k, v, r, out, stats_only=True)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 10)
gb = 2 * S * D * 2 * B * H / 1e9
print(f"{name} {os.path.basename(os.environ.get('PASA_LIB', 'in-tree'))}: kv_stats {best:.4f} ms, "
      f"{gb / best:.2f} TB/s algorithmic", flush=True)
