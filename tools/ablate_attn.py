#!/usr/bin/env python
"""Time the tensor-core attention kernel under
diagnostic ablations (pasa_debug_flags).  REPS > 1 interleaves the
configurations and reports min / median (the pool's clocks drift under power cap)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402
from paper_2604_12219_b200 import _C  # noqa: E402

cfg = synth.CONFIGS[os.environ.get("CFG", "wan14b_720p")]
B, S, H, D = cfg["B"], cfg["S"], int(os.environ.get("HEADS", cfg["H"])), cfg["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
route = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=32))
bud = P.Budget()
z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[cfg["rho"]] * 50)
route(q, k, bud, 1, 25)
out = P.attn(q, k, v, route, stats_only=True)
REPS = int(os.environ.get("REPS", "1"))
results = {}
for rep in range(REPS):
  for variant in os.environ.get("VARIANTS", "default").split(","):
    for flags in [int(f) for f in os.environ.get("FLAGS", "0,1,3").split(",")]:
        _C.lib().pasa_debug_flags(flags)
        for _ in range(2):
            P.attn(q, k, v, route, out, reuse_stats=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.attn(q, k, v, route, out, reuse_stats=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        results.setdefault((variant, flags), []).append(ms)
        if REPS == 1:
            print(f"{variant} flags={flags} attn {ms:.3f} ms", flush=True)
_C.lib().pasa_debug_flags(0)
if REPS > 1:   # interleaved repetitions: min and median per configuration
    import statistics
    for (variant, flags), v in results.items():
        print(f"{variant} flags={flags} attn min {min(v):.3f} median {statistics.median(v):.3f} ms "
              f"over {len(v)}", flush=True)
