#!/usr/bin/env python
"""A/B timing of the default persistent dual-tile attention kernel against round 1's
two-CTA kernel (PASA_ATTN_LEGACY) on one BASELINE config, interleaved repetitions
(the pool's clocks drift under the power cap): attn ms per launch, min / median.

    CFG=wan14b_720p REPS=5 python tools/ab_dual.py
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402
from paper_2604_12219_b200 import _C  # noqa: E402

name = os.environ.get("CFG", "wan14b_720p")
cfg = synth.CONFIGS[name]
B, S, H, D = cfg["B"], cfg["S"], int(os.environ.get("HEADS", cfg["H"])), cfg["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
route = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=int(os.environ.get("G", cfg["G"])),
                                       comp=os.environ.get("COMP", "grouped")))
bud = P.Budget()
z = torch.zeros(64, device="cuda")
rho = float(os.environ.get("RHO", cfg["rho"]))
bud(z, z, z, T=50, step=25, rho_table=[rho] * 50)
route(q, k, bud, 1, 25)
out = P.attn(q, k, v, route, stats_only=True)
a = P.attn(q, k, v, route, reuse_stats=True).float()
b = P.attn(q, k, v, route, reuse_stats=True, legacy=True).float()
torch.cuda.synchronize()
print(f"{name}: H={H} k={route.read()['k']} max|dual - legacy|/max|O| = "
      f"{((a - b).abs().max() / b.abs().max()).item():.3e}", flush=True)
variants = {"dual": dict(), "legacy": dict(legacy=True)}
if os.environ.get("POLY") == "1":
    variants["dual poly 1/4"] = dict(_dbg=128)
    variants["dual poly 1/2"] = dict(_dbg=4096)
for f in [int(x) for x in os.environ.get("ABL", "").split(",") if x]:
    # ablations of the dual kernel (pasa_debug_flags): 256 = softmax skips its math,
    # 512 = producers skip the TMA loads, 768 = both (bare MMA chain + handshakes)
    variants[f"dual abl={f}"] = dict(_dbg=f)
REPS = int(os.environ.get("REPS", "5"))
N = int(os.environ.get("N", "5"))
res = {kname: [] for kname in variants}
for rep in range(REPS):
    for kname, kw in variants.items():
        kw = dict(kw)
        old = _C.lib().pasa_debug_flags(kw.pop("_dbg", 0))
        for _ in range(2):
            P.attn(q, k, v, route, out, reuse_stats=True, **kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(N):
            P.attn(q, k, v, route, out, reuse_stats=True, **kw)
        e1.record()
        torch.cuda.synchronize()
        _C.lib().pasa_debug_flags(old)
        res[kname].append(e0.elapsed_time(e1) / N)
for kname, v_ in res.items():
    print(f"{name} {kname}: attn min {min(v_):.3f} median {statistics.median(v_):.3f} ms "
          f"({len(v_)} reps x {N})", flush=True)
