#!/usr/bin/env python
"""A/B timing of the tensor-core attention kernels on one config: the default
(single softmax warpgroup, 2 CTAs/SM) against the ping-pong variant (one CTA/SM,
Q in TMEM, two softmax warpgroups),
interleaved repetitions (the pool's clocks drift under power cap), min / median.
    CFG=wan14b_720p REPS=8 python tools/ab_attn.py"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402

cfg = synth.CONFIGS[os.environ.get("CFG", "wan14b_720p")]
B, S, H, D = cfg["B"], cfg["S"], int(os.environ.get("HEADS", cfg["H"])), cfg["D"]
G = int(os.environ.get("G", "32"))
comp = os.environ.get("COMP", "grouped")
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
route = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=G, comp=comp))
bud = P.Budget()
z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[float(os.environ.get("RHO", cfg["rho"]))] * 50)
route(q, k, bud, 1, 25)
out = P.attn(q, k, v, route, stats_only=True)
ref = torch.empty_like(q)
P.attn(q, k, v, route, ref, reuse_stats=True, pingpong=True)
P.attn(q, k, v, route, out, reuse_stats=True, pingpong=False)
torch.cuda.synchronize()
d = (out.float() - ref.float()).abs().max().item() / ref.float().abs().max().item()
print(f"max|default - pingpong| / max|O| = {d:.3e}", flush=True)
REPS = int(os.environ.get("REPS", "6"))
res = {}
for rep in range(REPS):
    for name, sw in (("default", False), ("pingpong", True)):
        for _ in range(2):
            P.attn(q, k, v, route, out, reuse_stats=True, pingpong=sw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            P.attn(q, k, v, route, out, reuse_stats=True, pingpong=sw)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(name, []).append(e0.elapsed_time(e1) / 5)
for name, v_ in res.items():
    print(f"{os.environ.get('CFG', 'wan14b_720p')} G={G} {comp} {name}: attn min {min(v_):.3f} "
          f"median {statistics.median(v_):.3f} ms", flush=True)
