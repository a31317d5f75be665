#!/usr/bin/env python
"""Time the default attention launch of one config with the library PASA_LIB points
at (A/B of two builds in alternating processes):
    for L in a.so b.so a.so b.so; do PASA_LIB=$L CFG=cogvideox5b python tools/lib_time.py; done"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402

name = os.environ.get("CFG", "cogvideox5b")
c = synth.CONFIGS[name]
B, S, H, D = c["B"], c["S"], c["H"], c["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
route = P.Route(B, S, H, D, P.RouteCfg(Bq=c["Bq"], G=c["G"]))
bud = P.Budget()
z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[c["rho"]] * 50)
route(q, k, bud, 1, 25)
out = P.attn(q, k, v, route, stats_only=True)
xs = []
for rep in range(int(os.environ.get("REPS", "8"))):
    for _ in range(2):
        P.attn(q, k, v, route, out, reuse_stats=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        P.attn(q, k, v, route, out, reuse_stats=True)
    e1.record()
    torch.cuda.synchronize()
    xs.append(e0.elapsed_time(e1) / 10)
_lib = os.environ.get("PASA_LIB", "in-tree")
_tag = os.path.basename(os.path.dirname(os.path.dirname(_lib))) if "ab_tmp" in _lib else "default"
print(f"{name} {_tag}: attn min {min(xs):.4f} "
      f"median {statistics.median(xs):.4f} ms, finite {bool(torch.isfinite(out).all())}", flush=True)
