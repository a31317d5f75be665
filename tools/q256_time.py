#!/usr/bin/env python
"""Bq = 256 against the default Bq = 128 on one config:
route + attention per layer, interleaved repetitions (min / median ms), and the
exact-attention FLOPs are the same (k kept blocks per query row either way).
Bq = 256 attention runs on both kernels: the one-CTA two-tile kernel ("256") and
the tcgen05 cta_group::2 pair ("256pair", d = 128 only).
    CFG=wan14b_720p REPS=6 python tools/q256_time.py"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402

name = os.environ.get("CFG", "wan14b_720p")
cfg = synth.CONFIGS[name]
B, S, H, D = cfg["B"], cfg["S"], int(os.environ.get("HEADS", cfg["H"])), cfg["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
bud = P.Budget()
z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[cfg["rho"]] * 50)
routes = {}
for bq in (128, 256):
    r = P.Route(B, S, H, D, P.RouteCfg(Bq=bq, G=cfg["G"]))
    r(q, k, bud, 1, 25)
    routes[bq] = r
outs = {bq: P.attn(q, k, v, routes[bq]) for bq in routes}
pair = D == 128
if pair:
    outs["256pair"] = P.attn(q, k, v, routes[256], cta_pair=True)
torch.cuda.synchronize()
if pair:
    dp = (outs["256pair"].float() - outs[256].float()).abs().max() / outs[256].float().abs().max()
    print(f"{name}: pair vs one-CTA Bq = 256 kernel max|dO|/max|O| {dp:.3e}, finite "
          f"{bool(torch.isfinite(outs['256pair']).all())}", flush=True)
d = (outs[256].float() - outs[128].float()).norm() / outs[128].float().norm()
print(f"{name}: k = {routes[128].read()['k']} (Bq 128) / {routes[256].read()['k']} (Bq 256); "
      f"relative Frobenius distance of the two outputs {d:.3e}", flush=True)
REPS = int(os.environ.get("REPS", "6"))
res = {}


def timed(fn, n=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for rep in range(REPS):
    for bq, r in routes.items():
        res.setdefault((bq, "route"), []).append(timed(lambda: r(q, k, bud, 1, 25), 3))
        P.attn(q, k, v, r, outs[bq], stats_only=True)
        res.setdefault((bq, "attn"), []).append(
            timed(lambda: P.attn(q, k, v, r, outs[bq], reuse_stats=True)))
        if bq == 256 and pair:
            res.setdefault(("256pair", "attn"), []).append(
                timed(lambda: P.attn(q, k, v, r, outs["256pair"], reuse_stats=True, cta_pair=True)))
dense_flops = 4.0 * S * S * D * B * H
for (bq, what), xs in sorted(res.items(), key=lambda kv: (str(kv[0][0]), kv[0][1])):
    extra = ""
    if what == "attn":
        extra = f"  ({dense_flops / (min(xs) * 1e-3) / 1e12:,.0f} TFLOP/s-equiv at min)"
    print(f"{name} Bq={bq} {what}: min {min(xs):.3f} median {statistics.median(xs):.3f} ms{extra}",
          flush=True)
