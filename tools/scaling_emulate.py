#!/usr/bin/env python
"""Per-rank work of the multi-GPU run, emulated on one GPU: the bench step (budget +
route + statistics + attention) of every rank r of N = 1, 2, 4, 8, with the same route
handles bench.py builds (global head offsets; for PART=flat, or heads that do not
divide N, the flattened (head, q-block) segments of dist.flat_partition).  Ranks share
nothing on the hot path, so the N-GPU step time is the max over ranks of these per-rank
times; the printed t_1 / (N t_N) is the strong-scaling efficiency this predicts (the
driver measures the real one).
    CFG=wan13b_480p PART=flat python tools/scaling_emulate.py"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402
from paper_2604_12219_b200 import dist as pdist  # noqa: E402

name = os.environ.get("CFG", "wan14b_720p")
part = os.environ.get("PART", "auto")
c = synth.CONFIGS[name]
B, S, H, D = c["B"], c["S"], c["H"], c["D"]
NQ = -(-S // c["Bq"])
tp = synth.ThreePhase(shape=c["latent"], T=50, seed=7, device="cuda")
x_t, x_tm1, x_tm2 = (x.contiguous() for x in tp.latents(25))
q_all, k_all, v_all = synth.iid_qkv(B, S, H, D, seed=1000, dtype=torch.bfloat16, device="cuda")
out_all = torch.empty_like(q_all)
bud = P.Budget()


def time_rank(segs):
    units = []
    for h, n, a, b in segs:
        cfg = P.RouteCfg(Bq=c["Bq"], G=c["G"], H_total=H, head_offset=h, qb_begin=a, qb_end=b)
        sl = slice(h, h + n)
        units.append((P.Route(B, S, n, D, cfg), q_all[:, :, sl], k_all[:, :, sl],
                      v_all[:, :, sl], out_all[:, :, sl]))

    def step():
        bud(x_t, x_tm1, x_tm2, T=50, step=25, rho=c["rho"], l1_mean=tp.expected_l1_mean(),
            h_t=1 / 50, h_tm1=1 / 50, rho_table=[c["rho"]] * 50)
        for r, q, k, v, o in units:
            r(q, k, bud, P.layer_seed(42, 0), 25)
            P.attn(q, k, v, r, o)

    for _ in range(3):
        step()
    xs = []
    for _ in range(int(os.environ.get("REPS", "7"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        xs.append(e0.elapsed_time(e1))
    return statistics.median(xs)


res = {}
for N in (1, 2, 4, 8):
    flat = part == "flat" or (part == "auto" and H % N)
    if flat:
        ranks = [pdist.flat_partition(H, NQ, N, r) for r in range(N)]
    else:
        ranks = [[(*pdist.head_range(H, N, r), 0, 0)] for r in range(N)]
    # ranks with identical work shapes time the same: time each distinct shape once
    shapes = {}
    for segs in ranks:
        key = tuple((n, a, b) for _, n, a, b in segs)
        if key not in shapes:
            shapes[key] = time_rank(segs)
    res[N] = (max(shapes.values()), "flat" if flat else "heads", len(shapes))
t1 = res[1][0]
for N, (t, how, nshapes) in res.items():
    print(f"{name} N={N} ({how} partition, {nshapes} distinct rank shapes): step {t:.3f} ms "
          f"(max over ranks), {4.0 * S * S * D * B * H / (t * 1e-3) / 1e12:,.0f} TFLOP/s-equiv "
          f"whole job, predicted strong-scaling efficiency {t1 / (N * t):.3f}", flush=True)
