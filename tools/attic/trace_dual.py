#!/usr/bin/env python
"""clock64 timeline of one CTA of the dual-tile attention kernel (pasa_debug_trace with
pasa_debug_flags bit 2048) and a per-op summary of where each tile's cycle goes.

    CTA=10 FLAGS=0 python tools/trace_dual.py > gpurun_out/trace_dual.txt
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402
from paper_2604_12219_b200 import _C  # noqa: E402

EV = ["MMA_PW", "MMA_PO", "MMA_ISS", "MMA_QK", "SM_SW", "SM_SO", "SM_AR", "SM_FW", "SM_FO"]
N = 4096
cfg = synth.CONFIGS[os.environ.get("CFG", "wan14b_720p")]
B, S, H, D = cfg["B"], cfg["S"], cfg["H"], cfg["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
route = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=cfg["G"]))
bud = P.Budget()
z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[cfg["rho"]] * 50)
route(q, k, bud, 1, 25)
out = P.attn(q, k, v, route)
buf = torch.zeros(len(EV) * 2 * N, dtype=torch.int64, device="cuda")
cta = int(os.environ.get("CTA", "10"))
_C.lib().pasa_debug_flags(2048 | int(os.environ.get("FLAGS", "0")))
_C.lib().pasa_debug_trace(buf.data_ptr(), cta, 0)
torch.cuda.synchronize()
P.attn(q, k, v, route, out, reuse_stats=True)
torch.cuda.synchronize()
_C.lib().pasa_debug_trace(None, 0, 0)
_C.lib().pasa_debug_flags(0)
tr = buf.view(len(EV), 2, N).cpu().numpy().astype(np.int64)
t0 = tr[tr > 0].min()
tr = np.where(tr > 0, tr - t0, -1)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({e: [tr[i, 0].tolist(), tr[i, 1].tolist()] for i, e in enumerate(EV)},
          open(os.path.join(ROOT, "gpurun_out", "trace_dual.json"), "w"))
E = {e: tr[i] for i, e in enumerate(EV)}
lo, hi = int(os.environ.get("LO", "300")), int(os.environ.get("HI", "600"))
for t in range(2):
    n = np.arange(lo, hi)
    ok = (E["SM_SO"][t, n] > 0) & (E["SM_AR"][t, n] > 0) & (E["MMA_ISS"][t, n] > 0)
    nS = n[ok]
    pr = lambda name, x: print(f"  {name:38s} median {np.median(x):7.0f}  p10 {np.percentile(x,10):7.0f}  p90 {np.percentile(x,90):7.0f}")  # noqa
    print(f"tile {t}: ops {lo}..{hi}, {len(nS)} S ops in window; total span "
          f"{E['SM_AR'][t, hi - 1] - E['SM_AR'][t, lo]} cycles for {hi - lo} ops "
          f"= {(E['SM_AR'][t, hi - 1] - E['SM_AR'][t, lo]) / (hi - lo):.0f} per op")
    pr("softmax: wait for S (SO - SW)", E["SM_SO"][t, nS] - E["SM_SW"][t, nS])
    pr("softmax: work (AR - SO)", E["SM_AR"][t, nS] - E["SM_SO"][t, nS])
    nx = nS[nS + 1 < hi]
    pr("arrive(n) -> MMA saw P(n) (PO - AR)", E["MMA_PO"][t, nx] - E["SM_AR"][t, nx])
    pr("MMA waited for P(n) (PO - PW)", E["MMA_PO"][t, nx] - E["MMA_PW"][t, nx])
    pr("MMA issue PV/F (ISS - PO)", E["MMA_ISS"][t, nx] - E["MMA_PO"][t, nx])
    q_ok = nx[E["MMA_QK"][t, nx + 1] > 0]
    pr("MMA issue QK(n+1) (QK[n+1] - ISS[n])", E["MMA_QK"][t, q_ok + 1] - E["MMA_ISS"][t, q_ok])
    pr("QK(n+1) issued -> S ready (SO[n+1]-QK)", E["SM_SO"][t, q_ok + 1] - E["MMA_QK"][t, q_ok + 1])
    pr("P(n) released -> S(n+1) ready", E["SM_SO"][t, q_ok + 1] - E["SM_AR"][t, q_ok])
    fo = n[(E["SM_FO"][t, n] > 0)]
    if len(fo):
        pr("F op: wait MMA(n-2) (FO - FW)", E["SM_FO"][t, fo] - E["SM_FW"][t, fo])
        pr("F op: Aq write (AR - FO)", E["SM_AR"][t, fo] - E["SM_FO"][t, fo])
