#!/usr/bin/env python
"""Record and summarise the clock64() timeline of one attention CTA
(pasa_debug_trace).  Usage (GPU box):  python tools/trace_attn.py [x y] > out.txt"""
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

EV = ["KPROD", "VPROD", "MMA_P", "MMA_V", "MMA_QK", "SA_W", "SA_OK", "SA_ARR", "SB_W", "SB_OK",
      "SB_ARR", "MMA_QKW", "KPROD_W", "SA_LD", "SA_MAX", "SA_EXP", "SA_ST"]


def main():
    x = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    y = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = synth.CONFIGS[os.environ.get("CFG", "wan14b_720p")]
    B, S, H, D = cfg["B"], cfg["S"], cfg["H"], cfg["D"]
    q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
    route = P.Route(B, S, H, D, P.RouteCfg(Bq=128, G=32))
    bud = P.Budget()
    z = torch.zeros(64, device="cuda")
    bud(z, z, z, T=50, step=25, rho_table=[cfg["rho"]] * 50)
    route(q, k, bud, 1, 25)
    out = P.attn(q, k, v, route)
    buf = torch.zeros(17 * 4096, dtype=torch.int64, device="cuda")
    _C.lib().pasa_debug_flags(int(os.environ.get("FLAGS", "0")))
    _C.lib().pasa_debug_trace(buf.data_ptr(), x, y)
    torch.cuda.synchronize()
    P.attn(q, k, v, route, out)
    torch.cuda.synchronize()
    _C.lib().pasa_debug_trace(None, 0, 0)
    tr = buf.view(17, 4096).cpu().numpy().astype(np.int64)
    t0 = tr[tr > 0].min()
    d = {e: tr[i] for i, e in enumerate(EV)}

    def col(e):
        a = d[e]
        n = int((a > 0).sum())
        return (a[:n] - t0).astype(np.int64)

    res = {e: col(e).tolist() for e in EV}
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "trace.json"), "w"))
    raw = {e: np.where(tr[i] > 0, tr[i] - t0, -1).tolist() for i, e in enumerate(EV)}
    json.dump(raw, open(os.path.join(ROOT, "gpurun_out", "trace_raw.json"), "w"))
    if os.environ.get("RAW_ONLY"):
        return
    sa_w, sa_ok, sa_arr = col("SA_W"), col("SA_OK"), col("SA_ARR")
    n = min(len(sa_ok), len(sa_arr))
    print("tile A ops:", len(sa_arr), "total cycles", int(sa_arr[-1]))
    print("tile A per-op period (median)", float(np.median(np.diff(sa_arr))))
    m = min(len(sa_w), len(sa_ok))
    print("tile A s_full wait median/mean", float(np.median(sa_ok[:m] - sa_w[:m])),
          float(np.mean(sa_ok[:m] - sa_w[:m])))
    # softmax busy: from s_full ok to arrive (same op index for S ops only; approx)
    print("first 12 ops A: W, OK, ARR")
    for i in range(12):
        print(i, sa_w[i] if i < len(sa_w) else -1, sa_ok[i] if i < len(sa_ok) else -1, sa_arr[i])
    mp, mv, mq, mqw = col("MMA_P"), col("MMA_V"), col("MMA_QK"), col("MMA_QKW")
    kp, kpw, vp = col("KPROD"), col("KPROD_W"), col("VPROD")
    print("MMA: p_full-ok times first 16:", mp[:16].tolist())
    print("MMA: v_full-ok minus p_full-ok (median)", float(np.median(mv - mp[:len(mv)])))
    print("MMA: QK k_full wait (median/mean)", float(np.median(mq - mqw)), float(np.mean(mq - mqw)))
    if len(kp) and len(kp) == len(kpw):
        print("Kprod: issue minus wait start (median/mean)", float(np.median(kp - kpw)),
              float(np.mean(kp - kpw)))
        lat = [mq[u] - kp[u] for u in range(min(len(kp), len(mq)))]
        print("K issue -> QK start (median)", float(np.median(lat)))
    ld, mxx, ex, st = col("SA_LD"), col("SA_MAX"), col("SA_EXP"), col("SA_ST")
    lo = 100 if len(ld) > 130 else max(0, len(ld) // 3)
    if len(ld) > lo + 12 and len(col("SB_ARR")) == 0:
        print(f"v1 ops {lo}..{lo + 12}: OK->LD, LD->MAX, MAX->EXP, EXP->ST, ST->ARR, ARR->W(next)")
        for i in range(lo, lo + 12):
            print(i, ld[i] - sa_ok[i], mxx[i] - ld[i], ex[i] - mxx[i], st[i] - ex[i], sa_arr[i] - st[i],
                  sa_w[i + 1] - sa_arr[i])
    elif len(ld) > 110:
        print("middle ops 100..110 A (S-type indices): OK->LD, LD->MAX, MAX->EXP, EXP->ST, ST->ARR")
        for i in range(100, 110):
            print(i, ld[i] - sa_ok[i], mxx[i] - ld[i], ex[i] - mxx[i], st[i] - ex[i], sa_arr[i] - st[i])
    # single-tile kernels: per op n, the MMA warp's view
    if len(col("SB_ARR")) == 0 and len(mp) > 120:
        print("op: OK-W(s_full wait) ARR-OK(softmax busy) P-ARR(p_full notice) "
              "QK(n+1)-QKW(n+1)(k wait) V-QK? period")
        for u in range(100, 120):
            print(u, sa_ok[u] - sa_w[u], sa_arr[u] - sa_ok[u], mp[u] - sa_arr[u],
                  (mq[u + 1] - mqw[u + 1]) if u + 1 < len(mq) else -1, mv[u] - mp[u] if u < len(mv) else -1,
                  sa_arr[u + 1] - sa_arr[u])
        per = np.diff(sa_arr[50:-50])
        print("median period", float(np.median(per)), "mean", float(np.mean(per)))
        kw = col("SB_W")
        if len(kw) > 120:
            print("K(n+1) wait only (QKW -> K landed), median over ops 50..-50:",
                  float(np.median(kw[50:-50] - mqw[50:len(kw) - 50])))
        pv = col("KPROD_W")
        if len(pv) > 120:
            print("MMA warp per op: QKW->QK(n+1) | QK(n+1)->V(n) | V->P(n) | P->PVdone(n) | PVdone->QKW(n+2)")
            for u in range(100, 120):
                print(u, mq[u + 1] - mqw[u + 1], mv[u] - mq[u + 1], mp[u] - mv[u], pv[u] - mp[u],
                      mqw[u + 2] - pv[u])
        k = min(len(sa_ok), len(sa_w)) - 50
        print("median softmax busy", float(np.median(sa_arr[50:k] - sa_ok[50:k])),
              "median s_full wait", float(np.median(sa_ok[50:k] - sa_w[50:k])),
              "median p_full notice", float(np.median(mp[50:k] - sa_arr[50:k])))
    print("middle window ops 100..110 A: W OK ARR")
    for i in range(100, 110):
        print(i, sa_w[i] if i < len(sa_w) else -1, sa_ok[i] if i < len(sa_ok) else -1,
              sa_arr[i] if i < len(sa_arr) else -1)


if __name__ == "__main__":
    main()


def mma_view(path=os.path.join(ROOT, "gpurun_out", "trace.json"), lo=200, hi=216):
    d = json.load(open(path))
    mp, mv, qk, qkw = d["MMA_P"], d["MMA_V"], d["MMA_QK"], d["MMA_QKW"]
    for u in range(lo, hi):
        t, n = u & 1, u >> 1
        arr = (d["SA_ARR"] if t == 0 else d["SB_ARR"])[n]
        pos2 = 2 * (n + 2) + t
        print(u, t, n, "ARR", arr, "MMA_P", mp[u], "MMA_V", mv[u], "QKW", qkw[pos2] if pos2 < len(qkw) else -1,
              "QK", qk[pos2] if pos2 < len(qk) else -1)
