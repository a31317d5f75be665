#!/usr/bin/env python
"""Summarise gpurun_out/trace.json for the v3 (single-tile, paired-block) kernel."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "trace.json")))
a = {k: np.array(v) for k, v in d.items()}
mv, mp, mq = a["MMA_V"], a["MMA_P"], a["MMA_QK"]
n = min(len(mv), len(mp), len(mq))
print("ops", n, "first MMA_V", mv[0], "last MMA_QK", mq[n - 1])
print("per-op MMA period median", float(np.median(np.diff(mq[:n]))))
print("wait v/k (MMA_V - prev MMA_QK) median", float(np.median(mv[1:n] - mq[:n - 1])))
print("wait p_full (MMA_P - MMA_V) median", float(np.median(mp[:n] - mv[:n])))
print("issue (MMA_QK - MMA_P) median", float(np.median(mq[:n] - mp[:n])))
sw, sok, sarr = a["SA_W"], a["SA_OK"], a["SA_ARR"]
print("softmax: s_full wait median", float(np.median(sok - sw[:len(sok)])) if len(sok) else None)
if len(a.get("SA_ST", [])):
    ld, mx, ex, st = a["SA_LD"], a["SA_MAX"], a["SA_EXP"], a["SA_ST"]
    k = min(len(ld), len(mx), len(ex), len(st))
    print("softmax OK->LD, LD->MAX, MAX->EXP, EXP->ST (median):",
          float(np.median(ld[:k] - sok[:k])), float(np.median(mx[:k] - ld[:k])),
          float(np.median(ex[:k] - mx[:k])), float(np.median(st[:k] - ex[:k])))
print("ops 40..50: MMA_V MMA_P MMA_QK | SA_W SA_OK SA_ARR")
for i in range(40, 50):
    print(i, mv[i], mp[i], mq[i], "|", sw[i] if i < len(sw) else -1, sok[i] if i < len(sok) else -1,
          sarr[i] if i < len(sarr) else -1)
kp = a["KPROD"]
print("K producer issue times 40..50:", kp[40:50].tolist())
