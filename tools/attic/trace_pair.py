#!/usr/bin/env python
"""Summarise gpurun_out/trace.json of the paired-block variant (PASA_ATTN_PAIRED,
attn_sm100_pair.cu): per-op phases of the two softmax warpgroups and the two
MMA issuers."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "trace.json")))
a = {k: np.array(v) for k, v in d.items()}
qkw, qk = a["MMA_QKW"], a["MMA_QK"]      # QK warp: before k_full wait (after buf_free), after issue (index m)
mv, mp = a["MMA_V"], a["MMA_P"]          # PV warp: after v/k waits, after PV issue+commits (index n)
sw, sok, sarr = a["SA_W"], a["SA_OK"], a["SA_ARR"]
print("n | QKW  QK(n) | SA_W SA_OK SA_ARR | MMA_V MMA_P(end)")
for n in range(40, 52):
    print(n, "|", qkw[n], qk[n], "|", sw[n], sok[n], sarr[n], "|", mv[n], mp[n])
n = min(len(qk), len(mp)) - 2
print("median QK issue dur (QK - QKW)", np.median(qk[:n] - qkw[:n]))
print("median PV iter dur (MMA_P - MMA_V)", np.median(mp[:n] - mv[:n]))
print("median buf_free wait: QKW(n+2) - MMA_P(n)", np.median(qkw[2:n] - mp[:n - 2]))
print("median s_full latency: SA_OK(n) - QK(n)", np.median(sok[:n] - qk[:n]))
print("median p_full->PV: MMA_P(n) - SA_ARR(n)", np.median(mp[:n] - sarr[:n]))
