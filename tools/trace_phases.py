#!/usr/bin/env python
"""Per-op phase medians of a raw attention trace (tools/trace_attn.py RAW_ONLY=1 output):
    python tools/trace_phases.py gpurun_out/trace_raw.json"""
import json
import sys

import numpy as np

for f in sys.argv[1:]:
    d = {k: np.array(v) for k, v in json.load(open(f)).items()}
    ok, ld, ex, st, arr, w = (d[k] for k in ("SA_OK", "SA_LD", "SA_EXP", "SA_ST", "SA_ARR", "SA_W"))
    mp, mqw, mq = d["MMA_P"], d["MMA_QKW"], d["MMA_QK"]
    n = int((arr >= 0).sum())
    rows = [(ld[i] - ok[i], ex[i] - ld[i], st[i] - ex[i], arr[i] - st[i], ok[i] - w[i],
             w[i] - arr[i - 1], mp[i] - arr[i]) for i in range(10, n - 10) if ld[i] >= 0]
    r = np.median(np.array(rows), axis=0)
    so = [arr[i] - arr[i - 1] for i in range(10, n - 10) if ld[i] >= 0]
    fo = [arr[i] - arr[i - 1] for i in range(10, n - 10) if ld[i] < 0]
    print(f"{f}: ops {n}, total {arr[n - 1]} cycles; S-op period {np.median(so):.0f}, "
          f"F-op period {np.median(fo) if fo else float('nan'):.0f} ({len(fo)})")
    print("  median  OK->LD %.0f  LD->EXP %.0f  EXP->ST %.0f  ST->ARR %.0f  W->OK %.0f  "
          "ARR(prev)->W %.0f  ARR->MMA sees P %.0f" % tuple(r))
