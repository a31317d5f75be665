#!/usr/bin/env python
"""Energy per launch of the default attention kernel under the diagnostics ablations
(pasa_debug_flags: 8 = diagnostics build, no ablation; +1 the softmax skips its
arithmetic; +2 the producers skip the TMA loads), NVML-sampled while each runs back
to back for SECS seconds: where the joules of a power-capped launch go.
    CFG=wan14b_720p SECS=4 python tools/energy_ablate.py"""
import os
import statistics
import sys
import threading
import time

import pynvml
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2604_12219_b200 as P  # noqa: E402
from paper_2604_12219_b200 import _C  # noqa: E402

name = os.environ.get("CFG", "wan14b_720p")
SECS = float(os.environ.get("SECS", "4"))
c = synth.CONFIGS[name]
B, S, H, D = c["B"], c["S"], c["H"], c["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
bud = P.Budget()
z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[c["rho"]] * 50)
r = P.Route(B, S, H, D, P.RouteCfg(Bq=c["Bq"], G=c["G"]))
r(q, k, bud, 1, 25)
out = P.attn(q, k, v, r, stats_only=True)
pynvml.nvmlInit()
dev = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.time(), pynvml.nvmlDeviceGetPowerUsage(dev) / 1000.0,
                        pynvml.nvmlDeviceGetClockInfo(dev, pynvml.NVML_CLOCK_SM)))
        time.sleep(0.02)


threading.Thread(target=sampler, daemon=True).start()
names = {0: "production", 8: "diagnostics build", 9: "no softmax arithmetic",
         10: "no TMA loads", 11: "bare MMA chain (neither)"}
for rep in range(2):
    for fl in [int(x) for x in os.environ.get("FLAGS", "0,8,9,10,11").split(",")]:
        _C.lib().pasa_debug_flags(fl)
        for _ in range(3):
            P.attn(q, k, v, r, out, reuse_stats=True)
        torch.cuda.synchronize()
        t0 = time.time()
        n = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.time() - t0 < SECS:
            for _ in range(5):
                P.attn(q, k, v, r, out, reuse_stats=True)
            n += 5
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.time()
        ms = e0.elapsed_time(e1) / n
        win = [s for s in samples if t0 + 0.3 <= s[0] <= t1]
        w = statistics.median(s[1] for s in win)
        mhz = statistics.median(s[2] for s in win)
        print(f"rep {rep} flags {fl:2d} {names[fl]:26s}: {ms:7.3f} ms, {mhz:5.0f} MHz, {w:4.0f} W, "
              f"{w * ms / 1000:6.2f} J/launch, {ms * mhz / 1000:6.1f} Mcycles", flush=True)
_C.lib().pasa_debug_flags(0)
stop.set()
