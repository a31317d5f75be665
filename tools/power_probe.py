#!/usr/bin/env python
"""Power / clock probe: each attention variant runs back to back for SECS seconds
while NVML samples board power, SM clock and throttle reasons (every 20 ms).  Reports
per variant: ms per launch, median SM MHz, median W, throttle reasons, and
energy per launch (J) = median W x ms.  If every variant sits at the board power
limit, time per launch is energy per launch / power: the kernel is power-bound.
    CFG=wan14b_720p SECS=4 [DENSE_HEADS=8] python tools/power_probe.py
(DENSE_HEADS: also torch's dense SDPA on that many heads, the library kernel on the same
box and cap; pJ/FLOP uses the algorithmic FLOPs of each.)"""
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

name = os.environ.get("CFG", "wan14b_720p")
SECS = float(os.environ.get("SECS", "4"))
cfg = synth.CONFIGS[name]
B, S, H, D = cfg["B"], cfg["S"], cfg["H"], cfg["D"]
q, k, v = synth.iid_qkv(B, S, H, D, seed=1, dtype=torch.bfloat16, device="cuda")
bud = P.Budget()
z = torch.zeros(64, device="cuda")
bud(z, z, z, T=50, step=25, rho_table=[cfg["rho"]] * 50)
variants = {}
for bq in (128, 256):
    r = P.Route(B, S, H, D, P.RouteCfg(Bq=bq, G=cfg["G"]))
    r(q, k, bud, 1, 25)
    out = P.attn(q, k, v, r)
    if bq == 128:
        variants["default (Bq 128, 2 CTAs/SM)"] = (r, out, {})
    else:
        variants["q256 (Bq 256, 1 CTA/SM, 2 tiles)"] = (r, out, {})
        if D == 128:
            variants["pair (Bq 256, cta_group::2)"] = (r, torch.empty_like(out), {"cta_pair": True})
# algorithmic FLOPs per launch (the same for Bq = 128 and 256)
NK, NG = variants["default (Bq 128, 2 CTAs/SM)"][0].NK, variants["default (Bq 128, 2 CTAs/SM)"][0].NG
kk = variants["default (Bq 128, 2 CTAs/SM)"][0].read()["k"]
flops = {vn: (4.0 * S * kk * 64 * D + 4.0 * S * NK * D + 2.0 * S * D * D * NG) * B * H
         for vn in variants}
DENSE_H = int(os.environ.get("DENSE_HEADS", "0"))   # > 0: also dense SDPA on that many heads
if DENSE_H:
    qd, kd, vd = (t[:, :, :DENSE_H].transpose(1, 2).contiguous() for t in (q, k, v))
    variants[f"dense SDPA ({DENSE_H} heads, torch / cuDNN)"] = (None, None, {"dense": (qd, kd, vd)})
    flops[f"dense SDPA ({DENSE_H} heads, torch / cuDNN)"] = 4.0 * S * S * D * B * DENSE_H


def launch(r, out, kw):
    if "dense" in kw:
        torch.nn.functional.scaled_dot_product_attention(*kw["dense"])
    else:
        P.attn(q, k, v, r, out, reuse_stats=True, **kw)

pynvml.nvmlInit()
dev = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(dev) / 1000.0
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.time(), pynvml.nvmlDeviceGetPowerUsage(dev) / 1000.0,
                        pynvml.nvmlDeviceGetClockInfo(dev, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(dev)))
        time.sleep(0.02)


th = threading.Thread(target=sampler, daemon=True)
th.start()
print(f"{name}: enforced power limit {limit_w:.0f} W", flush=True)
for rep in range(2):
    for vname, (r, out, kw) in variants.items():
        for _ in range(3):
            launch(r, out, kw)
        torch.cuda.synchronize()
        t0 = time.time()
        n = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        while time.time() - t0 < SECS:
            for _ in range(10):
                launch(r, out, kw)
            n += 10
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.time()
        ms = e0.elapsed_time(e1) / n
        win = [s for s in samples if t0 + 0.3 <= s[0] <= t1]
        w = statistics.median(s[1] for s in win)
        mhz = statistics.median(s[2] for s in win)
        reasons = 0
        for s in win:
            reasons |= s[3]
        names = [nm for bit, nm in ((0x4, "sw_power_cap"), (0x8, "hw_slowdown"),
                                    (0x20, "sw_thermal"), (0x40, "hw_thermal"),
                                    (0x80, "hw_power_brake")) if reasons & bit]
        print(f"rep {rep} {vname}: {ms:.3f} ms/launch, SM {mhz:.0f} MHz, {w:.0f} W, "
              f"{w * ms / 1000:.2f} J/launch, {ms * mhz / 1000:.0f} kcycles/launch, "
              f"{flops[vname] / (ms * 1e-3) / 1e12:,.0f} TFLOP/s, "
              f"{w * ms * 1e-3 / flops[vname] * 1e12:.3f} pJ/FLOP, reasons {names}", flush=True)
stop.set()
