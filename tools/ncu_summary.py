#!/usr/bin/env python
"""Summarise an `ncu --set full` report (.ncu-rep) or a launch-list CSV into
markdown for profiles/.  Usage:
    python tools/ncu_summary.py report  gpurun_out/prof_attn.ncu-rep  > profiles/x.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv      > profiles/y.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (registers), CTAs/SM"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem), CTAs/SM"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def report(path):
    for d, u in raw(path):
        print(f"### {d.get('Kernel Name', '?')[:110]}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k, name in KEYS:
            if k in d:
                print(f"| {name} (`{k}`) | {d[k]} | {u.get(k, '')} |")
        stalls = [(k, d[k]) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("_not_issued") and d[k] not in ("", "0")]
        tot = sum(float(v.replace(",", "")) for _, v in stalls) or 1.0
        top = sorted(stalls, key=lambda kv: -float(kv[1].replace(",", "")))[:8]
        print("\nTop warp-stall reasons (pc sampling, share of samples):\n")
        for k, v in top:
            print(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: "
                  f"{100 * float(v.replace(',', '')) / tot:.1f}%")
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = {}
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"]
            unit = d.get("Metric Unit", "ns")
            v = float(d["Metric Value"].replace(",", ""))
            v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)  # -> us
            if name not in agg:
                agg[name] = []
                order.append(name)
            agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |\n|---|---|---|---|---|")
    for n in order:
        v = agg[n]
        print(f"| `{n[:90]}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | "
              f"{100 * sum(v) / tot:.1f}% |")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
