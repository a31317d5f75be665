#!/usr/bin/env python
"""Top source lines of an ncu report by warp-stall samples (needs -lineinfo):
    python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, total = [], "?", 0
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] and rec[0].isdigit() and len(rec) > 6 and rec[4].isdigit():
        s = int(rec[4])
        total += s
        rows.append((s, fname, int(rec[0]), rec[1].strip()[:90]))
rows.sort(reverse=True)
print(f"total samples {total}")
for s, f, ln, src in rows[:n]:
    print(f"{100.0 * s / max(total, 1):5.1f}%  {f}:{ln}  {src}")
