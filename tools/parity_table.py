#!/usr/bin/env python
"""gpurun_out/parity_errors.json (written by the GPU parity tests, tests/conftest.py
parity_log) -> a markdown table of every achieved error, worst first.

    python tools/parity_table.py [in.json] > profiles/rNN_parity_errors.md
"""
import json
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity_errors.json"
rows = json.load(open(src))
print("# GPU parity: achieved errors of every compared output\n")
print("Written by `pytest tests -m gpu` (tests/conftest.py `parity_log`); reference = the fp64 "
      "oracle on the GPU route (`oracle`) or fp32 dense attention for the constant-key-block "
      "cases (`dense`).  Contract: max|dO|/max|O| <= 2e-2 (bf16 I/O), <= 1e-5 (fp32 I/O); "
      "regression bound asserted by the tests: 8e-3 (bf16), 1e-5 (fp32).  FP8 QK^T variant "
      "(R-30): its own bound 1e-1 max / 6e-2 Frobenius.\n")
print("| case | ref | max\\|dO\\|/max\\|O\\| | rel. Frobenius | bound | test |")
print("|---|---|---|---|---|---|")
for r in sorted(rows, key=lambda r: -r["max_rel"]):
    print(f"| {r['case']} | {r['ref']} | {r['max_rel']:.2e} | {r['frob_rel']:.2e} | "
          f"{r['bound']:.0e} | `{r['test'].split('::', 1)[1]}` |")
print(f"\n{len(rows)} compared outputs; worst bf16 {max(r['max_rel'] for r in rows):.2e}.")
