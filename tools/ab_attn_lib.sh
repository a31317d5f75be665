#!/usr/bin/env bash
# A/B of the default library against ab_tmp/$VAR (built here; run on the GPU box)
set -u
VAR=${VAR:-c3}
B=paper_2604_12219_b200/lib/libpasa.so
A=ab_tmp/$VAR/lib/libpasa.so
PASA_LIB=$A timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -q -x -k "${KSEL:-not nothing}" 2>&1 | tail -4
for c in ${CFGS:-cogvideox5b}; do
for L in $B $A $B $A $B $A; do PASA_LIB=$L CFG=$c REPS=${REPS:-6} timeout 300 python tools/lib_time.py; done
done
if [ -n "${TCFG:-}" ]; then
PASA_LIB=$A CFG=$TCFG RAW_ONLY=1 timeout 300 python tools/trace_attn.py ${TX:-100} ${TY:-20} && cp gpurun_out/trace_raw.json gpurun_out/trace_raw_$VAR.json
fi
