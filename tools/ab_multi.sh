#!/usr/bin/env bash
# A/B of the default library against several ab_tmp/<VAR> builds (run on the GPU box):
#   VARS="crit3 warp" CFGS="wan14b_720p cogvideox5b" bash tools/ab_multi.sh
# Each variant first runs the d = 64 / d = 128 tensor-core parity cases (KSEL), then all
# libraries are timed in interleaved rounds (tools/lib_time.py, min of REPS x 10 launches).
set -u
B=paper_2604_12219_b200/lib/libpasa.so
for V in $VARS; do
  echo "$V parity: $(PASA_LIB=ab_tmp/$V/lib/libpasa.so timeout 400 python -m pytest tests/test_gpu_parity.py -q -x \
      -k "${KSEL:-tc_d128_4100_g32 or tc_d64_4100_g32 or tc_d128_odd_k or tc_d64_g16 or repeat_finite_bitwise and default}" 2>&1 | tail -1)"
done
for c in ${CFGS:-wan14b_720p}; do
  for r in $(seq ${ROUNDS:-2}); do
    for L in $B $(for V in $VARS; do echo ab_tmp/$V/lib/libpasa.so; done); do
      PASA_LIB=$L CFG=$c REPS=${REPS:-4} timeout 300 python tools/lib_time.py
    done
  done
done
