#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over the GPU parity tests (run on the
# B200 box from the repo root):  /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/sanitize.sh'
# SURVEY.md §4.2 T6.  Small shapes only: the sanitizers slow kernels down ~100x.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export PYTEST_ADDOPTS="-p no:cacheprovider"
ATTN="tc_d128_1000 or tc_d128_4100_g32 or tc_d64_4100_g32 or tc_d128_g8 or tc_d64_g16 or tc_d128_4100_zeroth or tc_d64_4100_none or S65 or k1 or q256_d128_4100_g32 or q256_d64_4100_g32"
ROUTE="ragged1000 or iid16k or clustered or budget"
run() {  # tool, log-stem, pytest -k expression, files...
  local tool=$1 stem=$2 expr=$3; shift 3
  timeout 1500 compute-sanitizer --tool "$tool" --print-limit 20 --log-file "gpurun_out/san_${stem}.txt" \
    python -m pytest "$@" -q -x -k "$expr" > "gpurun_out/san_${stem}.log" 2>&1
  echo "== $tool $stem rc=$?"; tail -2 "gpurun_out/san_${stem}.log"
  grep "ERROR SUMMARY\|RACECHECK SUMMARY\|SYNCCHECK SUMMARY" "gpurun_out/san_${stem}.txt" | sort | uniq -c | head
}
run memcheck  memcheck_attn  "$ATTN or $ROUTE" tests/test_gpu_parity.py
run racecheck racecheck_attn "$ATTN" tests/test_gpu_parity.py
run synccheck synccheck_attn "$ATTN" tests/test_gpu_parity.py
run racecheck racecheck_route "$ROUTE" tests/test_gpu_parity.py
run memcheck  memcheck_stats "kv_stats or stats" tests/test_gpu_stats.py
run racecheck racecheck_stats "kv_stats or stats" tests/test_gpu_stats.py
run synccheck synccheck_stats "kv_stats or stats" tests/test_gpu_stats.py
# round 2: the fused route kernel, the persistent statistics kernel, q-block ranges, FP8 QK^T
run memcheck  memcheck_r2 "qblock or sharded or fp8_qk_parity" tests/test_gpu_dist.py tests/test_gpu_fp8.py
run racecheck racecheck_r2 "qblock_range_equals or fp8_qk_parity" tests/test_gpu_dist.py tests/test_gpu_fp8.py
run synccheck synccheck_r2 "qblock_range_equals or fp8_qk_parity" tests/test_gpu_dist.py tests/test_gpu_fp8.py
