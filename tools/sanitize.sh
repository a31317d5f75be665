#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck over a subset of the GPU parity tests (run on the
# B200 box from the repo root):  /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/sanitize.sh'
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export PYTEST_ADDOPTS="-p no:cacheprovider"
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/san_memcheck.txt \
  python -m pytest tests/test_gpu_parity.py -q -x -k "tc_d128_4100_g32 or tc_d64_4100_g32 or tc_d128_g8 or tc_d64_g16 or ragged1000 or iid16k or tc_d128_20000_g128 or budget" > gpurun_out/san_memcheck.log 2>&1
tail -3 gpurun_out/san_memcheck.log; grep -c "Invalid\|ERROR SUMMARY" gpurun_out/san_memcheck.txt; grep "ERROR SUMMARY" gpurun_out/san_memcheck.txt | head
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/san_memcheck2.txt \
  python -m pytest tests/test_gpu_prior.py tests/test_gpu_stats.py -q -x > gpurun_out/san_memcheck2.log 2>&1
tail -3 gpurun_out/san_memcheck2.log; grep "ERROR SUMMARY" gpurun_out/san_memcheck2.txt | head
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --log-file gpurun_out/san_race.txt \
  python -m pytest tests/test_gpu_parity.py -q -x -k "ragged1000 or iid16k or clustered" > gpurun_out/san_race.log 2>&1
tail -3 gpurun_out/san_race.log; grep "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/san_race.txt | head
# the round's attention variants: ping-pong (one CTA/SM, Q in TMEM) and Bq = 256 (two tiles)
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/san_memcheck3.txt \
  python -m pytest tests/test_gpu_parity.py -q -x -k "pingpong and (tc_d128_4100_g32 or tc_d64_4100_g32 or S65 or k1) or q256_d128_4100_g32 or q256_d64_4100_g32 or q256_d128_20000 or test_attn_q256_edges" > gpurun_out/san_memcheck3.log 2>&1
tail -3 gpurun_out/san_memcheck3.log; grep "ERROR SUMMARY" gpurun_out/san_memcheck3.txt | head
