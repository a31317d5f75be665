#!/usr/bin/env bash
# One GPU measurement pass (run on the B200 box via gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/measure_round.sh'
# Writes everything under gpurun_out/; copy the summaries you keep into profiles/.
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
cat gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in wan13b_480p cogvideox5b hunyuan_720p; do
  timeout 400 python bench.py --config "$c" --no-cpu > "gpurun_out/bench_$c.json" 2> "gpurun_out/bench_$c.err"
done
timeout 400 python bench.py --config cogvideox5b --schedule --no-cpu --no-e2e > gpurun_out/bench_cogvideox5b_schedule.json 2> gpurun_out/bench_cogvideox5b_schedule.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# power / clock per attention variant (the long configs run under the 1000 W cap)
timeout 300 python tools/power_probe.py > gpurun_out/power_wan14b.txt 2>&1
CFG=cogvideox5b SECS=3 timeout 200 python tools/power_probe.py > gpurun_out/power_cogvideox5b.txt 2>&1
timeout 300 python tools/q256_time.py > gpurun_out/q256_wan14b.txt 2>&1
timeout 400 python tools/energy_ablate.py > gpurun_out/energy_ablate.txt 2>&1
timeout 400 python tools/scaling_emulate.py > gpurun_out/scaling_emulate.txt 2>&1
# launch list (serialised, cold cache: only the shares are comparable with bench.py)
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:'budget|pool|scores|select|stats|attn|rowstats' -c 16 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > /dev/null 2>&1
# one full capture of the dominant kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 1 -c 1 \
  -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph \
  > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
