python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; tail -c 1200 gpurun_out/bench_default.json
for c in wan13b_480p cogvideox5b hunyuan_720p; do timeout 400 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'budget|pool|scores|select|stats|attn|rowstats' -c 16 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 1 -c 1 -o gpurun_out/prof_attn5 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > gpurun_out/ncu_full5.log 2>&1
ls gpurun_out | head -50
