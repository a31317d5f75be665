# round-1 measurement pass: tests, bench lines, launch list, ncu captures
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; tail -c 1500 gpurun_out/bench_default.json
for c in wan13b_480p cogvideox5b hunyuan_720p; do timeout 400 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; tail -c 600 gpurun_out/bench_ref.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 1 -c 1 -o gpurun_out/prof_attn4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'stats|select|scores|pool' -s 4 -c 4 -o gpurun_out/prof_aux4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_aux4.log 2>&1
ls -la gpurun_out/
