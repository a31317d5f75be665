python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prior.py -q -x 2>&1 | tail -2
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'select|scores|pool|rowstats' -c 8 --csv --log-file gpurun_out/launches6.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches6.csv
