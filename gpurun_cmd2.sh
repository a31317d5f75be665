timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench3.json 2>gpurun_out/bench3.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'budget|pool|scores|select|stats|attn|rowstats' -c 16 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
