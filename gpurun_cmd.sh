set -x
timeout 600 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'budget|pool|scores|select|stats|attn' -c 14 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch2.log 2>&1
timeout 500 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 1 -c 1 -o gpurun_out/prof_attn2 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full2.log 2>&1
echo done
