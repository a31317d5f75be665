python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
VARIANTS=default FLAGS=0,0,0 timeout 300 python tools/ablate_attn.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stats.py -q -x 2>&1 | tail -2
timeout 300 python tools/trace_attn.py 100 20 > gpurun_out/tr0.txt 2>&1; grep -A12 "v1 ops" gpurun_out/tr0.txt
