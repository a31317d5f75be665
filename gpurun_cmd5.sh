python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
VARIANTS=default FLAGS=0,0,0,3 timeout 300 python tools/ablate_attn.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stats.py -q -x 2>&1 | tail -2
