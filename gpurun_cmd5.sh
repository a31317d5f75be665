python -c "from paper_2604_12219_b200 import build; build.build()" > /dev/null 2>&1
VARIANTS=default FLAGS=0,0,0,1,2,3 timeout 300 python tools/ablate_attn.py 2>&1 | tail -6
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
