python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_stats.py -q -x -k variant > gpurun_out/tv.log 2>&1; tail -3 gpurun_out/tv.log
REPS=8 VARIANTS=default FLAGS=0,64 timeout 600 python tools/ablate_attn.py > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt | tail -3
