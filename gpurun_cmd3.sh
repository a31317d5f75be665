python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
VARIANTS=default FLAGS=0,4,3,7 timeout 300 python tools/ablate_attn.py > gpurun_out/abl3.log 2>&1
cat gpurun_out/abl3.log | tail -4
for f in 0 3; do FLAGS=$f timeout 300 python tools/trace_attn.py 100 20 > gpurun_out/tr$f.txt 2>&1; done
