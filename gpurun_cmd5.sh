python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x > gpurun_out/tpipe.log 2>&1; tail -15 gpurun_out/tpipe.log
for ch in 1 8 20; do timeout 600 python bench.py --no-cpu --no-graph --steps 5 --e2e-chunks $ch > gpurun_out/b_e2e_$ch.json 2> gpurun_out/b_e2e_$ch.err; python -c "
import json; d=json.loads(open('gpurun_out/b_e2e_$ch.json').read().strip().splitlines()[-1]); print($ch, d['ms_per_step'], d['e2e'])"; tail -2 gpurun_out/b_e2e_$ch.err; done
