python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_prior.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-e2e --no-graph --prior global --steps 5 > gpurun_out/b_prior.json 2> gpurun_out/b_prior.err; python -c "
import json; d=json.loads(open('gpurun_out/b_prior.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['ms_layer'])"; tail -3 gpurun_out/b_prior.err
