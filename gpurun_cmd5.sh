python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/b_graph.json 2> gpurun_out/b_graph.err; tail -c 700 gpurun_out/b_graph.json; tail -3 gpurun_out/b_graph.err
timeout 600 python bench.py --no-cpu --no-e2e --no-graph --prior global > gpurun_out/b_prior.json 2> gpurun_out/b_prior.err; python -c "
import json; d=json.loads(open('gpurun_out/b_prior.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['ms_layer'])"; tail -3 gpurun_out/b_prior.err
