#!/usr/bin/env bash
# One GPU measurement pass of round 2 (third session: + the Bq = 256 CTA pair, torchrun N = 1) (run on the B200 box from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/measure_round.sh'
# Writes everything under gpurun_out/; the summaries kept are copied into profiles/r02_*.
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
cat gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in wan13b_480p cogvideox5b hunyuan_720p; do
  timeout 400 python bench.py --config "$c" --no-cpu > "gpurun_out/bench_$c.json" 2> "gpurun_out/bench_$c.err"
done
timeout 400 python bench.py --qk-precision fp8 --no-cpu > gpurun_out/bench_wan14b_fp8.json 2> gpurun_out/bench_wan14b_fp8.err
timeout 400 python bench.py --bq 256 --cta-pair --no-cpu --no-dense > gpurun_out/bench_wan14b_q256_pair.json 2> gpurun_out/bench_wan14b_q256_pair.err
timeout 400 python bench.py --bq 256 --no-cpu --no-dense > gpurun_out/bench_wan14b_q256.json 2> gpurun_out/bench_wan14b_q256.err
# the zero-copy sequence-parallel path (no all-to-all; the exchange fused into PASA's kernels)
timeout 400 python bench.py --config hunyuan_720p --ulysses zc --no-cpu --no-dense > gpurun_out/bench_hunyuan_720p_zc.json 2> gpurun_out/bench_hunyuan_720p_zc.err
# the NCCL plumbing at N = 1 (init, barriers, MAX all-reduce), as the driver launches N > 1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 1 --no-cpu --no-dense > gpurun_out/bench_wan14b_torchrun1.json 2> gpurun_out/bench_wan14b_torchrun1.err
timeout 400 python bench.py --config cogvideox5b --schedule --no-cpu --no-e2e > gpurun_out/bench_cogvideox5b_schedule.json 2> gpurun_out/bench_cogvideox5b_schedule.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --config hunyuan_720p --gpus 2 --dist-backend gloo --no-cpu --steps 2 --no-dense --no-e2e > gpurun_out/bench_hy_gloo2.json 2> gpurun_out/bench_hy_gloo2.err
timeout 900 python bench.py --config wan13b_480p --gpus 2 --partition flat --dist-backend gloo --no-cpu --steps 3 --no-dense --no-e2e > gpurun_out/bench_w13_flat_gloo2.json 2> gpurun_out/bench_w13_flat_gloo2.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --no-cpu --steps 3 --no-dense --no-e2e > gpurun_out/bench_wan14b_gloo2.json 2> gpurun_out/bench_wan14b_gloo2.err
for c in wan14b_720p wan13b_480p hunyuan_720p; do CFG=$c timeout 600 python tools/scaling_emulate.py > gpurun_out/scaling_$c.txt 2>&1; done
CFG=wan13b_480p PART=heads timeout 600 python tools/scaling_emulate.py > gpurun_out/scaling_wan13b_480p_heads.txt 2>&1
# launch list (serialised, cold cache: only the shares are comparable with bench.py)
timeout 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'budget|pool|route_fused|stats|attn' -c 12 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph --no-dense > /dev/null 2>&1
# full captures: attention, the fused route kernel, the statistics pass
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 1 -c 1 \
  -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph --no-dense \
  > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'route_fused|pool_kernel|kv_stats' -s 3 -c 3 \
  -o gpurun_out/prof_aux python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph --no-dense \
  > gpurun_out/ncu_aux.log 2>&1
ls gpurun_out
