python -c "from paper_2604_12219_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stats.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 900 python -m paper_2604_12219_b200.sweep --S 16384 --H 4 --D 128 --seeds 4 --out gpurun_out/sweep_corr.json > /dev/null 2> gpurun_out/sweep.err; tail -3 gpurun_out/sweep.err
timeout 900 python -m paper_2604_12219_b200.sweep --S 16384 --H 4 --D 128 --seeds 4 --generator video --out gpurun_out/sweep_video.json > /dev/null 2>> gpurun_out/sweep.err; tail -3 gpurun_out/sweep.err
python - <<'PY'
import json
for f in ("gpurun_out/sweep_corr.json","gpurun_out/sweep_video.json"):
    d=json.load(open(f)); print(f)
    for r in d["rows"]: print(r["G"], r["comp"], r["kernel"], round(r["rel_frobenius_mean"],5), round(r["rel_frobenius_std"],5), round(r["attn_ms_median"],3))
PY
