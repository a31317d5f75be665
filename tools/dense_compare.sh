set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
CFG=wan14b_720p DENSE_HEADS=8 SECS=4 timeout 600 python tools/power_probe.py > gpurun_out/power_dense.txt 2>&1; cat gpurun_out/power_dense.txt
MODE=dense timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dense_list.csv python tools/dense_compare.py > /dev/null 2>&1
python - > gpurun_out/dense_name.txt <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/dense_list.csv')) if len(r)>10]
hdr=rows[0]; iK=hdr.index('Kernel Name'); iV=hdr.index('Metric Value')
best=max(rows[1:], key=lambda r: float(r[iV].replace(',','')))
print(best[iK].split('(')[0].split('<')[0].split()[-1])
PY
KN=$(cat gpurun_out/dense_name.txt); echo "dense kernel: $KN"
MODE=dense timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$KN" -s 2 -c 1 -o gpurun_out/prof_dense python tools/dense_compare.py > gpurun_out/ncu_dense.log 2>&1; tail -2 gpurun_out/ncu_dense.log
