#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_gp.py -x -q 2>&1 | tail -3
for cfg in c2gp c4gp; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
  python -c "
import json; b=json.load(open('gpurun_out/q_bench.json'))
print('$cfg ms/step', round(b['ms_per_step'],2), 'pcg ms/iter', round(b['roofline']['kernel_ms']/max(b['roofline']['cg_iters'],1),4), 'frac', b['roofline']['frac'], 'share', b['roofline']['kernel_share_of_step'], 'cg', b['cg_iters_per_step'])" || tail -3 gpurun_out/q_bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv python bench.py --config c4gp --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null > gpurun_out/q_gp_launch.csv
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/q_gp_launch.csv')) if len(r)>10]
h=rows[0]; t=collections.defaultdict(float)
for r in rows[1:]:
    d=dict(zip(h,r))
    if d['Metric Name']=='gpu__time_duration.sum': t[d['Kernel Name'].split('(')[0]]+=float(d['Metric Value'])
for k,v in sorted(t.items(), key=lambda x:-x[1])[:10]: print(f"{v/1e6:9.3f} ms  {k[:60]}")
PY
