#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_gp.py -x -q 2>&1 | tail -2
for cfg in c4gp c2gp; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/q.json 2>/dev/null
  python -c "
import json; b=json.load(open('gpurun_out/q.json'))
print('$cfg ms/step', round(b['ms_per_step'],3), 'pcg ms/iter', round(b['roofline']['kernel_ms']/max(1,b['roofline']['cg_iters']),4), 'frac', b['roofline']['frac'])"
done
