#!/usr/bin/env bash
SSFM_TMA=1 SSFM_PCG_GRAPH=1 timeout 300 python -m pytest tests/test_gpu_ba.py -x -q -k "trajectory or c1 or damped or shared" 2>&1 | tail -2
for t in 1 0; do
  SSFM_TMA=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/q.json 2>/dev/null
  python -c "
import json; b=json.load(open('gpurun_out/q.json'))
print('c5 tma=$t ms/step', round(b['ms_per_step'],3), 'pcg ms/iter', round(b['roofline']['kernel_ms']/b['roofline']['cg_iters'],4), 'frac', b['roofline']['frac'], b['cg_iters_per_step'])"
done
