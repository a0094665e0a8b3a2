#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for cfg in c5 c3 c1; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
  python -c "
import json; b=json.load(open('gpurun_out/q_bench.json'))
print('$cfg ms/step', round(b['ms_per_step'],3), 'pcg ms/iter', round(b['roofline']['kernel_ms']/b['roofline']['cg_iters'],4), 'frac', b['roofline']['frac'], 'cg', b['cg_iters_per_step'])"
done
