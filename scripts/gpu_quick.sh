#!/usr/bin/env bash
timeout 300 python scripts/dev_passes.py 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/q.json 2>/dev/null
python -c "
import json; b=json.load(open('gpurun_out/q.json'))
print('c5 ms/step', round(b['ms_per_step'],3), 'pcg ms/iter', round(b['roofline']['kernel_ms']/b['roofline']['cg_iters'],4), 'frac', b['roofline']['frac'])"
