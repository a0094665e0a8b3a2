#!/usr/bin/env bash
# quick A/B: BA parity subset, per-pass times, C5 and C4-BA benches
timeout 600 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py -q -x 2>&1 | tail -2
timeout 300 python scripts/dev_passes.py 2>&1 | tail -2
for cfg in c5 c4ba; do
  timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/fq.json 2>gpurun_out/fq.err
  python -c "
import json; b=json.load(open('gpurun_out/fq.json'))
r=b['roofline']; print('$cfg ms/step', round(b['ms_per_step'],3), 'lm med', b.get('lm_ms_median'), 'pcg ms/iter', round(r['kernel_ms']/r['cg_iters'],4), 'frac', r['frac'], b.get('cg_iters_per_step'))" || tail -5 gpurun_out/fq.err
done
