#!/usr/bin/env bash
# quick check: full GPU tests, then C5 / C4-GP / C4 pipeline benches
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in c5 c4gp c4; do
  timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/fq.json 2>gpurun_out/fq.err
  python -c "
import json; b=json.load(open('gpurun_out/fq.json'))
r=b.get('roofline') or {}; print('$cfg', '%.4g'%b['value'], 'ms/step', round(b['ms_per_step'],3), 'lm med', b.get('lm_ms_median'), 'frac', r.get('frac'))" || tail -5 gpurun_out/fq.err
done
