#!/usr/bin/env bash
# quick check: full GPU tests, then C5 (with and without the factored record) / C4-BA benches
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for mode in "SSFM_FACTORED=1" "SSFM_FACTORED=0"; do
for cfg in c5 c4ba; do
  env $mode timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/fq.json 2>gpurun_out/fq.err
  python -c "
import json; b=json.load(open('gpurun_out/fq.json'))
r=b.get('roofline') or {}; print('$cfg $mode', '%.4g'%b['value'], 'ms/step', round(b['ms_per_step'],3), 'lm med', b.get('lm_ms_median'), 'frac', r.get('frac'), b.get('cg_iters_per_step'))" || tail -5 gpurun_out/fq.err
done
done
