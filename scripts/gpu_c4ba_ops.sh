#!/usr/bin/env bash
# C4-BA / C3: fused persistent (default) vs two-pass factored graph
for cfg in c4ba c3; do
for f in 1 0; do
  SSFM_FUSED=$f timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 8 > gpurun_out/fq.json 2>gpurun_out/fq.err
  python -c "
import json; b=json.load(open('gpurun_out/fq.json'))
r=b['roofline']; print('$cfg fused=$f ms/step', round(b['ms_per_step'],3), 'lm med', b.get('lm_ms_median'), 'pcg ms/iter', round(r['kernel_ms']/r['cg_iters'],4), 'frac', r['frac'], b.get('cg_iters_per_step'))" || tail -5 gpurun_out/fq.err
done
done
