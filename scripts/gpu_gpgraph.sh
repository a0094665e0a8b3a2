#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x -k "gp" 2>&1 | tail -2
for cfg in c4gp c2gp; do
for mode in "SSFM_FUSED=1" "SSFM_FUSED=0 SSFM_GP_GRAPH=0" "SSFM_FUSED=0 SSFM_GP_GRAPH=1"; do
  env $mode timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/fq.json 2>gpurun_out/fq.err
  python -c "
import json; b=json.load(open('gpurun_out/fq.json'))
r=b['roofline']; print('$cfg $mode ms/step', round(b['ms_per_step'],3), 'lm med', b.get('lm_ms_median'), 'pcg ms/iter', round(r['kernel_ms']/r['cg_iters'],4), b.get('cg_iters_per_step'))" || tail -5 gpurun_out/fq.err
done
done
