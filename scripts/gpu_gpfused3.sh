#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fused.py -x -q -k gp 2>&1 | tail -2
for cfg in c4gp c2gp; do
  for f in 1 0; do
    SSFM_FUSED=$f timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/gq.json 2>gpurun_out/gq.err
    python -c "
import json; b=json.load(open('gpurun_out/gq.json'))
r=b['roofline']; print('$cfg fused=$f ms/step', round(b['ms_per_step'],3), 'pcg ms/iter', round(r.get('kernel_ms',0)/max(r.get('cg_iters',1),1),4), 'share', r['kernel_share_of_step'], 'lm med', b.get('lm_ms_median'))" || tail -5 gpurun_out/gq.err
  done
done
