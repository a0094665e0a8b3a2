#!/usr/bin/env bash
# GP fused operator: parity tests, then c4gp / c2gp fused vs two-pass
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_gp.py tests/test_gpu_dist.py -x -q 2>&1 | tail -15
for cfg in c4gp c2gp; do
  for f in 0 1; do
    SSFM_FUSED=$f timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/gq.json 2>gpurun_out/gq.err
    python -c "
import json; b=json.load(open('gpurun_out/gq.json'))
r=b['roofline']; print('$cfg fused=$f ms/step', round(b['ms_per_step'],3), 'pcg ms/iter', round(r.get('kernel_ms',0)/max(r.get('cg_iters',1),1),4), 'frac', r['frac'], b.get('cg_iters_per_step'))" || tail -5 gpurun_out/gq.err
  done
done
