#!/usr/bin/env bash
# factored camera pass: parity, per-pass times, then C5 factored vs Jacobian records
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ba.py tests/test_gpu_dist.py -x -q 2>&1 | tail -6
for f in 1 0; do echo "factored=$f"; SSFM_FACTORED=$f timeout 300 python scripts/dev_passes.py 2>&1 | tail -2; done
for f in 1 0; do
  SSFM_FACTORED=$f timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/fq.json 2>gpurun_out/fq.err
  python -c "
import json; b=json.load(open('gpurun_out/fq.json'))
r=b['roofline']; print('c5 factored=$f ms/step', round(b['ms_per_step'],3), 'lm med', b.get('lm_ms_median'), 'pcg ms/iter', round(r['kernel_ms']/r['cg_iters'],4), 'frac', r['frac'], b.get('cg_iters_per_step'))" || tail -5 gpurun_out/fq.err
done
