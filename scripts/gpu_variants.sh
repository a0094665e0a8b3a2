#!/usr/bin/env bash
# kernel variants: per-pass time at C5 for the default library, with the compact
# point pass off, and for each library in _lib/variants; then parity + C5 bench
echo "default"; timeout 300 python scripts/dev_passes.py 2>&1 | tail -2
echo "SSFM_FACTORED_POINT=0"; SSFM_FACTORED_POINT=0 timeout 300 python scripts/dev_passes.py 2>&1 | tail -2
for f in paper_2510_13310_b200/_lib/variants/*.so; do
  echo "$(basename $f)"; SSFM_LIB_PATH=$PWD/$f timeout 300 python scripts/dev_passes.py 2>&1 | tail -2
done
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x 2>&1 | tail -2
for f in 1 0; do
  SSFM_FACTORED_POINT=$f timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 6 > gpurun_out/fq.json 2>gpurun_out/fq.err
  python -c "
import json; b=json.load(open('gpurun_out/fq.json'))
r=b['roofline']; print('c5 factored_point=$f ms/step', round(b['ms_per_step'],3), 'lm med', b.get('lm_ms_median'), 'pcg ms/iter', round(r['kernel_ms']/r['cg_iters'],4), 'frac', r['frac'], b.get('cg_iters_per_step'))" || tail -5 gpurun_out/fq.err
done
