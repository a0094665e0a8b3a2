#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -2
for cfg in c4ba c3; do
for v in "SSFM_FUSED=1"; do
  env $v timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
  python -c "
import json; b=json.load(open('gpurun_out/q_bench.json'))
print('$cfg $v', 'ms/step', round(b['ms_per_step'],2), 'pcg ms/iter', round(b['roofline']['kernel_ms']/b['roofline']['cg_iters'],4), 'frac', b['roofline']['frac'], 'cg', b['cg_iters_per_step'])" || tail -3 gpurun_out/q_bench.err
done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ba_k_pcg -c 1 -o gpurun_out/q_pcg_c4 -f python bench.py --config c4ba --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_ncu.log 2>&1
