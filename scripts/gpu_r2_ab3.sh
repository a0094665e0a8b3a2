#!/usr/bin/env bash
# A/B at C5: linearize / preconditioner index prefetch (LIN_PF), camera-pass prefetch distance (CAMF_PFD 3, 4),
# 16-CTA vector-phase cluster (GV_CL=16); parity of the default build on the BA tests; C4-GP with GV_CL=16
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 1200 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-LIN_PF-0.so: $V/lib_-CAMF_PF-3.so: $V/lib_-CAMF_PF-4.so: $V/lib_-GV_CL-16.so: $L: > gpurun_out/ab3_c5.log 2>&1; tail -n 12 gpurun_out/ab3_c5.log
timeout 300 python bench.py --config c4gp --no-cpu-baseline --no-e2e > gpurun_out/c4gp_def.json 2>&1
SSFM_LIB_PATH=$V/lib_-GV_CL-16.so timeout 300 python bench.py --config c4gp --no-cpu-baseline --no-e2e > gpurun_out/c4gp_cl16.json 2>&1
grep -h ms_per_step gpurun_out/c4gp_*.json | cut -c1-260
timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py tests/test_gpu_lm_graph.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_ab3.log 2>&1; tail -n 3 gpurun_out/pytest_ab3.log
