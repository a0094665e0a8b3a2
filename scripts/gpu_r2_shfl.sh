#!/usr/bin/env bash
# warp-shuffle segmented scan in the point pass (PTW_SHFL) A/B at C5, parity tests on the variant
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-PTW_SHFL-1.so: $L: $V/lib_-PTW_SHFL-1.so: > gpurun_out/ab_shfl_c5.log 2>&1; tail -n 4 gpurun_out/ab_shfl_c5.log
SSFM_LIB_PATH=$V/lib_-PTW_SHFL-1.so timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_shfl.log 2>&1; tail -n 3 gpurun_out/pytest_shfl.log
