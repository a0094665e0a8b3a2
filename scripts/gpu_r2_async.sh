#!/usr/bin/env bash
# cp.async-staged point pass (PTW_ASYNC) A/B at C5 and C4-BA, and its parity: the GPU BA tests on the variant
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-PTW_ASYNC-1.so: $V/lib_-PTW_ASYNC-1_-PTP_MINB-3.so: $L: > gpurun_out/ab_async_c5.log 2>&1; tail -n 4 gpurun_out/ab_async_c5.log
timeout 600 python scripts/dev_ab.py 1000 500000 8 $L: $V/lib_-PTW_ASYNC-1.so: > gpurun_out/ab_async_c4.log 2>&1; tail -n 2 gpurun_out/ab_async_c4.log
SSFM_LIB_PATH=$V/lib_-PTW_ASYNC-1.so timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_async.log 2>&1; tail -n 3 gpurun_out/pytest_async.log
