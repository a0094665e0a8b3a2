#!/usr/bin/env bash
# warp transpose-reduction of the tile-group sums (LIN_TR) in linearize / preconditioner: A/B at C5 + parity tests
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-LIN_TR-1_-LIN_MINB-2_-PRE_MINB-2.so: $V/lib_-LIN_TR-1.so: $L: $V/lib_-LIN_TR-1_-LIN_MINB-2_-PRE_MINB-2.so: > gpurun_out/ab_tr_c5.log 2>&1; tail -n 5 gpurun_out/ab_tr_c5.log
SSFM_LIB_PATH=$V/lib_-LIN_TR-1_-LIN_MINB-2_-PRE_MINB-2.so timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py tests/test_gpu_fused.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_tr.log 2>&1; tail -n 3 gpurun_out/pytest_tr.log
