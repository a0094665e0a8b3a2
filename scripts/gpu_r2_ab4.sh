#!/usr/bin/env bash
# default (transpose-reduced tile-group sums + 16-byte shared sums in ba_k_lin_points) vs LIN_TR=0, camera pass
# at 3 CTAs per SM; then the BA / scale / LM-graph GPU tests on the default build
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-LIN_TR-0.so: $V/lib_-CAMF_MINB-3.so: $L: > gpurun_out/ab4_c5.log 2>&1; tail -n 4 gpurun_out/ab4_c5.log
timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py tests/test_gpu_fused.py tests/test_gpu_failure_paths.py tests/test_gpu_cauchy.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_ab4.log 2>&1; tail -n 3 gpurun_out/pytest_ab4.log
