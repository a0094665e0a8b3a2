#!/usr/bin/env bash
# back-substitution through the pipelined point pass (ba_k_backsub_w) vs HEAD, + GPU tests
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_head.so: $L: $V/lib_head.so: > gpurun_out/ab6_c5.log 2>&1; grep -v "^\[" gpurun_out/ab6_c5.log | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py tests/test_gpu_fused.py tests/test_gpu_failure_paths.py tests/test_gpu_arena.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_ab6.log 2>&1; tail -n 2 gpurun_out/pytest_ab6.log
