#!/usr/bin/env bash
# TMA-bulk point pass variants at C5 / C4; parity tests on the bulk variant; GP shard stall diagnostics
set -x
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $V/lib_-PTW_BULK-0.so $V/lib_-PTW_BULK-1.so $V/lib_-PTW_BULK-1_-PTP_THREAS-128.so $V/lib_-PTW_BULK-1_-PTW_BULK_CI-1_-PTP_THREAS-128.so > gpurun_out/bulk_c5.log 2>&1
timeout 400 python scripts/dev_ab.py 1000 500000 8 $V/lib_-PTW_BULK-0.so $V/lib_-PTW_BULK-1.so $V/lib_-PTW_BULK-1_-PTP_THREAS-128.so $V/lib_-PTW_BULK-1_-PTW_BULK_CI-1_-PTP_THREAS-128.so > gpurun_out/bulk_c4.log 2>&1
SSFM_LIB_PATH=$V/lib_-PTW_BULK-1_-PTW_BULK_CI-1_-PTP_THREAS-128.so timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py -m gpu -q -x > gpurun_out/pytest_bulk.log 2>&1
for k in 1 2 3 4 5 6; do timeout 400 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -s -k "gp_shards" 2>&1 | grep -E "ssfm comm|passed|failed" >> gpurun_out/gpshard_loop.log; done
cat gpurun_out/bulk_c5.log gpurun_out/bulk_c4.log; tail -3 gpurun_out/pytest_bulk.log; cat gpurun_out/gpshard_loop.log
