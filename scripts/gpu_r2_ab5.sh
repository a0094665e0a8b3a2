#!/usr/bin/env bash
# point-pass 16-byte shared sums (PTW_V2) A/B at C5, then the ab4 test sequence (which failed once) four times
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-PTW_V2-0.so: $L: $V/lib_-PTW_V2-0.so: > gpurun_out/ab5_c5.log 2>&1; grep -v "^\[" gpurun_out/ab5_c5.log | cut -c1-200
for rep in 1 2 3 4; do
  timeout 600 python -m pytest tests/test_gpu_ba.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py tests/test_gpu_fused.py tests/test_gpu_failure_paths.py tests/test_gpu_cauchy.py -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_ab5_$rep.log 2>&1
  tail -n 1 gpurun_out/pytest_ab5_$rep.log; grep -E "^FAILED|At index" gpurun_out/pytest_ab5_$rep.log | head -4
done
