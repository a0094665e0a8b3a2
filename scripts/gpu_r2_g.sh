#!/usr/bin/env bash
# eager-loading fix for same-device shards; LIN_FRAME / GP_AOS A/B; sanitizer; GP passes; full suite
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -s --timeout 240 2>&1 | grep -E "ssfm comm|passed|failed|Error" > gpurun_out/dist.log
cat gpurun_out/dist.log
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-LIN_FRAME-1.so: > gpurun_out/ab_linframe.log 2>&1
SSFM_LIB_PATH=$V/lib_-LIN_FRAME-1.so timeout 900 python -m pytest tests/test_gpu_ba.py tests/test_gpu_scale.py tests/test_gpu_fused.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_linframe.log 2>&1
timeout 300 python scripts/dev_gp_passes.py c4gp > gpurun_out/gp_passes.log 2>&1
SSFM_LIB_PATH=$V/lib_-GP_AOS-0.so timeout 300 python scripts/dev_gp_passes.py c4gp >> gpurun_out/gp_passes.log 2>&1
timeout 300 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp.json 2> gpurun_out/bench_c4gp.err
SSFM_LIB_PATH=$V/lib_-GP_AOS-0.so timeout 300 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp_soa.json 2> gpurun_out/bench_c4gp_soa.err
bash scripts/gpu_sanitize.sh > gpurun_out/sanitize.out 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 300 --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
cat gpurun_out/ab_linframe.log; tail -3 gpurun_out/pytest_linframe.log; cat gpurun_out/gp_passes.log
grep timed gpurun_out/bench_c4gp*.err
tail -12 gpurun_out/sanitize.out
tail -25 gpurun_out/pytest_gpu.log
