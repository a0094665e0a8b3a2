#!/usr/bin/env bash
# AoS omega-form point pass + one-evaluation linearize: A/B, GPU suite, C5 bench
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
timeout 600 python scripts/dev_ab.py 5000 2000000 10 $L: $L:SSFM_LIN2=0 $L:SSFM_WFORM=0 > gpurun_out/ab_c5.log 2>&1
timeout 300 python scripts/dev_ab.py 1000 500000 8 $L: $L:SSFM_LIN2=0 $L:SSFM_WFORM=0 > gpurun_out/ab_c4.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -rA -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
SSFM_TIMING=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
cat gpurun_out/ab_c5.log gpurun_out/ab_c4.log
tail -5 gpurun_out/pytest_gpu.log
cut -c1-300 gpurun_out/bench_c5.json
