#!/usr/bin/env bash
# stall fix check (dist tests), KOBS/GVEC A/B, pass variants, GP LM-graph overhead, full suite (per-test timeout)
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -s --timeout 240 2>&1 | grep -E "ssfm comm|passed|failed|Error" > gpurun_out/dist.log
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $L:SSFM_KOBS=0 $L:SSFM_GVEC=0 $V/lib_-PTW_CIEARLY-1.so $V/lib_-CAMF_UNROLL-4.so $V/lib_-CAMF_MINB-3.so > gpurun_out/ab_c5.log 2>&1
SSFM_TIMING=1 timeout 300 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp.json 2> gpurun_out/bench_c4gp.err
SSFM_LM_GRAPH=0 timeout 300 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp_host.json 2> gpurun_out/bench_c4gp_host.err
SSFM_GVEC=0 SSFM_TIMING=1 timeout 300 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp_nogvec.json 2> gpurun_out/bench_c4gp_nogvec.err
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 300 --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
cat gpurun_out/dist.log gpurun_out/ab_c5.log
grep -E "timed|build" gpurun_out/bench_c4gp*.err
tail -25 gpurun_out/pytest_gpu.log
