#!/usr/bin/env bash
# shard entry barrier check; GP overhead diagnosis; Fcm AoS A/B; C5 profiles; full suite
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 1200 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -s --timeout 240 2>&1 | grep -E "ssfm comm|passed|failed|Error" > gpurun_out/dist.log
timeout 300 python scripts/dev_lm_overhead.py c4gp 10 > gpurun_out/overhead_c4gp.log 2>&1
timeout 300 python scripts/dev_lm_overhead.py c1 10 > gpurun_out/overhead_c1.log 2>&1
SSFM_LM_GRAPH=0 timeout 600 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4gp.csv python bench.py --config c4gp --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-FCM_AOS-0.so > gpurun_out/ab_fcm.log 2>&1
bash scripts/gpu_r2_prof.sh > gpurun_out/prof.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 300 --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
cat gpurun_out/dist.log gpurun_out/overhead_c4gp.log gpurun_out/overhead_c1.log gpurun_out/ab_fcm.log
python scripts/launch_table.py gpurun_out/launches_c4gp.csv 12
tail -25 gpurun_out/pytest_gpu.log
