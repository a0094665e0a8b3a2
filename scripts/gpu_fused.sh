#!/usr/bin/env bash
# round-1 fused-operator check: GPU tests, bench A/B (fused vs two-pass), launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_fused.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err
SSFM_FUSED=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_twopass.json 2> gpurun_out/bench_twopass.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:ba_k_pcg -c 3 --csv --log-file gpurun_out/pcg_fused_metrics.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/pytest_fused.log gpurun_out/pytest_gpu.log gpurun_out/bench_fused.json gpurun_out/bench_twopass.json
tail -5 gpurun_out/bench_fused.err
cat gpurun_out/pcg_fused_metrics.csv | tail -12
