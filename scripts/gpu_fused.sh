#!/usr/bin/env bash
# fused-operator check: GPU tests, CG-count diagnostic, bench A/B, launch metrics
set -x
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_fused.log
timeout 300 python scripts/dev_cgcounts.py > gpurun_out/cgcounts.log 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:ba_k_pcg -c 2 --csv --log-file gpurun_out/pcg_fused_metrics.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/pytest_fused.log gpurun_out/cgcounts.log gpurun_out/pytest_gpu.log gpurun_out/bench_fused.json
tail -3 gpurun_out/bench_fused.err
grep -o '"Metric Name.*\|"[a-z_]*__[a-z_.]*","[a-z]*","[0-9.]*"' gpurun_out/pcg_fused_metrics.csv | tail -8
