#!/usr/bin/env bash
# C5 launch list of the final build with the host LM loop (the non-PCG kernels one by one)
set -x
SSFM_LM_GRAPH=0 timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2d_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_r2d_c5.log 2>&1
python scripts/launch_table.py gpurun_out/launches_r2d_c5.csv 16
