#!/usr/bin/env bash
# round-2 profiles at C5: launch list (host LM loop so non-PCG kernels show one by one; the PCG graph is one unit)
# and ncu --set full of the linearize tile pass, the point sums and the preconditioner
set -x
SSFM_LM_GRAPH=0 timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_r2_c5.log 2>&1
timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2_c5_graph.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_r2_c5_graph.log 2>&1
SSFM_LM_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ba_k_lin_tile|ba_k_lin_points|ba_k_precond|ba_k_kobs|ba_k_cost_tile" -s 5 -c 5 -o gpurun_out/ncu_r2_c5_lin -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_lin.log 2>&1
python scripts/launch_table.py gpurun_out/launches_r2_c5.csv 20
ls -la gpurun_out/*.ncu-rep
