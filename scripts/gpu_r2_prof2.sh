#!/usr/bin/env bash
# after the index prefetch + DMMA change: ncu --set full of the C5 operator passes (standalone k_op_* = the graph's
# body kernels) and of the DMMA linearize / preconditioner kernels, the PCG DRAM traffic per CG iteration, and
# the C5 launch list (host LM loop so the non-PCG kernels show one by one)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_op_point -s 2 -c 1 -o gpurun_out/ncu_r2b_point -f python scripts/dev_passes.py > gpurun_out/ncu_p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_op_camera -s 2 -c 1 -o gpurun_out/ncu_r2b_camera -f python scripts/dev_passes.py > gpurun_out/ncu_c.log 2>&1
SSFM_LM_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"ba_k_lin_tile|ba_k_precond_grp|ba_k_lin_points" -s 3 -c 3 -o gpurun_out/ncu_r2b_lin -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_lin.log 2>&1
timeout 900 ncu --graph-profiling graph --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_r2b_c5.csv python scripts/dev_pcg_traffic.py c5 > gpurun_out/traffic_r2b_c5.log 2>&1
SSFM_LM_GRAPH=0 timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2b_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_r2b_c5.log 2>&1
python scripts/launch_table.py gpurun_out/launches_r2b_c5.csv 20
tail -3 gpurun_out/traffic_r2b_c5.log
ls -la gpurun_out/*.ncu-rep
