#!/usr/bin/env bash
# C4-GP: launch list (host LM loop: the non-PCG kernels one by one; the PCG graph is one unit) and ncu --set full
# of the GP point / camera passes (standalone operator kernels)
set -x
SSFM_LM_GRAPH=0 timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r2b_c4gp.csv python bench.py --config c4gp --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_r2b_c4gp.log 2>&1
python scripts/launch_table.py gpurun_out/launches_r2b_c4gp.csv 25
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gop_point|k_gop_camera" -s 2 -c 2 -o gpurun_out/ncu_r2b_gp -f python scripts/dev_gp_passes.py c4gp > gpurun_out/ncu_gp.log 2>&1
ls -la gpurun_out/*.ncu-rep
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-PTW_WL1-1.so: $L: $V/lib_-PTW_WL1-1.so: > gpurun_out/ab_wl1_c5.log 2>&1; tail -n 4 gpurun_out/ab_wl1_c5.log
