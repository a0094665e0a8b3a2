#!/usr/bin/env bash
# round-1 record: GPU tests, default bench (C5, e2e, CPU reference), reference arm,
# C4 pipeline / C4-GP / C4-BA benches, launch list, ncu captures of the C5
# two-pass operator passes (standalone k_op_* = the graph's body kernels), the
# C4-BA fused PCG and the C4-GP fused PCG
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config c4 --steps 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp.json 2> gpurun_out/bench_c4gp.err
timeout 600 python bench.py --config c4ba --no-cpu-baseline --steps 10 > gpurun_out/bench_c4ba.json 2> gpurun_out/bench_c4ba.err
timeout 600 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_op_point -s 2 -c 1 -o gpurun_out/op_point_c5 -f python scripts/dev_passes.py > gpurun_out/ncu_p.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_op_camera -s 2 -c 1 -o gpurun_out/op_camera_c5 -f python scripts/dev_passes.py > gpurun_out/ncu_c.log 2>&1
SSFM_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ba_k_pcg -c 1 -o gpurun_out/pcg_c4ba_full -f python bench.py --config c4ba --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
SSFM_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gp_k_pcg -c 1 -o gpurun_out/pcg_c4gp_full -f python bench.py --config c4gp --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_gp.log 2>&1
cat gpurun_out/pytest_gpu.log
