#!/usr/bin/env bash
# round-2 record: GPU suite (junit), smoke(), the C5 bench (+ reference arm), the other bench configs,
# the PCG DRAM traffic per CG iteration and the C5 launch list of the final build
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/nvsmi.txt
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 300 --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
tail -n 6 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c4ba c4gp c4 c1 c2gp c3; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cut -c1-250 gpurun_out/bench_*.json
timeout 900 ncu --graph-profiling graph --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_r2c_c5.csv python scripts/dev_pcg_traffic.py c5 > gpurun_out/traffic_r2c_c5.log 2>&1
tail -n 2 gpurun_out/traffic_r2c_c5.log
timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2c_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_r2c_c5.log 2>&1
