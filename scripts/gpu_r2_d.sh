#!/usr/bin/env bash
# cluster vector-phase kernel A/B; stall fix (shard loop); full suite; benches; PCG traffic capture
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
timeout 600 python scripts/dev_ab.py 5000 2000000 10 $L: $L:SSFM_GVEC=0 > gpurun_out/gvec_c5.log 2>&1
timeout 300 python scripts/dev_ab.py 1000 500000 8 $L: $L:SSFM_GVEC=0 > gpurun_out/gvec_c4.log 2>&1
timeout 300 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp.json 2> gpurun_out/bench_c4gp.err
SSFM_GVEC=0 timeout 300 python bench.py --config c4gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c4gp_nogvec.json 2> gpurun_out/bench_c4gp_nogvec.err
for k in 1 2 3 4 5; do timeout 400 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -s -k "gp_shards or shared_focal" 2>&1 | grep -E "ssfm comm|passed|failed" >> gpurun_out/gpshard_loop2.log; done
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_c5.csv python scripts/dev_pcg_traffic.py c5 > gpurun_out/traffic_c5.log 2>&1
cat gpurun_out/gvec_c5.log gpurun_out/gvec_c4.log gpurun_out/gpshard_loop2.log
tail -20 gpurun_out/pytest_gpu.log
cut -c1-200 gpurun_out/bench_c4gp*.json gpurun_out/bench_c5.json
cat gpurun_out/traffic_c5.log
