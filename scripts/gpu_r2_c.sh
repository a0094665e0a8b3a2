#!/usr/bin/env bash
# LM loop as a CUDA graph + AoS omega-form record: GPU suite, benches, ncu of the point pass
set -x
timeout 2400 python -m pytest tests -m gpu -q -rA -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
SSFM_LM_GRAPH=0 timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 10 > gpurun_out/bench_c1_host.json 2> gpurun_out/bench_c1_host.err
timeout 300 python bench.py --config c2gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c2gp.json 2> gpurun_out/bench_c2gp.err
SSFM_TIMING=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 400 python bench.py --config c4ba --no-cpu-baseline > gpurun_out/bench_c4ba.json 2> gpurun_out/bench_c4ba.err
timeout 300 python scripts/dev_passes.py > gpurun_out/passes.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_op_point -s 2 -c 1 -o gpurun_out/ncu_point -f python scripts/dev_passes.py > gpurun_out/ncu1.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
cut -c1-200 gpurun_out/bench_*.json
cat gpurun_out/passes.log
