#!/usr/bin/env bash
# round 2: GPU test suite (junit properties carry the scale-parity numbers) + C1/C2 latency benches
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} -o junit_family=legacy --junitxml=gpurun_out/junit.xml 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --config c2gp --no-cpu-baseline --steps 10 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
cat gpurun_out/pytest_gpu.log
