#!/usr/bin/env bash
# re-entry check of HEAD: GPU suite, smoke, C5 bench, C1/C4 benches
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/nvsmi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 300 --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c4ba c4gp c4 c1 c2gp c3; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
cut -c1-300 gpurun_out/bench_*.json
