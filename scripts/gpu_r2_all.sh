#!/usr/bin/env bash
# round 2: full GPU suite (junit carries the scale-parity numbers), smoke, C5 bench, C1/C2/C4 benches
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/nvsmi.txt
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=25 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c1 c2gp c4ba c4gp c4 c3; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
tail -40 gpurun_out/pytest_gpu.log
cat gpurun_out/bench_*.json | cut -c1-400
