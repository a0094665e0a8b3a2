#!/usr/bin/env bash
# the NVML clock sampler: C4-GP, C4 pipeline and C5 bench lines (host stalls in the timed regions?)
set -x
for c in c4gp c4 c1; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/s_$c.json 2> gpurun_out/s_$c.err; tail -n 3 gpurun_out/s_$c.err | cut -c1-160; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s_c5.json 2> gpurun_out/s_c5.err; tail -n 3 gpurun_out/s_c5.err | cut -c1-160
cut -c1-200 gpurun_out/s_*.json; grep -o '"clocks": {[^}]*}' gpurun_out/s_*.json
