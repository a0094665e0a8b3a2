#!/usr/bin/env bash
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ba_k_pcg -c 1 -o gpurun_out/q_pcg_c4 -f python bench.py --config c4ba --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_ncu.log 2>&1
tail -2 gpurun_out/q_ncu.log
