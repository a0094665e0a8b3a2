#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_ba.py tests/test_gpu_gp.py -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ba_k_precond|ba_k_linearize_cm|ba_k_linearize" -c 6 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | cut -c1-80
