#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_ba.py -x -q -k "reproj or pipeline or shared or c1" 2>&1 | tail -3
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
cut -c1-900 gpurun_out/bench_c4.json; tail -2 gpurun_out/bench_c4.err
