#!/usr/bin/env bash
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/q.json 2> gpurun_out/q.err
tail -2 gpurun_out/q.err
