#!/usr/bin/env bash
set -x
timeout 1500 python -m pytest tests/test_gpu_failure_paths.py tests/test_gpu_scale.py tests/test_gpu_schur_explicit.py tests/test_gpu_dist.py -m gpu -q -rA -s > gpurun_out/pytest_b.log 2>&1
grep -E "^(ba|ba_|gp) \{|world|passed|failed|Error|assert" gpurun_out/pytest_b.log | head -60
