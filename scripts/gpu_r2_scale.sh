#!/usr/bin/env bash
# round 2: scale parity + explicit Schur tests, then the rest of the GPU suite
set -x
timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_schur_explicit.py -m gpu -q -rA -o junit_family=legacy --junitxml=gpurun_out/junit_scale.xml > gpurun_out/pytest_scale.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_scale.py > gpurun_out/pytest_gpu.log 2>&1
grep -E "^(ba|ba_|gp) \{|passed|failed|Error" gpurun_out/pytest_scale.log | head -40
tail -15 gpurun_out/pytest_gpu.log
