#!/usr/bin/env bash
for i in 1 2 3; do
s=$(date +%s); timeout 300 python -m pytest tests/test_gpu_dist.py -q -x 2>&1 | grep -E "^E  |passed|failed" | head -4; echo "$(( $(date +%s) - s )) s"
done
