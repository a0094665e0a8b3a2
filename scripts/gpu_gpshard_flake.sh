#!/usr/bin/env bash
# same-device GP shards: flake hunt
for i in 1 2 3 4 5; do
  timeout 250 python -m pytest tests/test_gpu_dist.py -q -x -k "gp_shards or local_shards" -rf 2>&1 | grep -E "passed|failed|FAILED|in [0-9.]+s" | head -2
done
