#!/usr/bin/env bash
# camera-pass variants: per-pass time at C5 for each library in _lib/variants
echo "default"; timeout 300 python scripts/dev_passes.py 2>&1 | tail -1
for f in paper_2510_13310_b200/_lib/variants/*.so; do
  echo "$(basename $f)"; SSFM_LIB_PATH=$PWD/$f timeout 300 python scripts/dev_passes.py 2>&1 | tail -1
done
