#!/usr/bin/env bash
# kernel variants: per-pass time at C5 for the default library and each library in _lib/variants
echo "default"; timeout 300 python scripts/dev_passes.py 2>&1 | tail -2
for f in paper_2510_13310_b200/_lib/variants/*.so; do
  echo "$(basename $f)"; SSFM_LIB_PATH=$PWD/$f timeout 300 python scripts/dev_passes.py 2>&1 | tail -2
done
