#!/usr/bin/env bash
# LM-graph / host-loop bit equality after the BA and scale tests (the order that failed once)
set -x
V=paper_2510_13310_b200/_lib/variants
T="tests/test_gpu_ba.py tests/test_gpu_scale.py tests/test_gpu_lm_graph.py"
for lib in paper_2510_13310_b200/_lib/libssfm_b200.so $V/lib_-LP_V2-0.so $V/lib_-LIN_TR-0.so paper_2510_13310_b200/_lib/libssfm_b200.so $V/lib_-LP_V2-0_-PTW_V2-0.so; do
  for rep in 1 2; do
    SSFM_LIB_PATH=$lib timeout 400 python -m pytest $T -m gpu -q --timeout 200 -p no:cacheprovider > gpurun_out/dbg.log 2>&1
    tail -n 1 gpurun_out/dbg.log | sed "s#^#$(basename $lib) $rep: #"
    grep -E "^FAILED|^E  .*At index" gpurun_out/dbg.log | head -4
  done
done
