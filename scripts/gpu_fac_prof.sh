#!/usr/bin/env bash
mkdir -p gpurun_out
for f in 1 0; do echo "factored=$f"; SSFM_FACTORED=$f timeout 300 python scripts/dev_passes.py 2>&1 | tail -2; done
SSFM_FACTORED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_op_point -s 2 -c 1 -o gpurun_out/fac_point -f python scripts/dev_passes.py > gpurun_out/ncu1.log 2>&1
SSFM_FACTORED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_op_camera -s 2 -c 1 -o gpurun_out/fac_camera -f python scripts/dev_passes.py > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
