#!/usr/bin/env bash
# point-pass variants (record layout x X source) at C5 and C4; C1 fused bench; GP same-device shard stall rate
set -x
V=paper_2510_13310_b200/_lib/variants
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $V/lib_-GPM_AOS-0_-PTW_OWNERX-0.so $V/lib_-GPM_AOS-1_-PTW_OWNERX-0.so $V/lib_-GPM_AOS-1_-PTW_OWNERX-1.so $V/lib_-GPM_AOS-0_-PTW_OWNERX-1.so $V/lib_-GPM_AOS-0_-PTW_OWNERX-0.so:SSFM_WFORM=0 > gpurun_out/var_c5.log 2>&1
timeout 400 python scripts/dev_ab.py 1000 500000 8 $V/lib_-GPM_AOS-0_-PTW_OWNERX-0.so $V/lib_-GPM_AOS-1_-PTW_OWNERX-0.so $V/lib_-GPM_AOS-1_-PTW_OWNERX-1.so $V/lib_-GPM_AOS-0_-PTW_OWNERX-1.so > gpurun_out/var_c4.log 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline --steps 10 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for k in 1 2 3 4 5 6 7 8; do timeout 400 python -m pytest tests/test_gpu_dist.py -m gpu -q -x -k "gp_shards" 2>&1 | tail -2 >> gpurun_out/gpshard_loop.log; done
cat gpurun_out/var_c5.log gpurun_out/var_c4.log gpurun_out/gpshard_loop.log
cut -c1-250 gpurun_out/bench_c1.json; tail -3 gpurun_out/bench_c1.err
