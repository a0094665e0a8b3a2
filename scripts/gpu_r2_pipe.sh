#!/usr/bin/env bash
# index prefetch (PTW_PIPE / CAMF_PF / GP_PIPE) and DMMA group sums (SSFM_MMA) A/B at C5 and C4-GP;
# the new GPU tests first, then the GPU suite and benches
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 600 python -m pytest tests/test_gpu_mma.py tests/test_gpu_lm_graph.py tests/test_gpu_fused.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_new.log 2>&1
tail -5 gpurun_out/pytest_new.log
timeout 1500 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-PTW_PIPE-0_-CAMF_PF-0_-GP_PIPE-0_-LIN_MMA-0_-PRE_MMA-0.so: $L:SSFM_MMA=0 $V/lib_-CAMF_PF-0.so: $V/lib_-PTW_PIPE-0.so: $V/lib_-PTW_L2PF-1.so: $V/lib_-CAMF_L2PF-1.so: $V/lib_-PTW_L2PF-1_-CAMF_L2PF-1.so: $L: > gpurun_out/ab_pipe_c5.log 2>&1
tail -8 gpurun_out/ab_pipe_c5.log
timeout 300 python scripts/dev_gp_passes.py c4gp > gpurun_out/gp_pipe_new.log 2>&1
SSFM_LIB_PATH=$V/lib_-PTW_PIPE-0_-CAMF_PF-0_-GP_PIPE-0_-LIN_MMA-0_-PRE_MMA-0.so timeout 300 python scripts/dev_gp_passes.py c4gp > gpurun_out/gp_pipe_old.log 2>&1
tail -3 gpurun_out/gp_pipe_*.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c4gp c4ba c4 c1; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
cut -c1-300 gpurun_out/bench_*.json
