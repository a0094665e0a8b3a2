#!/usr/bin/env bash
# one GPU call: the new tests first, A/B of the index prefetch vs the baseline variant at C5, the GPU suite
# (junit), smoke(), the C5 bench and the C4-BA / C4-GP / C4 / C1 / C2 / C3 bench lines
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/nvsmi.txt
timeout 600 python -m pytest tests/test_gpu_mma.py -m gpu -q -x --timeout 300 > gpurun_out/pytest_new.log 2>&1; tail -3 gpurun_out/pytest_new.log
timeout 900 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-PTW_PIPE-0_-CAMF_PF-0_-GP_PIPE-0.so: $L: > gpurun_out/ab_c5.log 2>&1; tail -3 gpurun_out/ab_c5.log
timeout 300 python scripts/dev_gp_passes.py c4gp > gpurun_out/gp_new.log 2>&1
SSFM_LIB_PATH=$V/lib_-PTW_PIPE-0_-CAMF_PF-0_-GP_PIPE-0.so timeout 300 python scripts/dev_gp_passes.py c4gp > gpurun_out/gp_old.log 2>&1
tail -n 3 gpurun_out/gp_new.log gpurun_out/gp_old.log
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 300 --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
tail -n 25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c4ba c4gp c4 c1 c2gp c3; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
cut -c1-300 gpurun_out/bench_*.json
