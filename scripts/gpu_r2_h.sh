#!/usr/bin/env bash
# tile-group linearize / preconditioner variants; GPU suite; C5 / C4 / C1 / C2 benches
set -x
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
timeout 1200 python scripts/dev_ab.py 5000 2000000 10 $L: $V/lib_-SSFM_GRP-1.so $V/lib_-LIN_MINB-2_-PRE_MINB-2.so $V/lib_-SSFM_GRP-2_-LIN_MINB-2_-PRE_MINB-2.so > gpurun_out/ab_grp.log 2>&1
cat gpurun_out/ab_grp.log
timeout 2400 python -m pytest tests -m gpu -q -rA --timeout 300 --durations=15 -o junit_family=legacy --junitxml=gpurun_out/junit.xml > gpurun_out/pytest_gpu.log 2>&1
tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c4ba c4gp c1 c2gp c3; do timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
cut -c1-220 gpurun_out/bench_*.json
bash scripts/gpu_sanitize.sh > gpurun_out/sanitize.out 2>&1
grep -E "Read  at|Write  at|Read Thread|Write Thread" gpurun_out/sanitize_racecheck.log | sed 's/Thread ([0-9,]*)//; s/+0x[0-9a-f]*//' | sort | uniq -c | head
tail -3 gpurun_out/sanitize_racecheck.log gpurun_out/sanitize_synccheck.log gpurun_out/sanitize_memcheck.log
