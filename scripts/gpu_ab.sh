#!/usr/bin/env bash
# A/B of kernel-variant libraries at one problem shape (one GPU call):
#   bash scripts/build_variants.sh "-DFLAG=0" ...          (here, before the call)
#   gpurun -- 'bash scripts/gpu_ab.sh 5000 2000000 10 out.log variants/lib_-FLAG-0.so ...'
# Each library runs twice, interleaved with the default build (scripts/dev_ab.py); the
# log lines name the variant. The r2b logs under profiles/ were made this way.
set -x
C=$1; P=$2; K=$3; OUT=$4; shift 4
L=paper_2510_13310_b200/_lib/libssfm_b200.so
V=paper_2510_13310_b200/_lib/variants
SPECS="$L:"
for v in "$@"; do SPECS="$SPECS $V/$v:"; done
timeout 1500 python scripts/dev_ab.py $C $P $K $SPECS $L: > gpurun_out/$OUT 2>&1
grep -v "^\[" gpurun_out/$OUT | cut -c1-220
