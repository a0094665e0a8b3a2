#!/usr/bin/env bash
# kernel-variant libraries for A/B timing (SSFM_LIB_PATH=...); not part of the product build
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2510_13310_b200/_lib/variants
build() {
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -shared \
    --expt-relaxed-constexpr -cudart static -ldl -I include "$@" \
    paper_2510_13310_b200/csrc/ssfm.cu paper_2510_13310_b200/csrc/synth_host.cpp paper_2510_13310_b200/csrc/bal_host.cpp
}
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '_-' | tr -d 'D')
  build -o paper_2510_13310_b200/_lib/variants/lib_$name.so $v &
done
wait
ls paper_2510_13310_b200/_lib/variants
