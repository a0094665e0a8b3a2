#!/usr/bin/env bash
# Build the UNMODIFIED reference package (sparsesfm, Python + one Cython/OpenMP
# extension) from /root/reference/pkg into oracle/_ref/ (git-ignored, travels to
# the GPU box with gpurun). Test/bench infrastructure only: the product path never
# imports it.  /root/reference is read-only, so the build runs on a copy in /tmp.
# CC=/usr/bin/gcc: the default /opt/gcc toolchain fails to link libgomp
# (SURVEY.md section 7, step 1).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference sources not present ($SRC); keeping existing $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/ssfm_ref.XXXXXX)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
mkdir -p "$OUT"
( cd "$TMP/pkg" && CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" \
    python -m pip install --no-index --no-build-isolation --no-deps -q \
    --target "$OUT" . )
rm -rf "$TMP"
python - <<PY
import sys; sys.path.insert(0, "$OUT")
import sparsesfm, sparsesfm._kernels as k
assert k._HAVE_CYTHON, "compiled backend missing"
print("oracle/_ref built:", sparsesfm.__file__, "backend", sparsesfm.kernel_backend())
PY
