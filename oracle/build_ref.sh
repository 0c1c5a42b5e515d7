#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY.  Compiles the reference's *own* propagation kernel
# (/root/reference/pkg/src/kinopax/_kernel.pyx, Cython -> C -> .so) from the
# sources where they lie, writing outputs only into oracle/_ref/ (git-ignored,
# NOT gpurun-ignored, so the built .so travels to the GPU box).  No reference
# source is copied into the repository history.
# Flags follow the reference's own build (pkg/setup.py:21): -O3 -fopenmp -ffp-contract=off.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${KPX_REFERENCE_ROOT:-/root/reference}"
SRC="$REF/pkg/src/kinopax/_kernel.pyx"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "build_ref: $SRC not present (GPU box?) - keeping prebuilt $OUT if any" >&2
  exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python3}"
NPINC="$($PY -c 'import numpy; print(numpy.get_include())')"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
EXT="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
$PY -m cython -3 "$SRC" -o "$OUT/_kernel.c" 2> "$OUT/cython.log"
/usr/bin/gcc -O3 -fopenmp -ffp-contract=off -fPIC -shared \
    -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$NPINC" -I"$PYINC" "$OUT/_kernel.c" -o "$OUT/_kernel$EXT"
rm -f "$OUT/_kernel.c"
echo "build_ref: built $OUT/_kernel$EXT"
