#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (/root/reference/pkg, `kinopax`) with its own compiled kernel into
# baseline/_ref/ (git-ignored, NOT gpurun-ignored: it travels to the GPU box).  `bench.py --impl reference` and the
# `cpu_baseline.reference_unmodified` leg import it from there and time the reference's own plan() on host cores.
# The reference tree is read-only and its setup.py writes the cythonized C file next to the .pyx, so the install
# runs from a copy under /tmp; /usr/bin/gcc is named because the image's default gcc cannot link OpenMP.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${KPX_REFERENCE_ROOT:-/root/reference}"
if [ ! -f "$REF/pkg/setup.py" ]; then
  echo "install_ref: $REF/pkg not present (GPU box?) - keeping prebuilt $HERE/_ref if any" >&2
  exit 0
fi
PY="${PYTHON:-python3}"
if [ -f "$HERE/_ref/kinopax/planner.py" ] && ls "$HERE/_ref/kinopax/"_kernel*.so >/dev/null 2>&1; then
  echo "install_ref: $HERE/_ref already holds the reference with its compiled kernel"
  exit 0
fi
TMP="$(mktemp -d /tmp/kpx_refpkg.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF/pkg" "$TMP/pkg"
rm -rf "$HERE/_ref"
CC=/usr/bin/gcc LDSHARED="/usr/bin/gcc -shared" KINOPAX_REQUIRE_KERNEL=1 \
  "$PY" -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/_ref" "$TMP/pkg"
echo "install_ref: installed $("$PY" -c "import sys; sys.path.insert(0, '$HERE/_ref'); import kinopax; print(kinopax.__name__, kinopax.available_backends())")"
