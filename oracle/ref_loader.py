"""TEST INFRASTRUCTURE ONLY -- loader for the *unmodified* reference package.

Only usable in the build container, where /root/reference is mounted.  It puts
the reference's ``pkg/src`` on ``sys.path`` and resolves ``kinopax._kernel`` to
the extension that ``oracle/build_ref.sh`` compiled from the reference's own
``_kernel.pyx`` into ``oracle/_ref/`` (the reference tree itself is read-only,
so the .so cannot be placed next to the sources).

Nothing in the product package imports this module; it is used by
``oracle/make_golden.py`` and by tests that are skipped when the reference is
absent (e.g. on the GPU box).
"""
from __future__ import annotations

import glob
import importlib.abc
import importlib.machinery
import importlib.util
import os
import sys

REFERENCE_ROOT = os.environ.get("KPX_REFERENCE_ROOT", "/root/reference")
_REF_SRC = os.path.join(REFERENCE_ROOT, "pkg", "src")
_HERE = os.path.dirname(os.path.abspath(__file__))


def reference_available() -> bool:
    return os.path.isfile(os.path.join(_REF_SRC, "kinopax", "planner.py"))


def ref_kernel_path():
    hits = sorted(glob.glob(os.path.join(_HERE, "_ref", "_kernel*.so")))
    return hits[0] if hits else None


class _KernelFinder(importlib.abc.MetaPathFinder):
    def find_spec(self, fullname, path=None, target=None):
        if fullname != "kinopax._kernel":
            return None
        so = ref_kernel_path()
        if so is None:
            return None
        loader = importlib.machinery.ExtensionFileLoader(fullname, so)
        return importlib.util.spec_from_file_location(fullname, so, loader=loader)


def load_reference():
    """Import and return the reference ``kinopax`` package (compiled kernel if built)."""
    if not reference_available():
        raise ImportError(f"reference not present under {REFERENCE_ROOT}")
    if not any(isinstance(f, _KernelFinder) for f in sys.meta_path):
        sys.meta_path.insert(0, _KernelFinder())
    if _REF_SRC not in sys.path:
        sys.path.insert(0, _REF_SRC)
    import kinopax  # noqa: WPS433

    return kinopax
