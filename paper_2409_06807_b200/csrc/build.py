#!/usr/bin/env python3
"""Build libkpx.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Seven translation units: the f64 parity instantiations (``-fmad=false``, the
reference is built with ``-ffp-contract=off``), the f32 throughput
instantiations, the f32 single-query (latency) instantiations, the same three
drawing from Philox4x32-10 instead of the reference's SplitMix64 streams, and the C ABI.  The shared library lands next to the Python
package (``paper_2409_06807_b200/libkpx.so``) so it travels to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(PKG, "libkpx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off", "--expt-relaxed-constexpr"]
UNITS = [
    ("kpx_inst_f64.cu", ["-fmad=false"]),
    ("kpx_inst_f32.cu", []),
    ("kpx_inst_f32lat.cu", []),
    # the same kernels drawing from Philox4x32-10 (the random stream is a compile-time property of a kernel)
    ("kpx_inst_f64p.cu", ["-fmad=false"]),
    ("kpx_inst_f32p.cu", []),
    ("kpx_inst_f32latp.cu", []),
    ("kpx_api.cu", []),
]
HEADERS = ["kpx_device.cuh", "kpx_plan.cuh", "kpx_launch.h", "kpx_inst.inl", os.path.join("..", "..", "include", "kpx.h")]


def _stale(target: str, sources) -> bool:
    if not os.path.isfile(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB, obj_dir: str = OBJ) -> str:
    """defines / lib / obj_dir let tuning scripts build side-by-side variants (e.g. -DKPX_MINB_F32_SMALL=3)."""
    OBJ, LIB = obj_dir, lib  # noqa: N806
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(HERE, h) for h in HEADERS]
    jobs = []
    for src, extra in UNITS:
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        if force or _stale(obj, [os.path.join(HERE, src)] + hdrs):
            cmd = [NVCC] + ARCH + COMMON + extra + list(defines) + (["-Xptxas", "-v"] if verbose else []) + \
                  ["-c", os.path.join(HERE, src), "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stderr

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        logs = list(ex.map(run, jobs))
    if verbose:
        for l in logs:
            sys.stderr.write(l)
    objs = [os.path.join(OBJ, s.replace(".cu", ".o")) for s, _ in UNITS]
    if jobs or force or _stale(LIB, objs):
        run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs)
    return LIB


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    tag = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--tag=")), None)
    if tag:
        print(build(force=True, verbose="-v" in sys.argv, defines=defs, lib=os.path.join(PKG, f"libkpx_{tag}.so"),
                    obj_dir=os.path.join(HERE, f"_obj_{tag}")))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs))
