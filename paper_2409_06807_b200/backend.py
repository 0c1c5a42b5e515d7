"""The reference's backend seam, served by the CUDA kernel.

Reference ``backend.py`` resolves a name to an object with ``.name`` and
``.propagate_batch(ctx, states, e_slots, lam, iteration) -> Batch``
(``backend.py:47-122``).  This module keeps ``PlanContext`` and ``Batch`` field
for field and registers two CUDA backends behind the same call:

* ``"cuda"``      -- float64 instantiation, bit-parity with the reference kernel,
* ``"cuda-f32"``  -- float32 instantiation (end states within 1e-5 relative),
* ``"cuda-philox"`` / ``"cuda-f32-philox"`` -- the same kernels drawing from the production Philox4x32-10 stream
  instead of the reference's SplitMix64 chains (other random numbers, hence other trees: not a parity mode).

``KINOPAX_BACKEND`` overrides the default exactly as in the reference.  Unknown
names and models without a CUDA kernel raise ``ConfigError``; a missing
``libkpx.so`` raises ``DeviceError`` -- there is no silent CPU path.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import ConfigError
from .dynamics import DynamicsModel


@dataclass(frozen=True)
class PlanContext:
    model: DynamicsModel
    seed: int
    t_prop: float
    state_lo: np.ndarray
    state_hi: np.ndarray
    obs_min: np.ndarray
    obs_max: np.ndarray
    check_res: float
    grid_lo: np.ndarray
    grid_width: np.ndarray
    grid_cells: np.ndarray
    grid_strides: np.ndarray
    subcells: int
    threads: int = 1


@dataclass
class Batch:
    valid: np.ndarray
    region: np.ndarray
    sub: np.ndarray
    end: np.ndarray
    control: np.ndarray
    dt: np.ndarray
    accept_u: np.ndarray
    # B200 additions (None unless requested)
    substeps: np.ndarray = None
    points: np.ndarray = None
    kernel_ms: float = 0.0

    @property
    def items(self) -> int:
        return len(self.valid)


class CudaBackend:
    """``propagate_batch`` through ``kpx_propagate_batch`` (host arrays in, host arrays out)."""

    name = "cuda"
    precision = _lib.F64
    rng = _lib.RNG_SPLITMIX64      # the reference's streams; the "-philox" backends draw from Philox4x32-10 instead

    def __init__(self, counters: bool = False):
        self.counters = counters

    def propagate_batch(self, ctx: PlanContext, states: np.ndarray, e_slots: np.ndarray, lam: int,
                        iteration: int) -> Batch:
        lib = _lib.load()
        m = ctx.model
        if m.kernel_id is None:
            raise ConfigError(f"model '{m.name}' has no CUDA kernel")
        prob, keep = _lib.make_problem(
            m.kernel_id, m.n, m.control_dim, max(len(states), 1), 1, ctx.t_prop, ctx.check_res, 0.5, 1.0,
            m.control_lo, m.control_hi, ctx.state_lo, ctx.state_hi, ctx.obs_min, ctx.obs_max, ctx.grid_lo,
            ctx.grid_width, ctx.grid_cells, ctx.grid_strides, ctx.subcells, rng=self.rng)
        states = np.ascontiguousarray(states, dtype=np.float64)
        e_slots = np.ascontiguousarray(e_slots, dtype=np.int64)
        items = len(e_slots) * int(lam)
        out = Batch(valid=np.zeros(items, np.uint8), region=np.full(items, -1, np.int64),
                    sub=np.zeros(items, np.int64), end=np.zeros((items, m.n)),
                    control=np.zeros((items, m.control_dim)), dt=np.zeros(items), accept_u=np.zeros(items))
        if self.counters:
            out.substeps, out.points = np.zeros(items, np.int64), np.zeros(items, np.int64)
        ms = _lib.C.c_double(0.0)
        rc = lib.kpx_propagate_batch(
            _lib.C.byref(prob), _lib.ptr(states), states.shape[0], _lib.ptr(e_slots), len(e_slots), int(lam),
            int(ctx.seed) & 0xFFFFFFFFFFFFFFFF, int(iteration) & 0xFFFFFFFFFFFFFFFF, self.precision,
            _lib.ptr(out.valid), _lib.ptr(out.region), _lib.ptr(out.sub), _lib.ptr(out.end), _lib.ptr(out.control),
            _lib.ptr(out.dt), _lib.ptr(out.accept_u), _lib.ptr(out.substeps), _lib.ptr(out.points),
            _lib.C.byref(ms), None)
        _lib.check(rc, "kpx_propagate_batch")
        out.kernel_ms = ms.value
        del keep
        return out


class CudaF32Backend(CudaBackend):
    name = "cuda-f32"
    precision = _lib.F32


class CudaPhiloxBackend(CudaBackend):
    name = "cuda-philox"
    rng = _lib.RNG_PHILOX


class CudaF32PhiloxBackend(CudaF32Backend):
    name = "cuda-f32-philox"
    rng = _lib.RNG_PHILOX


_BACKENDS = {"cuda": CudaBackend, "cuda-f32": CudaF32Backend, "cuda-philox": CudaPhiloxBackend,
             "cuda-f32-philox": CudaF32PhiloxBackend}


def cuda_available() -> bool:
    return os.path.isfile(_lib.LIB_PATH)


def available_backends() -> list:
    return list(_BACKENDS) if cuda_available() else []


def get_backend(name=None, model=None):
    """Explicit name -> ``KINOPAX_BACKEND`` -> ``"cuda"`` (reference ``backend.py:103-122``)."""
    if name is None:
        name = os.environ.get("KINOPAX_BACKEND")
    if name is None:
        name = "cuda"
    if name not in _BACKENDS:
        raise ConfigError(f"unknown backend '{name}' (choose from {list(_BACKENDS)})")
    if model is not None and model.kernel_id is None:
        raise ConfigError(f"model '{model.name}' has no CUDA kernel")
    _lib.load()  # fail loudly now if the extension is not built
    return _BACKENDS[name]()


def precision_of(backend_name) -> int:
    return get_backend(backend_name).precision
