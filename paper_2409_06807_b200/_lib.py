"""ctypes binding of ``libkpx.so`` (the C ABI in ``include/kpx.h``).

There is deliberately no fallback: if the shared library is missing or an entry
point fails, a ``DeviceError`` is raised.  The product path never routes through
the CPU oracle.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .core import ConfigError, DeviceError

MAX_DIM, MAX_CONTROL, MAX_CHAIN = 48, 24, 4096
F64, F32 = 0, 1
RNG_SPLITMIX64, RNG_PHILOX = 0, 1
SOLVED, TIMEOUT, CAPACITY_EXHAUSTED, ERROR, RUNNING, STOPPED = range(6)
E_ARG, E_CUDA, E_LIMIT, E_STATE = 1, 2, 3, 4

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KPX_LIB_PATH") or os.path.join(_PKG, "libkpx.so")   # override: tuning variants only

_vp = C.c_void_p


class Problem(C.Structure):
    _fields_ = [
        ("model_id", C.c_int32), ("n", C.c_int32), ("nu", C.c_int32), ("n_obs", C.c_int32),
        ("subcells", C.c_int32), ("grid_n", C.c_int32), ("lambda_max", C.c_int32), ("rng", C.c_int32),
        ("t_e", C.c_int64), ("t_e_start", C.c_int64), ("t_e_growth", C.c_double),
        ("t_prop", C.c_double), ("check_res", C.c_double), ("epsilon", C.c_double), ("delta", C.c_double),
        ("control_lo", C.c_double * MAX_CONTROL), ("control_hi", C.c_double * MAX_CONTROL),
        ("state_lo", C.c_double * MAX_DIM), ("state_hi", C.c_double * MAX_DIM),
        ("grid_lo", C.c_double * MAX_DIM), ("grid_width", C.c_double * MAX_DIM),
        ("grid_cells", C.c_int64 * MAX_DIM), ("grid_strides", C.c_int64 * MAX_DIM),
        ("obs_min", _vp), ("obs_max", _vp),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("iterations", C.c_int32), ("tree_size", C.c_int64), ("solution_slot", C.c_int64),
        ("chain_len", C.c_int64), ("device_ms", C.c_double), ("reset_ms", C.c_double),
        ("items", C.c_uint64), ("substeps", C.c_uint64), ("points", C.c_uint64), ("boxsteps", C.c_uint64), ("launches", C.c_uint64),
        ("free_items", C.c_uint64), ("capacity", C.c_int64),
    ]


class Trace(C.Structure):
    _fields_ = [
        ("iteration", C.c_int32), ("branching", C.c_int32), ("ve_size", C.c_int64), ("vo_size", C.c_int64),
        ("attempted", C.c_int64), ("valid", C.c_int64), ("staged", C.c_int64), ("appended", C.c_int64),
        ("tree_size", C.c_int64), ("elapsed_ms", C.c_double), ("phase_ms", C.c_double * 6),
    ]


class QueryResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("iterations", C.c_int32), ("tree_size", C.c_int64), ("solution_slot", C.c_int64),
        ("chain_len", C.c_int64), ("device_ms", C.c_double),
        ("items", C.c_uint64), ("substeps", C.c_uint64), ("points", C.c_uint64), ("boxsteps", C.c_uint64),
        ("free_items", C.c_uint64), ("capacity", C.c_int64), ("checked", C.c_int32), ("check_code", C.c_int32),
    ]


QUERY_RESULT_DTYPE = np.dtype([
    ("status", np.int32), ("iterations", np.int32), ("tree_size", np.int64), ("solution_slot", np.int64),
    ("chain_len", np.int64), ("device_ms", np.float64), ("items", np.uint64), ("substeps", np.uint64),
    ("points", np.uint64), ("boxsteps", np.uint64), ("free_items", np.uint64), ("capacity", np.int64), ("checked", np.int32),
    ("check_code", np.int32)], align=True)

_SIGNATURES = {
    "kpx_last_error": (C.c_char_p, []),
    "kpx_version": (C.c_int, []),
    "kpx_struct_size": (C.c_int, [C.c_int]),
    "kpx_fma_peak": (C.c_int, [C.c_int, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "kpx_cull_thresholds": (C.c_int, [C.POINTER(Problem), C.c_int32, _vp]),
    "kpx_cull_tables": (C.c_int, [C.POINTER(Problem), C.c_int32, _vp, _vp, _vp]),
    "kpx_sample_goals": (C.c_int, [C.c_int64, _vp, C.c_int32, _vp, _vp, _vp, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_double, _vp, _vp]),
    "kpx_philox4x32": (C.c_int, [_vp, _vp, _vp, _vp]),
    "kpx_device_info": (C.c_int, [C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "kpx_propagate_batch": (C.c_int, [C.POINTER(Problem), _vp, C.c_int64, _vp, C.c_int64, C.c_int32, C.c_uint64,
                                      C.c_uint64, C.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                      C.POINTER(C.c_double), _vp]),
    "kpx_plan_create": (C.c_int, [C.POINTER(Problem), C.c_int32, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "kpx_plan_destroy": (None, [_vp]),
    "kpx_plan_reset": (C.c_int, [_vp, C.c_uint64, _vp, _vp]),
    "kpx_plan_set_epoch": (C.c_int, [_vp, C.c_uint32]),
    "kpx_plan_set_obstacles": (C.c_int, [_vp, C.c_int32, _vp, _vp]),
    "kpx_plan_run": (C.c_int, [_vp, C.c_double, C.c_int32, C.c_int32, _vp, _vp, C.c_int32, C.POINTER(Stats), _vp]),
    "kpx_plan_snapshot": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kpx_plan_regions": (C.c_int, [_vp] * 9),
    "kpx_plan_solution": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, _vp]),
    "kpx_plan_trajectory": (C.c_int, [_vp, _vp, _vp, C.c_double, C.c_int64, C.c_int64, _vp, _vp, _vp, _vp,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "kpx_trajectory": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int64, _vp, _vp, _vp, C.c_int32, _vp, C.c_int64,
                                 _vp]),
    "kpx_trajectory_valid": (C.c_int, [C.POINTER(Problem), C.c_int64, _vp, _vp, _vp, C.c_double,
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "kpx_plan_trace": (C.c_int, [_vp, C.c_int32, _vp, C.POINTER(C.c_int32)]),
    "kpx_plan_items": (C.c_int, [_vp, C.c_int64, C.POINTER(C.c_int64), _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "kpx_plan_load": (C.c_int, [_vp, C.c_uint64, _vp, C.c_int32, C.c_int64] + [_vp] * 13),
    "kpx_batch_create": (C.c_int, [C.POINTER(Problem), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                   C.POINTER(_vp)]),
    "kpx_batch_info": (C.c_int, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "kpx_batch_destroy": (None, [_vp]),
    "kpx_batch_upload": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, C.c_int32, _vp]),
    "kpx_batch_set_scenes": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp]),
    "kpx_batch_upload_scenes": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, C.c_int32, _vp]),
    "kpx_batch_launch": (C.c_int, [_vp, C.c_double, _vp]),
    "kpx_batch_set_handoff": (C.c_int, [_vp, C.c_int32]),
    "kpx_batch_handoff_counts": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "kpx_batch_validate": (C.c_int, [_vp, C.c_double, _vp]),
    "kpx_batch_download": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "kpx_batch_run": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, C.c_double, _vp, _vp, _vp, _vp,
                                C.POINTER(C.c_double), _vp]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def library_path() -> str:
    return LIB_PATH


def load():
    """Load libkpx.so; raises DeviceError when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.isfile(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2409_06807_b200.csrc.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        try:
            lib = C.CDLL(LIB_PATH)
        except OSError as exc:
            raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        for which, cls in enumerate((Problem, Stats, Trace, QueryResult)):
            if lib.kpx_struct_size(which) != C.sizeof(cls):
                raise DeviceError(f"ABI mismatch: {cls.__name__} is {C.sizeof(cls)} bytes here, "
                                  f"{lib.kpx_struct_size(which)} in libkpx.so")
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = load().kpx_last_error().decode(errors="replace")
    if rc == E_LIMIT and "dimension exceeds" in msg:
        raise ValueError(msg)  # reference: ValueError (_kernel.pyx:318-319)
    if rc == E_ARG:
        raise ConfigError(f"{what}: {msg}")
    raise DeviceError(f"{what} failed (code {rc}): {msg}")


def ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


def make_problem(model_id, n, nu, t_e, lambda_max, t_prop, check_res, epsilon, delta, control_lo, control_hi,
                 state_lo, state_hi, obs_min, obs_max, grid_lo, grid_width, grid_cells, grid_strides, subcells,
                 rng=RNG_SPLITMIX64, t_e_max=None, t_e_growth=2.0):
    """Flatten into ``kpx_problem``.  Returns (struct, keepalive) -- keep both alive during calls."""
    if n > MAX_DIM or nu > MAX_CONTROL:
        raise ValueError("state/control dimension exceeds kernel limits")
    p = Problem()
    p.model_id, p.n, p.nu, p.subcells = int(model_id), int(n), int(nu), int(subcells)
    p.grid_n, p.lambda_max, p.t_e = len(grid_lo), int(lambda_max), int(t_e)
    if t_e_max is not None and int(t_e_max) != int(t_e):     # adaptive capacity: allocate for t_e_max, start at t_e
        if int(t_e_max) < int(t_e) or not float(t_e_growth) > 1.0:
            raise ConfigError("adaptive capacity needs t_e_max >= t_e and t_e_growth > 1")
        p.t_e, p.t_e_start, p.t_e_growth = int(t_e_max), int(t_e), float(t_e_growth)
    p.rng = int(rng)
    p.t_prop, p.check_res, p.epsilon, p.delta = float(t_prop), float(check_res), float(epsilon), float(delta)
    for j in range(nu):
        p.control_lo[j], p.control_hi[j] = float(control_lo[j]), float(control_hi[j])
    for d in range(n):
        p.state_lo[d], p.state_hi[d] = float(state_lo[d]), float(state_hi[d])
    for d in range(p.grid_n):
        p.grid_lo[d], p.grid_width[d] = float(grid_lo[d]), float(grid_width[d])
        p.grid_cells[d], p.grid_strides[d] = int(grid_cells[d]), int(grid_strides[d])
    omin = np.ascontiguousarray(np.asarray(obs_min, dtype=np.float64).reshape(-1, 3))
    omax = np.ascontiguousarray(np.asarray(obs_max, dtype=np.float64).reshape(-1, 3))
    p.n_obs = omin.shape[0]
    p.obs_min = omin.ctypes.data if p.n_obs else None
    p.obs_max = omax.ctypes.data if p.n_obs else None
    return p, (omin, omax)


def problem_from(prob, rng=RNG_SPLITMIX64, t_e_max=None, t_e_growth=2.0) -> tuple:
    """``Problem`` (problem.py) -> ``kpx_problem``."""
    m, g, c = prob.model, prob.grid, prob.cfg
    if m.kernel_id is None:
        raise ConfigError(f"model '{m.name}' has no CUDA kernel")
    return make_problem(m.kernel_id, m.n, m.control_dim, c.t_e, c.lambda_max, c.t_prop, prob.check_resolution,
                        c.epsilon, c.delta, m.control_lo, m.control_hi, prob.state_lo, prob.state_hi,
                        prob.env.obstacles_min, prob.env.obstacles_max, g.lo, g.widths, g.cells, g.strides,
                        g.subcells, rng=rng, t_e_max=t_e_max, t_e_growth=t_e_growth)
