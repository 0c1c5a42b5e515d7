"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle (kpx_oracle.c).

The oracle is the checker for the CUDA path, never the thing shipped or
measured as the product: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
Parity pinned against the unmodified reference: see tests/test_oracle_pin.py.

The Python surface mirrors the reference's names so parity tests read like the
reference's own: ``propagate_batch`` (backend.py:80), ``OraclePlan.step`` /
``.solve`` (planner.py:271), ``snapshot`` (planner.py:92), ``propagate_ode``
(dynamics.py:242), ``trajectory_valid`` (validity.py:108).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

MAXD, MAXU = 48, 24
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libkpx_oracle.so")

STATUS_NAMES = {0: "solved", 1: "timeout", 2: "capacity_exhausted", 3: "error", 4: "running"}


class Ctx(C.Structure):
    _fields_ = [
        ("model_id", C.c_int32), ("n", C.c_int32), ("nu", C.c_int32), ("n_obs", C.c_int32),
        ("subcells", C.c_int32), ("grid_n", C.c_int32),
        ("t_prop", C.c_double), ("check_res", C.c_double),
        ("control_lo", C.c_double * MAXU), ("control_hi", C.c_double * MAXU),
        ("state_lo", C.c_double * MAXD), ("state_hi", C.c_double * MAXD),
        ("grid_lo", C.c_double * MAXD), ("grid_width", C.c_double * MAXD),
        ("grid_cells", C.c_int64 * MAXD), ("grid_strides", C.c_int64 * MAXD),
        ("obs_min", C.c_void_p), ("obs_max", C.c_void_p),
    ]


_P = C.c_void_p


class Plan(C.Structure):
    _fields_ = [
        ("ctx", Ctx),
        ("t_e", C.c_int64), ("lambda_max", C.c_int32), ("epsilon", C.c_double), ("delta", C.c_double),
        ("seed", C.c_uint64), ("threads", C.c_int32), ("goal", C.c_double * 4),
        ("n_regions", C.c_int64), ("subs_per_region", C.c_int64), ("vol", C.c_double),
        ("n_valid", _P), ("n_invalid", _P), ("cov", _P), ("free_vol", _P), ("score", _P), ("p_accept", _P),
        ("visited", _P), ("avail", _P),
        ("states", _P), ("control", _P), ("dt", _P), ("parent", _P), ("region", _P), ("tag", _P),
        ("size", C.c_int64),
        ("b_valid", _P), ("b_region", _P), ("b_sub", _P), ("b_end", _P), ("b_control", _P), ("b_dt", _P),
        ("b_accept", _P), ("e_slots", _P), ("stage_idx", _P), ("b_substeps", _P), ("b_points", _P),
        ("tmp_score", _P),
        ("iteration", C.c_int64), ("solution_slot", C.c_int64), ("status", C.c_int32),
        ("tr_branching", C.c_int64), ("tr_ve", C.c_int64), ("tr_vo", C.c_int64), ("tr_attempted", C.c_int64),
        ("tr_valid", C.c_int64), ("tr_staged", C.c_int64), ("tr_appended", C.c_int64),
        ("total_substeps", C.c_int64), ("total_points", C.c_int64), ("total_items", C.c_int64),
        ("t_e_alloc", C.c_int64), ("growth", C.c_double), ("growths", C.c_int64),
    ]


_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.isfile(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "kpx_oracle.c"))):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.kpo_mix64.restype = C.c_uint64
        L.kpo_mix64.argtypes = [C.c_uint64]
        L.kpo_stream_key.restype = C.c_uint64
        L.kpo_stream_key.argtypes = [C.c_uint64] * 5
        L.kpo_draw.restype = C.c_uint64
        L.kpo_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.kpo_unit.restype = C.c_double
        L.kpo_unit.argtypes = [C.c_uint64]
        L.kpo_default_substeps.restype = C.c_int
        L.kpo_default_substeps.argtypes = [C.c_double]
        L.kpo_densify_steps.restype = C.c_int64
        L.kpo_densify_steps.argtypes = [C.c_double, C.c_double]
        L.kpo_propagate_ode.restype = C.c_int
        L.kpo_propagate_ode.argtypes = [C.c_int, C.c_int, _P, _P, C.c_double, _P]
        L.kpo_segment_valid.restype = C.c_int
        L.kpo_segment_valid.argtypes = [C.POINTER(Ctx), _P, C.c_int, C.c_double]
        L.kpo_trajectory_valid.restype = C.c_int
        L.kpo_trajectory_valid.argtypes = [C.POINTER(Ctx), C.c_int, _P, _P, _P, _P, _P, C.c_double,
                                           C.POINTER(C.c_int)]
        L.kpo_propagate_batch.restype = None
        L.kpo_propagate_batch.argtypes = [C.POINTER(Ctx), _P, _P, C.c_int64, C.c_int, C.c_uint64, C.c_uint64,
                                          _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int]
        L.kpo_plan_create.restype = C.POINTER(Plan)
        L.kpo_plan_create.argtypes = [C.POINTER(Ctx), C.c_int64, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                      _P, _P, C.c_int]
        L.kpo_plan_destroy.restype = None
        L.kpo_plan_destroy.argtypes = [C.POINTER(Plan)]
        L.kpo_plan_step.restype = C.c_int
        L.kpo_plan_step.argtypes = [C.POINTER(Plan), C.c_int]
        L.kpo_plan_step_given.restype = C.c_int
        L.kpo_plan_step_given.argtypes = [C.POINTER(Plan), C.c_int, C.c_int64, _P, _P, _P, _P, _P]
        L.kpo_plan_set_capacity.restype = C.c_int
        L.kpo_plan_set_capacity.argtypes = [C.POINTER(Plan), C.c_int64, C.c_double]
        L.kpo_plan_solve.restype = C.c_int
        L.kpo_plan_solve.argtypes = [C.POINTER(Plan), C.c_double, C.c_int64, C.POINTER(C.c_double)]
        L.kpo_plan_chain.restype = C.c_int64
        L.kpo_plan_chain.argtypes = [C.POINTER(Plan), C.c_int64, _P, C.c_int64]
        L.kpo_sizeof_plan.restype = C.c_int64
        L.kpo_sizeof_ctx.restype = C.c_int64
        assert L.kpo_sizeof_ctx() == C.sizeof(Ctx), (L.kpo_sizeof_ctx(), C.sizeof(Ctx))
        assert L.kpo_sizeof_plan() == C.sizeof(Plan), (L.kpo_sizeof_plan(), C.sizeof(Plan))
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(_P)


def make_ctx(model_id, n, nu, control_lo, control_hi, t_prop, state_lo, state_hi, obs_min, obs_max,
             check_res, grid_lo, grid_width, grid_cells, grid_strides, subcells):
    """Build the static per-run context (backend.py:27-44).  Returns (Ctx, keepalive)."""
    if n > MAXD or nu > MAXU:
        raise ValueError("state/control dimension exceeds oracle limits")
    c = Ctx()
    c.model_id, c.n, c.nu, c.subcells = int(model_id), int(n), int(nu), int(subcells)
    c.t_prop, c.check_res = float(t_prop), float(check_res)
    for j in range(nu):
        c.control_lo[j], c.control_hi[j] = float(control_lo[j]), float(control_hi[j])
    c.grid_n = len(grid_lo)
    for d in range(n):
        c.state_lo[d], c.state_hi[d] = float(state_lo[d]), float(state_hi[d])
    for d in range(c.grid_n):
        c.grid_lo[d], c.grid_width[d] = float(grid_lo[d]), float(grid_width[d])
        c.grid_cells[d], c.grid_strides[d] = int(grid_cells[d]), int(grid_strides[d])
    omin = _f64(np.asarray(obs_min).reshape(-1, 3))
    omax = _f64(np.asarray(obs_max).reshape(-1, 3))
    c.n_obs = omin.shape[0]
    c.obs_min = omin.ctypes.data if c.n_obs else None
    c.obs_max = omax.ctypes.data if c.n_obs else None
    return c, (omin, omax)


def propagate_batch(ctx: Ctx, states, e_slots, lam, seed, iteration, threads=1, counters=False):
    """Oracle twin of ``_kernel.propagate_batch`` (_kernel.pyx:299); returns the Batch dict."""
    L = lib()
    states = _f64(states)
    e_slots = np.ascontiguousarray(e_slots, dtype=np.int64)
    m, n, nu = len(e_slots), ctx.n, ctx.nu
    items = m * int(lam)
    out = {
        "valid": np.zeros(items, np.uint8), "region": np.empty(items, np.int64), "sub": np.empty(items, np.int64),
        "end": np.zeros((items, n)), "control": np.zeros((items, nu)), "dt": np.zeros(items),
        "accept_u": np.zeros(items),
    }
    sub = np.zeros(items, np.int64) if counters else None
    pts = np.zeros(items, np.int64) if counters else None
    L.kpo_propagate_batch(C.byref(ctx), _ptr(states), _ptr(e_slots), m, int(lam),
                          int(seed) & 0xFFFFFFFFFFFFFFFF, int(iteration) & 0xFFFFFFFFFFFFFFFF,
                          _ptr(out["valid"]), _ptr(out["region"]), _ptr(out["sub"]), _ptr(out["end"]),
                          _ptr(out["control"]), _ptr(out["dt"]), _ptr(out["accept_u"]),
                          _ptr(sub) if counters else None, _ptr(pts) if counters else None, int(threads))
    if counters:
        out["substeps"], out["points"] = sub, pts
    return out


def propagate_ode(model_id, x, u, dt):
    """dynamics.py:242 -- returns sampled_states (S+1, n)."""
    L = lib()
    x, u = _f64(x), _f64(u)
    n = len(x)
    S = L.kpo_default_substeps(float(dt))
    buf = np.empty((S + 1, n))
    got = L.kpo_propagate_ode(int(model_id), n, _ptr(x), _ptr(u), float(dt), _ptr(buf))
    assert got == S
    return buf


def trajectory_valid(ctx: Ctx, seg_start, seg_control, seg_dt, start, goal4, res):
    """validity.py:108 applied to extract_trajectory's chain.  Returns (ok, fail_code)."""
    L = lib()
    seg_start, seg_control, seg_dt = _f64(seg_start), _f64(seg_control), _f64(seg_dt)
    start, goal4 = _f64(start), _f64(goal4)
    code = C.c_int(0)
    ok = L.kpo_trajectory_valid(C.byref(ctx), len(seg_dt), _ptr(seg_start), _ptr(seg_control), _ptr(seg_dt),
                                _ptr(start), _ptr(goal4), float(res), C.byref(code))
    return bool(ok), code.value


def _view(ptr, dtype, shape):
    n = int(np.prod(shape))
    if n == 0:
        return np.zeros(shape, dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


class OraclePlan:
    """One planning run of the oracle (KinoPax, planner.py:134)."""

    def __init__(self, ctx: Ctx, t_e, lambda_max, epsilon, delta, seed, start, goal4, threads=1, keep=None):
        self._L = lib()
        self._keep = keep
        start, goal4 = _f64(start), _f64(goal4)
        self._p = self._L.kpo_plan_create(C.byref(ctx), int(t_e), int(lambda_max), float(epsilon), float(delta),
                                          int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(start), _ptr(goal4), int(threads))
        self.n, self.nu = ctx.n, ctx.nu

    def close(self):
        if self._p:
            self._L.kpo_plan_destroy(self._p)
            self._p = None

    def __del__(self):
        self.close()

    @property
    def raw(self) -> Plan:
        return self._p.contents

    def step(self, lam_override=0) -> int:
        return self._L.kpo_plan_step(self._p, int(lam_override))

    def step_given(self, valid, region, sub, end, goal_hit=None, lam_override=0) -> int:
        """One iteration on a supplied Batch (another integrator's verdicts / cells / end states): the
        bookkeeping of planner.py:185-265 alone.  Raises if the item count differs from this plan's |V_E| x lambda."""
        valid = np.ascontiguousarray(valid, dtype=np.uint8)
        region = np.ascontiguousarray(region, dtype=np.int64)
        sub = np.ascontiguousarray(sub, dtype=np.int64)
        end = _f64(end)
        goal = None if goal_hit is None else np.ascontiguousarray(goal_hit, dtype=np.uint8)
        st = self._L.kpo_plan_step_given(self._p, int(lam_override), len(valid), _ptr(valid), _ptr(region), _ptr(sub),
                                         _ptr(end), None if goal is None else _ptr(goal))
        if st < 0:
            raise ValueError("supplied batch does not match this plan's item count")
        return st

    def set_capacity(self, t_e_start, growth):
        """Adaptive capacity (Remark 1 -- an extension the reference package does not have): this
        plan was created with room for its t_e nodes; start with ``t_e_start`` in effect and multiply by ``growth``
        (never beyond the allocation) whenever the run would end with capacity_exhausted."""
        if self._L.kpo_plan_set_capacity(self._p, int(t_e_start), float(growth)) != 0:
            raise ValueError("bad capacity arguments (or the plan has already stepped)")

    def solve(self, t_max=60.0, max_iters=0):
        el = C.c_double(0.0)
        st = self._L.kpo_plan_solve(self._p, float(t_max), int(max_iters), C.byref(el))
        return st, el.value

    @property
    def status(self):
        return STATUS_NAMES[self.raw.status]

    def snapshot(self) -> dict:
        """planner.py:92-102."""
        p, s = self.raw, int(self.raw.size)
        return {
            "size": s,
            "states": _view(p.states, np.float64, (s, self.n)).copy(),
            "parent": _view(p.parent, np.int64, (s,)).copy(),
            "control": _view(p.control, np.float64, (s, self.nu)).copy(),
            "dt": _view(p.dt, np.float64, (s,)).copy(),
            "tag": _view(p.tag, np.uint8, (s,)).copy(),
            "region": _view(p.region, np.int64, (s,)).copy(),
        }

    def decomposition(self) -> dict:
        p, R = self.raw, int(self.raw.n_regions)
        return {
            "n_valid": _view(p.n_valid, np.int64, (R,)).copy(), "n_invalid": _view(p.n_invalid, np.int64, (R,)).copy(),
            "cov": _view(p.cov, np.int64, (R,)).copy(), "free_vol": _view(p.free_vol, np.float64, (R,)).copy(),
            "score": _view(p.score, np.float64, (R,)).copy(), "p_accept": _view(p.p_accept, np.float64, (R,)).copy(),
            "visited": _view(p.visited, np.uint8, (R * int(p.subs_per_region),)).copy(),
            "avail": _view(p.avail, np.uint8, (R,)).copy(),
        }

    def last_batch(self) -> dict:
        p = self.raw
        I = int(p.tr_attempted)
        return {
            "valid": _view(p.b_valid, np.uint8, (I,)).copy(), "region": _view(p.b_region, np.int64, (I,)).copy(),
            "sub": _view(p.b_sub, np.int64, (I,)).copy(), "end": _view(p.b_end, np.float64, (I, self.n)).copy(),
            "control": _view(p.b_control, np.float64, (I, self.nu)).copy(), "dt": _view(p.b_dt, np.float64, (I,)).copy(),
            "accept_u": _view(p.b_accept, np.float64, (I,)).copy(),
            "e_slots": _view(p.e_slots, np.int64, (int(p.tr_ve),)).copy(),
            "staged_idx": _view(p.stage_idx, np.int64, (int(p.tr_staged),)).copy(),
        }

    def trace(self) -> dict:
        p = self.raw
        return {"iteration": int(p.iteration), "branching": int(p.tr_branching), "ve_size": int(p.tr_ve),
                "vo_size": int(p.tr_vo), "attempted": int(p.tr_attempted), "valid": int(p.tr_valid),
                "staged": int(p.tr_staged), "appended": int(p.tr_appended), "tree_size": int(p.size)}

    def chain(self, slot=None):
        p = self.raw
        slot = int(p.solution_slot) if slot is None else int(slot)
        out = np.zeros(65536, np.int64)
        ln = self._L.kpo_plan_chain(self._p, slot, _ptr(out), len(out))
        if ln < 0:
            raise RuntimeError("corrupted parent chain")
        return out[:ln].copy()


def ctx_from_problem(prob):
    """Build the oracle context from a host ``Problem`` (paper_2409_06807_b200.problem)."""
    m, g = prob.model, prob.grid
    return make_ctx(m.kernel_id, m.n, m.control_dim, m.control_lo, m.control_hi, prob.cfg.t_prop,
                    prob.state_lo, prob.state_hi, prob.env.obstacles_min, prob.env.obstacles_max,
                    prob.check_resolution, g.lo, g.widths, g.cells, g.strides, g.subcells)


def plan_from_problem(prob, threads=1) -> "OraclePlan":
    ctx, keep = ctx_from_problem(prob)
    c = prob.cfg
    return OraclePlan(ctx, c.t_e, c.lambda_max, c.epsilon, c.delta, c.seed, prob.env.start, prob.goal4,
                      threads=threads, keep=(ctx, keep))
