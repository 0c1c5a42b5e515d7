"""Planner facade: the reference's ``KinoPax`` / ``plan()`` API over the device-resident loop.

Reference ``planner.py`` runs three NumPy/Cython passes per iteration on the
host (``planner.py:176-267``) inside a Python ``while`` (``:271-303``).  Here the
whole loop -- propagation, region update, node-set update, termination -- is one
persistent CUDA kernel (``csrc/kpx_plan.cuh``); this module only

* flattens the query (``problem.build_problem`` = reference ``__init__``, ``:137-172``),
* owns the device handle (arena + region state live in HBM between calls),
* launches ``kpx_plan_run`` and reads back a few hundred bytes of result,
* rebuilds the solution trajectory on the host in float64 with ``propagate_ode``
  exactly as the reference does (``:325-341``).

``KinoPax.step()`` runs a single iteration per launch so that parity tests can
compare tree and region state with the oracle after every iteration.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .backend import get_backend
from .core import (ConfigError, DeviceError, Environment, PlannerConfig, PlanResult, PlanStats, PlanStatus,
                   TrajectorySegment)
from .decomposition import RegionState
from .dynamics import DynamicsModel, propagate_ode
from .problem import Problem, build_problem

TAG_EMPTY, TAG_EXPAND, TAG_OPEN, TAG_UNEXPLORED = 0, 1, 2, 3

_STATUS = {_lib.SOLVED: PlanStatus.SOLVED, _lib.TIMEOUT: PlanStatus.TIMEOUT,
           _lib.CAPACITY_EXHAUSTED: PlanStatus.CAPACITY_EXHAUSTED, _lib.ERROR: PlanStatus.ERROR,
           _lib.STOPPED: PlanStatus.TIMEOUT}


def compute_branching_factor(t_e: int, tree_size: int, ve_size: int, lambda_max: int) -> int:
    """Eq. 6 with a floor of 1 (reference ``planner.py:37-48``); the kernel evaluates the same expression."""
    if ve_size < 1:
        raise ValueError("ve_size must be >= 1")
    if tree_size > t_e:
        raise ValueError("tree_size exceeds capacity")
    return max(1, min(lambda_max, (t_e - tree_size) // ve_size))


@dataclass
class IterationTrace:
    iteration: int
    branching: int
    ve_size: int
    vo_size: int
    attempted: int
    staged: int
    appended: int
    tree_size: int
    elapsed_s: float
    valid: int = 0
    phase_ms: tuple = ()   # device time per phase: order, propagate, gate, append+estimates, node sets, epilogue


class TreeArena:
    """Host copy of the device tree in the reference's layout (``planner.py:51-102``)."""

    def __init__(self, snap: dict, capacity: int):
        self.capacity = capacity
        self.size = snap["size"]
        self.states, self.parent, self.control = snap["states"], snap["parent"], snap["control"]
        self.dt, self.tag, self.region = snap["dt"], snap["tag"], snap["region"]

    def slots_with_tag(self, tag: int) -> np.ndarray:
        return np.flatnonzero(self.tag[: self.size] == tag)

    @property
    def remaining(self) -> int:
        return self.capacity - self.size

    def snapshot(self) -> dict:
        return {"size": self.size, "states": self.states.copy(), "parent": self.parent.copy(),
                "control": self.control.copy(), "dt": self.dt.copy(), "tag": self.tag.copy(),
                "region": self.region.copy()}


def extract_trajectory(arena, slot: int, model: DynamicsModel) -> list:
    """Re-propagate the parent chain root -> slot (reference ``planner.py:325-341``)."""
    chain, s = [], int(slot)
    while s != 0:
        p = int(arena.parent[s])
        if p < 0 or p >= arena.size:
            raise RuntimeError(f"corrupted parent chain at slot {s}")
        chain.append(s)
        s = p
    return [propagate_ode(model, arena.states[int(arena.parent[c])], arena.control[c], float(arena.dt[c]))
            for c in reversed(chain)]


class KinoPax:
    """One planning query bound to one device handle; ``reset()`` re-arms it for another query."""

    def __init__(self, cfg: PlannerConfig, env: Environment, model: DynamicsModel,
                 check_resolution: float = 0.05, backend: Optional[str] = None, team_ctas: int = 0,
                 device: int = 0, t_e_max: Optional[int] = None, t_e_growth: float = 2.0):
        """``t_e_max`` / ``t_e_growth``: adaptive tree capacity (the paper's Remark 1, not in the reference package):
        the arena is reserved for ``t_e_max`` nodes; the run starts with ``cfg.t_e`` in effect and, whenever it would
        end CAPACITY_EXHAUSTED, multiplies the capacity by ``t_e_growth`` (up to ``t_e_max``) and carries on."""
        self.problem: Problem = build_problem(cfg, env, model, check_resolution)
        self.cfg, self.env, self.model = cfg, env, model
        self.checker = self.problem.checker
        self.backend = get_backend(backend, model)
        self.precision = self.backend.precision
        self._lib = _lib.load()
        self.t_e_max, self.t_e_growth = t_e_max, t_e_growth
        self._prob_struct, self._keep = _lib.problem_from(self.problem, rng=self.backend.rng, t_e_max=t_e_max, t_e_growth=t_e_growth)
        self._handle = _lib._vp()
        self._traj_buf = None         # reusable host buffers of _trajectory
        _lib.check(self._lib.kpx_plan_create(C.byref(self._prob_struct), self.precision, int(team_ctas), int(device),
                                             C.byref(self._handle)), "kpx_plan_create")
        self.device = device
        self.team_ctas = team_ctas
        self.iteration = 0
        self.last_stats: Optional[_lib.Stats] = None
        self._retry: Optional["KinoPax"] = None
        self.reset()

    # -- lifecycle ---------------------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_handle", None):
            self._lib.kpx_plan_destroy(self._handle)
            self._handle = None
        if getattr(self, "_retry", None) is not None:
            self._retry.close()
            self._retry = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def reset(self, seed: Optional[int] = None, start=None, goal4=None) -> None:
        """Arm the handle for a (new) query on the same problem; the device reset runs inside the kernel."""
        self.seed = self.cfg.seed if seed is None else int(seed)
        if start is not None:          # the reference refuses an invalid start in __init__ (planner.py:144-145)
            start = np.ascontiguousarray(start, dtype=np.float64)
            if start.shape != (self.model.n,):
                raise ConfigError(f"start must have shape ({self.model.n},), got {start.shape}")
            if not self.checker.state_valid(start):
                raise ConfigError("start state is invalid (outside the state box or in collision)")
        if goal4 is not None:
            goal4 = np.ascontiguousarray(goal4, dtype=np.float64)
            if goal4.shape != (4,) or not np.isfinite(goal4).all() or not goal4[3] > 0:
                raise ConfigError("goal4 must be (cx, cy, cz, r) with a positive radius")
        self.start = np.ascontiguousarray(self.env.start if start is None else start, dtype=np.float64)
        self.goal4 = np.ascontiguousarray(self.problem.goal4 if goal4 is None else goal4, dtype=np.float64)
        _lib.check(self._lib.kpx_plan_reset(self._handle, self.seed & 0xFFFFFFFFFFFFFFFF, _lib.ptr(self.start),
                                            _lib.ptr(self.goal4)), "kpx_plan_reset")
        self.iteration = 0

    # -- device runs --------------------------------------------------------------------------
    def _run(self, t_max: float, max_iters: int = 0, lam_override: int = 0, stop_flag=None, peer_flags=None,
             stream=None) -> _lib.Stats:
        st = _lib.Stats()
        peers = None
        n_peers = 0
        if peer_flags:
            peers = (C.c_void_p * len(peer_flags))(*peer_flags)
            n_peers = len(peer_flags)
        _lib.check(self._lib.kpx_plan_run(self._handle, float(t_max), int(max_iters), int(lam_override),
                                          stop_flag, peers, n_peers, C.byref(st), stream), "kpx_plan_run")
        self.iteration = st.iterations
        self.last_stats = st
        return st

    def step(self, lam_override: int = 0) -> _lib.Stats:
        """Exactly one iteration (one kernel launch); state stays resident for the next call."""
        return self._run(self.cfg.t_max if self.cfg.t_max > 0 else 1e9, max_iters=1, lam_override=lam_override)

    def snapshot(self) -> dict:
        size = int(self.last_stats.tree_size) if self.last_stats is not None else 1
        n, nu = self.model.n, self.model.control_dim
        snap = {"size": size, "states": np.zeros((size, n)), "parent": np.zeros(size, np.int64),
                "control": np.zeros((size, nu)), "dt": np.zeros(size), "tag": np.zeros(size, np.uint8),
                "region": np.zeros(size, np.int64)}
        _lib.check(self._lib.kpx_plan_snapshot(self._handle, size, _lib.ptr(snap["states"]), _lib.ptr(snap["parent"]),
                                               _lib.ptr(snap["control"]), _lib.ptr(snap["dt"]), _lib.ptr(snap["tag"]),
                                               _lib.ptr(snap["region"])), "kpx_plan_snapshot")
        return snap

    @property
    def arena(self) -> TreeArena:
        return TreeArena(self.snapshot(), self.cfg.t_e)

    def region_state(self) -> RegionState:
        g = self.problem.grid
        R = g.n_regions
        arr = {"n_valid": np.zeros(R, np.int64), "n_invalid": np.zeros(R, np.int64), "cov": np.zeros(R, np.int64),
               "free_vol": np.zeros(R), "score": np.zeros(R), "p_accept": np.zeros(R),
               "visited": np.zeros(R * g.subs_per_region, np.uint8), "avail": np.zeros(R, np.uint8)}
        _lib.check(self._lib.kpx_plan_regions(self._handle, *[_lib.ptr(arr[k]) for k in
                                                               ("n_valid", "n_invalid", "cov", "free_vol", "score",
                                                                "p_accept", "visited", "avail")]), "kpx_plan_regions")
        return RegionState(g, arr)

    def last_items(self) -> dict:
        """The Batch of the most recent iteration as the kernel left it in HBM (+ keep flags)."""
        cap, n = int(self.t_e_max or self.cfg.t_e), self.model.n
        cnt = C.c_int64(0)
        out = {"valid": np.zeros(cap, np.uint8), "region": np.zeros(cap, np.int64), "sub": np.zeros(cap, np.int64),
               "end": np.zeros((cap, n)), "keep": np.zeros(cap, np.uint8), "parent_slot": np.zeros(cap, np.int64),
               "goal_hit": np.zeros(cap, np.uint8)}
        _lib.check(self._lib.kpx_plan_items(self._handle, cap, C.byref(cnt), _lib.ptr(out["valid"]),
                                            _lib.ptr(out["region"]), _lib.ptr(out["sub"]), _lib.ptr(out["end"]),
                                            _lib.ptr(out["keep"]), _lib.ptr(out["parent_slot"]),
                                            _lib.ptr(out["goal_hit"])), "kpx_plan_items")
        return {k: v[: cnt.value] for k, v in out.items()}

    def traces(self) -> list:
        buf = (_lib.Trace * 4096)()
        cnt = C.c_int32(0)
        _lib.check(self._lib.kpx_plan_trace(self._handle, 4096, buf, C.byref(cnt)), "kpx_plan_trace")
        return [IterationTrace(t.iteration, t.branching, t.ve_size, t.vo_size, t.attempted, t.staged, t.appended,
                               t.tree_size, t.elapsed_ms * 1e-3, t.valid, tuple(t.phase_ms)) for t in buf[: cnt.value]]

    def load_state(self, snapshot: dict, regions: dict, iteration: int, seed: Optional[int] = None) -> None:
        """Restore a tree + region state (checkpoint/resume; parity tests load oracle states)."""
        f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)   # noqa: E731
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)     # noqa: E731
        u8 = lambda a: np.ascontiguousarray(a, dtype=np.uint8)      # noqa: E731
        seed = self.seed if seed is None else int(seed)
        rows = int(snapshot["size"])
        args = [f64(snapshot["states"]), i64(snapshot["parent"]), f64(snapshot["control"]), f64(snapshot["dt"]),
                u8(snapshot["tag"]), i64(snapshot["region"]), i64(regions["n_valid"]), i64(regions["n_invalid"]),
                i64(regions["cov"]), f64(regions["score"]), f64(regions["p_accept"]), u8(regions["visited"]),
                u8(regions["avail"])]
        _lib.check(self._lib.kpx_plan_load(self._handle, seed & 0xFFFFFFFFFFFFFFFF, _lib.ptr(self.goal4),
                                           int(iteration), rows, *[_lib.ptr(a) for a in args]), "kpx_plan_load")
        self.seed = seed
        self.iteration = int(iteration)
        st = _lib.Stats()
        st.tree_size, st.iterations, st.status = rows, int(iteration), _lib.RUNNING
        self.last_stats = st

    # -- solution ------------------------------------------------------------------------------
    def solution_chain(self) -> dict:
        st = self.last_stats
        L, n, nu = int(st.chain_len), self.model.n, self.model.control_dim
        out = {"seg_start": np.zeros((L, n)), "seg_control": np.zeros((L, nu)), "seg_dt": np.zeros(L),
               "seg_slot": np.zeros(L, np.int64), "end_state": np.zeros(n)}
        if L > 0:
            _lib.check(self._lib.kpx_plan_solution(self._handle, L, _lib.ptr(out["seg_start"]),
                                                   _lib.ptr(out["seg_control"]), _lib.ptr(out["seg_dt"]),
                                                   _lib.ptr(out["seg_slot"]), _lib.ptr(out["end_state"])),
                       "kpx_plan_solution")
        return out

    _TRAJ_SEGS = 64            # segments the result packet carries; longer chains take the general path

    def _trajectory(self) -> tuple:
        """Segments from the device chain, rebuilt on the host in float64 by ONE native call
        (``kpx_plan_trajectory`` = ``extract_trajectory`` + ``propagate_ode``, ``planner.py:325-341``,
        ``dynamics.py:242-283``).  f64: every segment starts at the stored parent state, as in the reference.
        f32: the chain is re-integrated from the root (stored float32 node states cannot chain to 1e-9) and must
        still be collision-free and end in the goal (``validity.py:108-125``); ``ok`` reports that check."""
        n, nu = self.model.n, self.model.control_dim
        L = int(self.last_stats.chain_len)
        if L > self._TRAJ_SEGS:
            return self._trajectory_general()
        buf = self._traj_buf
        if buf is None:
            S = self._TRAJ_SEGS
            rows = S * (int(math.ceil(self.cfg.t_prop / 0.02)) + 2)
            ctrl, dts = np.zeros((S, nu)), np.zeros(S)
            sampled, off = np.empty((rows, n)), np.zeros(S + 1, np.int64)
            buf = self._traj_buf = (ctrl, dts, sampled, off, rows, _lib.ptr(ctrl), _lib.ptr(dts), _lib.ptr(sampled),
                                    _lib.ptr(off), C.c_int64(0), C.c_int32(0), C.c_int32(0))
        ctrl, dts, sampled, off, rows, p_ctrl, p_dts, p_sampled, p_off, nseg, okc, code = buf
        from_root = self.precision != _lib.F64
        _lib.check(self._lib.kpx_plan_trajectory(self._handle, _lib.ptr(self.start) if from_root else None,
                                                 _lib.ptr(self.goal4), self.problem.check_resolution, self._TRAJ_SEGS,
                                                 rows, p_ctrl, p_dts, p_sampled, p_off, C.byref(nseg), C.byref(okc),
                                                 C.byref(code)), "kpx_plan_trajectory")
        L = int(nseg.value)
        o = off[:L + 1].tolist()
        states = sampled[:o[L]].copy()                    # one copy: the buffers are reused by the next solve
        cc, dd = ctrl[:L].copy(), dts[:L].tolist()
        segs = [TrajectorySegment(control=cc[i], dt=dd[i], end_state=states[o[i + 1] - 1],
                                  sampled_states=states[o[i]:o[i + 1]]) for i in range(L)]
        return segs, bool(okc.value)

    def _trajectory_general(self) -> tuple:
        """The same through the separate entry points, for chains longer than the result packet."""
        chain = self.solution_chain()
        from_root = self.precision != _lib.F64
        n, nu = self.model.n, self.model.control_dim
        dts, ctrl = chain["seg_dt"], chain["seg_control"]
        starts = chain["seg_start"]
        if from_root:
            starts = starts.copy()
            starts[0] = self.start
        L = len(dts)
        rows = int((np.maximum(4, np.ceil(dts / 0.02)) + 1).sum())
        sampled = np.empty((rows, n))
        off = np.zeros(L + 1, np.int64)
        _lib.check(self._lib.kpx_trajectory(self.model.kernel_id, n, nu, L, _lib.ptr(starts), _lib.ptr(ctrl),
                                            _lib.ptr(dts), 1 if from_root else 0, _lib.ptr(sampled), rows,
                                            _lib.ptr(off)), "kpx_trajectory")
        segs = [TrajectorySegment(control=ctrl[i].copy(), dt=float(dts[i]), end_state=sampled[off[i + 1] - 1].copy(),
                                  sampled_states=sampled[off[i]:off[i + 1]]) for i in range(L)]
        ok = True
        if from_root:
            okc, code = C.c_int32(0), C.c_int32(0)
            _lib.check(self._lib.kpx_trajectory_valid(C.byref(self._prob_struct), L, _lib.ptr(sampled), _lib.ptr(off),
                                                      _lib.ptr(self.goal4), self.problem.check_resolution,
                                                      C.byref(okc), C.byref(code)), "kpx_trajectory_valid")
            ok = bool(okc.value)
        return segs, ok

    def solve(self, trace_fn: Optional[Callable[[IterationTrace], None]] = None,
              capture_tree: bool = False, t_max: Optional[float] = None, stop_flag=None, peer_flags=None) -> PlanResult:
        """``KinoPax.solve`` (``planner.py:271-316``).  ``stop_flag`` / ``peer_flags`` wire an OR-parallel race
        (``batch.race``): a device word that stops this run, device words this run raises when it solves."""
        t0 = time.perf_counter()
        st = self._run(self.cfg.t_max if t_max is None else t_max, stop_flag=stop_flag, peer_flags=peer_flags)
        status = _STATUS.get(st.status, PlanStatus.ERROR)
        trajectory, duration = [], 0.0
        retried = False
        if status is PlanStatus.SOLVED and st.solution_slot != 0:
            if st.chain_len < 0:
                trajectory = extract_trajectory(self.arena, int(st.solution_slot), self.model)
            else:
                trajectory, ok = self._trajectory()
                if not ok:
                    # float32 tree whose float64 re-integration leaves the goal / grazes an obstacle:
                    # plan the query again with the float64 kernel (still the CUDA path).
                    return self._solve_f64_retry(t0, trace_fn, capture_tree)
            duration = float(sum(s.dt for s in trajectory))
        result = PlanResult(status=status, trajectory=trajectory,
                            stats=PlanStats(iterations=int(st.iterations), tree_size=int(st.tree_size),
                                            wall_time_ms=(time.perf_counter() - t0) * 1e3,
                                            solution_duration_s=duration))
        result.device = {"device_ms": st.device_ms, "reset_ms": st.reset_ms, "items": int(st.items),
                         "substeps": int(st.substeps), "points": int(st.points), "boxsteps": int(st.boxsteps), "free_items": int(st.free_items), "capacity": int(st.capacity), "launches": int(st.launches),
                         "precision": "f64" if self.precision == _lib.F64 else "f32", "f64_retry": retried,
                         # the raw device status: PlanStatus keeps the reference's four values, so a run stopped by a
                         # race peer (5) reads TIMEOUT there; this tells the two apart
                         "status_code": int(st.status), "stopped_by_peer": int(st.status) == _lib.STOPPED}
        if trace_fn is not None:
            for tr in self.traces():
                trace_fn(tr)
        if capture_tree:
            result.tree_snapshot = self.snapshot()
        return result

    def _solve_f64_retry(self, t0, trace_fn, capture_tree) -> PlanResult:
        if self._retry is None:
            self._retry = KinoPax(self.cfg, self.env, self.model, self.problem.check_resolution,
                                  backend="cuda-philox" if self.backend.rng == _lib.RNG_PHILOX else "cuda",
                                  team_ctas=self.team_ctas, device=self.device, t_e_max=self.t_e_max,
                                  t_e_growth=self.t_e_growth)
        self._retry.reset(self.seed, self.start, self.goal4)
        res = self._retry.solve(trace_fn=trace_fn, capture_tree=capture_tree)
        res.stats.wall_time_ms = (time.perf_counter() - t0) * 1e3
        res.device["f64_retry"] = True
        return res


def plan(cfg: PlannerConfig, env: Environment, model: DynamicsModel, check_resolution: float = 0.05,
         backend: Optional[str] = None, trace_fn: Optional[Callable[[IterationTrace], None]] = None,
         capture_tree: bool = False) -> PlanResult:
    """Run one planning query end to end (reference ``planner.py:344-350``)."""
    with KinoPax(cfg, env, model, check_resolution, backend) as eng:
        return eng.solve(trace_fn=trace_fn, capture_tree=capture_tree)
