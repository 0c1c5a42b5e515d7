"""Many independent planning queries per launch, sharding across GPUs, and the OR-parallel race.

The reference plans one query per process and parallelises trials only for its
baseline planner (``bench.py:106-150``, ``rrt.py:139-157``).  Queries are
independent, so here:

* ``BatchPlanner`` keeps ``n_teams`` device workspaces; one persistent launch
  (``kpx_batch_run``) lets teams of ``team_ctas`` CTAs pull queries from a
  device-side queue until it is drained.  No collective is involved.
* ``shard_queries`` assigns query ``q`` to rank ``q mod world``; each
  rank plans its shard on its own GPU and the few bytes of per-query results are
  gathered once at the end, off the clock.
* ``RaceFlags`` wires the OR-parallel race: every rank polls a 4-byte device word
  once per iteration; the first rank to solve stores 1 into every peer's word
  over NVLink peer memory (``st.volatile`` + ``__threadfence_system`` in the kernel).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .backend import get_backend
from .core import ConfigError, Environment, PlannerConfig, PlanStatus, TrajectorySegment
from .dynamics import DynamicsModel
from .problem import build_problem

_STATUS = {_lib.SOLVED: PlanStatus.SOLVED, _lib.TIMEOUT: PlanStatus.TIMEOUT,
           _lib.CAPACITY_EXHAUSTED: PlanStatus.CAPACITY_EXHAUSTED, _lib.ERROR: PlanStatus.ERROR,
           _lib.STOPPED: PlanStatus.TIMEOUT}


@dataclass
class BatchResult:
    """Per-query outcomes of one ``BatchPlanner.run`` (arrays of length Q)."""

    records: np.ndarray            # structured: status, iterations, tree_size, solution_slot, chain_len, device_ms, ...
    chain_start: Optional[np.ndarray]   # (Q, max_chain, n)
    chain_control: Optional[np.ndarray]  # (Q, max_chain, nu)
    chain_dt: Optional[np.ndarray]      # (Q, max_chain)
    kernel_ms: float
    wall_ms: float
    starts: np.ndarray
    goals: np.ndarray
    replanned: Optional[np.ndarray] = None   # indices re-planned in float64 after the re-validation refused them
    scenes: Optional[np.ndarray] = None      # scene index per query (None: all in the planner's own environment)

    def __len__(self) -> int:
        return len(self.records)

    def status(self, q: int) -> PlanStatus:
        return _STATUS.get(int(self.records["status"][q]), PlanStatus.ERROR)

    @property
    def solved(self) -> np.ndarray:
        return self.records["status"] == _lib.SOLVED

    @property
    def success_rate(self) -> float:
        return float(self.solved.mean()) if len(self.records) else 0.0

    @property
    def validated(self) -> np.ndarray:
        """Per query: the solution passed the device's float64 re-validation (reference checker rules)."""
        return self.records["checked"] == 1

    @property
    def rejected(self) -> np.ndarray:
        """Per query: solved by the planner but refused by the float64 re-validation."""
        return self.records["checked"] == -1


def as_seed_array(seeds) -> np.ndarray:
    """Seeds as uint64 over the whole 64-bit domain: negative seeds wrap and seeds >= 2^63 are kept, exactly as
    ``KinoPax.reset`` masks a single seed (reference: tests/test_rng.py:32)."""
    a = np.asarray(seeds)
    if a.dtype.kind == "u":
        return np.ascontiguousarray(a.ravel(), dtype=np.uint64)
    if a.dtype.kind == "i":
        return np.ascontiguousarray(a.ravel().astype(np.int64).astype(np.uint64))
    return np.ascontiguousarray([int(s) & 0xFFFFFFFFFFFFFFFF for s in np.asarray(seeds, dtype=object).ravel()],
                                dtype=np.uint64)


class BatchPlanner:
    """Persistent multi-query planner bound to one GPU."""

    def __init__(self, cfg: PlannerConfig, env: Environment, model: DynamicsModel, check_resolution: float = 0.05,
                 backend: Optional[str] = None, n_teams: int = 0, team_ctas: int = 1, max_chain: int = 64,
                 device: int = 0, t_e_max: Optional[int] = None, t_e_growth: float = 2.0, handoff: bool = True):
        self.problem = build_problem(cfg, env, model, check_resolution)
        self.cfg, self.env, self.model = cfg, env, model
        self.backend = get_backend(backend, model)
        self.precision = self.backend.precision
        self._lib = _lib.load()
        self.t_e_max, self.t_e_growth = t_e_max, t_e_growth     # adaptive capacity, see KinoPax
        self._prob_struct, self._keep = _lib.problem_from(self.problem, rng=self.backend.rng, t_e_max=t_e_max, t_e_growth=t_e_growth)
        self.max_chain, self.device = int(max_chain), device
        self._handle = _lib._vp()
        # n_teams = 0: as many teams as are co-resident on the device for this model and precision; -k: at most k of them
        _lib.check(self._lib.kpx_batch_create(C.byref(self._prob_struct), self.precision, int(n_teams),
                                              int(team_ctas), self.max_chain, int(device), C.byref(self._handle)),
                   "kpx_batch_create")
        nt, tc = C.c_int32(0), C.c_int32(0)
        _lib.check(self._lib.kpx_batch_info(self._handle, C.byref(nt), C.byref(tc)), "kpx_batch_info")
        self.n_teams, self.team_ctas = int(nt.value), int(tc.value)
        # the last queries of a launch carry on on wider and wider teams (kpx_batch_set_handoff); same results
        self.handoff = bool(handoff)
        if not self.handoff:
            _lib.check(self._lib.kpx_batch_set_handoff(self._handle, 0), "kpx_batch_set_handoff")
        self._f64 = None              # float64 twin, created when a refused float32 solution needs re-planning
        self.scenes = [env]           # obstacle sets a query can name (set_scenes); scene 0 is `env`
        self._scene_probs = {0: (self._prob_struct, self._keep)}

    def handoff_counts(self) -> tuple:
        """Queries the last launch handed on to wider teams at the end of its first kernel and of every follow-up stage
        (``kpx_batch_handoff_counts``)."""
        c = (C.c_int32 * 6)()
        _lib.check(self._lib.kpx_batch_handoff_counts(self._handle, c), "kpx_batch_handoff_counts")
        return tuple(int(v) for v in c)

    def set_scenes(self, envs: Sequence[Environment]) -> None:
        """Obstacle sets the queries of a batch can name (``run(..., scenes=idx)``): the batched form of planning in
        several ``Environment`` s (reference: one per process, ``envgen.py:127-163``).  The scenes share this planner's
        workspace box, model and configuration; only the obstacles differ, and none may have more obstacles than the
        environment the planner was created with.  Starts / goals stay per query."""
        envs = list(envs)
        if not envs:
            raise ConfigError("need at least one scene")
        for e in envs:
            if not (np.array_equal(e.workspace_lo, self.env.workspace_lo) and np.array_equal(e.workspace_hi, self.env.workspace_hi)):
                raise ConfigError("scenes must share the planner's workspace box")
            if e.n_obstacles > self.env.n_obstacles:
                raise ConfigError(f"scene '{e.name}' has {e.n_obstacles} obstacles, the planner was created for {self.env.n_obstacles}")
        counts = np.ascontiguousarray([e.n_obstacles for e in envs], dtype=np.int32)
        omin = np.ascontiguousarray(np.concatenate([np.asarray(e.obstacles_min, dtype=np.float64).reshape(-1, 3) for e in envs]))
        omax = np.ascontiguousarray(np.concatenate([np.asarray(e.obstacles_max, dtype=np.float64).reshape(-1, 3) for e in envs]))
        _lib.check(self._lib.kpx_batch_set_scenes(self._handle, len(envs), _lib.ptr(counts), _lib.ptr(omin), _lib.ptr(omax)),
                   "kpx_batch_set_scenes")
        self.scenes = envs
        self._scene_probs = {}
        if self._f64 is not None:
            self._f64.set_scenes(envs)

    def _scene_problem(self, scene: int):
        """kpx_problem of one scene (host-side checks of a solution need that scene's obstacles)."""
        if scene not in self._scene_probs:
            import dataclasses
            env = dataclasses.replace(self.scenes[scene], start=self.env.start, goal=self.env.goal)
            prob = build_problem(self.cfg, env, self.model, self.problem.check_resolution)
            self._scene_probs[scene] = _lib.problem_from(prob, rng=self.backend.rng)
        return self._scene_probs[scene][0]

    def close(self) -> None:
        if getattr(self, "_f64", None) is not None:
            self._f64.close()
            self._f64 = None
        if getattr(self, "_handle", None):
            self._lib.kpx_batch_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _scene_index(self, scenes, q: int):
        if scenes is None:
            return None
        idx = np.ascontiguousarray(scenes, dtype=np.int32)
        if idx.shape != (q,) or (idx < 0).any() or (idx >= len(self.scenes)).any():
            raise ConfigError(f"scenes must be {q} indices into the {len(self.scenes)} scenes of set_scenes()")
        return idx

    def _check_starts_in_scenes(self, starts, scenes) -> None:
        """planner.py:144-145 per scene: every query's start must be a valid state among ITS scene's obstacles."""
        if scenes is None:
            return
        from .validity import ValidityChecker
        for sc in np.unique(scenes):
            ck = ValidityChecker(self.scenes[int(sc)], self.model, self.problem.check_resolution)
            if not ck.state_valid_batch(starts[scenes == sc]).all():
                raise ConfigError(f"a start state is invalid in scene {int(sc)} ('{self.scenes[int(sc)].name}')")

    def _queries(self, seeds, starts, goals) -> tuple:
        """Host arrays of a batch of queries, checked as the reference checks a single one (planner.py:144-145:
        the start must be a valid state): seeds over the whole uint64 domain (negative seeds wrap, as in
        ``KinoPax.reset``), starts (Q, n) inside the state box and outside every obstacle, goals (Q, 4)."""
        q, n = len(seeds), self.model.n
        seeds = as_seed_array(seeds)
        default_start = starts is None
        starts = np.ascontiguousarray(np.tile(self.env.start, (q, 1)) if starts is None else starts, dtype=np.float64)
        goals = np.ascontiguousarray(np.tile(self.problem.goal4, (q, 1)) if goals is None else goals, dtype=np.float64)
        if starts.shape != (q, n) or goals.shape != (q, 4):
            raise ConfigError("starts must be (Q, n) and goals (Q, 4)")
        if not default_start and not self.problem.checker.state_valid_batch(starts).all():
            raise ConfigError("a start state is invalid (outside the state box or in collision)")
        if not (np.isfinite(goals).all() and (goals[:, 3] > 0).all()):
            raise ConfigError("goals must be finite with a positive radius")
        return seeds, starts, goals

    def run(self, seeds: Sequence[int], starts=None, goals=None, t_max: Optional[float] = None,
            want_chains: bool = True, stream=None, replan_rejected: bool = True,
            validate_resolution: Optional[float] = None, scenes=None) -> BatchResult:
        """Plan ``len(seeds)`` queries; ``starts`` (Q, n) / ``goals`` (Q, 4) default to the environment's.

        With ``want_chains`` every solution is re-validated on the device in float64
        (``BatchResult.validated`` / ``rejected``; ``validate_resolution`` overrides the planner's check
        resolution).  A float32 tree is integrated in float32, so once in a few thousand queries its solution
        grazes an obstacle or the goal rim in float64: with ``replan_rejected`` those queries are planned again
        by the float64 kernels (same seeds, still on the GPU) and their records and chains replace the refused
        ones -- what ``KinoPax.solve`` does for a single query."""
        q = len(seeds)
        if q < 1:
            raise ConfigError("need at least one query")
        n, nu = self.model.n, self.model.control_dim
        seeds, starts, goals = self._queries(seeds, starts, goals)
        scenes = self._scene_index(scenes, q)
        self._check_starts_in_scenes(starts, scenes)
        tm = float(self.cfg.t_max if t_max is None else t_max)
        t0 = time.perf_counter()
        if scenes is None and (validate_resolution is None or not want_chains):
            rec = np.zeros(q, dtype=_lib.QUERY_RESULT_DTYPE)
            cs = cc = cd = None
            if want_chains:
                cs = np.zeros((q, self.max_chain, n))
                cc = np.zeros((q, self.max_chain, nu))
                cd = np.zeros((q, self.max_chain))
            ms = C.c_double(0.0)
            _lib.check(self._lib.kpx_batch_run(self._handle, q, _lib.ptr(seeds), _lib.ptr(starts), _lib.ptr(goals), tm,
                                               _lib.ptr(rec), _lib.ptr(cs), _lib.ptr(cc), _lib.ptr(cd), C.byref(ms),
                                               stream), "kpx_batch_run")
            res = BatchResult(rec, cs, cc, cd, ms.value, 0.0, starts, goals)
        else:
            self.upload(seeds, starts, goals, want_chains=want_chains, stream=stream, scenes=scenes)
            self.launch(tm, stream=stream)
            if want_chains:
                self.validate(validate_resolution, stream=stream)
            res = self.download(stream=stream)
        res.scenes = scenes
        if want_chains and replan_rejected and self.precision != _lib.F64:
            bad = np.flatnonzero(res.rejected)
            if len(bad):
                if self._f64 is None:       # few queries: teams of 16 CTAs each instead of one (a float64 plan on one
                    # CTA takes ~100x a float32 one; the GPU is otherwise idle here)
                    self._f64 = BatchPlanner(self.cfg, self.env, self.model, self.problem.check_resolution,
                                             "cuda-philox" if self.backend.rng == _lib.RNG_PHILOX else "cuda",
                                             n_teams=int(min(len(bad), 8)), team_ctas=16, max_chain=self.max_chain,
                                             device=self.device, t_e_max=self.t_e_max, t_e_growth=self.t_e_growth)
                    if len(self.scenes) > 1 or self.scenes[0] is not self.env:
                        self._f64.set_scenes(self.scenes)
                r64 = self._f64.run(seeds[bad], starts[bad], goals[bad], tm, True, stream, False,
                                    validate_resolution, None if scenes is None else scenes[bad])
                res.records[bad] = r64.records
                res.chain_start[bad], res.chain_control[bad], res.chain_dt[bad] = r64.chain_start, r64.chain_control, r64.chain_dt
                res.replanned = bad
        res.wall_ms = (time.perf_counter() - t0) * 1e3
        return res

    # -- resident-input form: upload once, launch many times (what bench.py times with CUDA events) ---
    def upload(self, seeds, starts=None, goals=None, want_chains: bool = False, stream=None, scenes=None) -> int:
        q = len(seeds)
        seeds, starts, goals = self._queries(seeds, starts, goals)
        scenes = self._scene_index(scenes, q)
        self._check_starts_in_scenes(starts, scenes)
        _lib.check(self._lib.kpx_batch_upload_scenes(self._handle, q, _lib.ptr(seeds), _lib.ptr(starts), _lib.ptr(goals),
                                                     _lib.ptr(scenes), 1 if want_chains else 0, stream), "kpx_batch_upload_scenes")
        self._uploaded = (q, starts, goals, want_chains)
        return q

    def launch(self, t_max: Optional[float] = None, stream=None) -> None:
        _lib.check(self._lib.kpx_batch_launch(self._handle, float(self.cfg.t_max if t_max is None else t_max), stream),
                   "kpx_batch_launch")

    def validate(self, resolution: Optional[float] = None, stream=None) -> None:
        """Re-validate every solved query of the last launch on the device in float64 (asynchronous): the
        batched form of ``extract_trajectory`` + ``ValidityChecker.trajectory_valid`` (``planner.py:325-341``,
        ``validity.py:108-125``).  Needs ``upload(..., want_chains=True)``; ``run`` does it by itself."""
        _lib.check(self._lib.kpx_batch_validate(self._handle, float(resolution or 0.0), stream), "kpx_batch_validate")

    def download(self, stream=None) -> BatchResult:
        q, starts, goals, want = self._uploaded
        n, nu = self.model.n, self.model.control_dim
        rec = np.zeros(q, dtype=_lib.QUERY_RESULT_DTYPE)
        cs = np.zeros((q, self.max_chain, n)) if want else None
        cc = np.zeros((q, self.max_chain, nu)) if want else None
        cd = np.zeros((q, self.max_chain)) if want else None
        _lib.check(self._lib.kpx_batch_download(self._handle, _lib.ptr(rec), _lib.ptr(cs), _lib.ptr(cc), _lib.ptr(cd),
                                                stream), "kpx_batch_download")
        return BatchResult(rec, cs, cc, cd, 0.0, 0.0, starts, goals)

    # -- host-side rebuild / re-validation of one solution ------------------------------------------
    def trajectory(self, result: BatchResult, q: int, resolution: Optional[float] = None) -> tuple:
        """(segments, ok): float64 rebuild of query q's solution from its chain on the host; ok = collision-free
        (checked at ``resolution``, default the planner's) and in goal.  ``BatchResult.validated`` holds the
        same verdict for every query, computed on the device."""
        L = int(result.records["chain_len"][q])
        if result.status(q) is not PlanStatus.SOLVED or L <= 0 or result.chain_dt is None:
            return [], result.status(q) is PlanStatus.SOLVED and L == 0
        n, nu = self.model.n, self.model.control_dim
        dts = np.ascontiguousarray(result.chain_dt[q, :L])
        ctrl = np.ascontiguousarray(result.chain_control[q, :L])
        starts = np.ascontiguousarray(result.chain_start[q, :L])
        from_root = self.precision != _lib.F64
        if from_root:
            starts[0] = result.starts[q]
        rows = int((np.maximum(4, np.ceil(dts / 0.02)) + 1).sum())
        sampled, off = np.empty((rows, n)), np.zeros(L + 1, np.int64)
        _lib.check(self._lib.kpx_trajectory(self.model.kernel_id, n, nu, L, _lib.ptr(starts), _lib.ptr(ctrl),
                                            _lib.ptr(dts), 1 if from_root else 0, _lib.ptr(sampled), rows,
                                            _lib.ptr(off)), "kpx_trajectory")
        okc, code = C.c_int32(0), C.c_int32(0)
        goal = np.ascontiguousarray(result.goals[q])
        prob_struct = self._scene_problem(0 if result.scenes is None else int(result.scenes[q]))
        _lib.check(self._lib.kpx_trajectory_valid(C.byref(prob_struct), L, _lib.ptr(sampled), _lib.ptr(off),
                                                  _lib.ptr(goal), float(resolution or self.problem.check_resolution), C.byref(okc),
                                                  C.byref(code)), "kpx_trajectory_valid")
        segs = [TrajectorySegment(control=ctrl[i].copy(), dt=float(dts[i]), end_state=sampled[off[i + 1] - 1].copy(),
                                  sampled_states=sampled[off[i]:off[i + 1]]) for i in range(L)]
        return segs, bool(okc.value)


def plan_batch(cfg: PlannerConfig, env: Environment, model: DynamicsModel, seeds: Sequence[int], starts=None,
               goals=None, check_resolution: float = 0.05, backend: Optional[str] = None, **kw) -> BatchResult:
    """One-shot convenience wrapper: plan all queries on the current GPU."""
    with BatchPlanner(cfg, env, model, check_resolution, backend, **kw) as bp:
        return bp.run(seeds, starts, goals)


# ---------------------------------------------------------------------------- multi-GPU plumbing

def shard_queries(n_queries: int, rank: int, world: int) -> np.ndarray:
    """Indices of the queries rank ``rank`` plans: q mod world == rank (independent units, no exchange)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return np.arange(rank, n_queries, world, dtype=np.int64)


def gather_records(local_idx: np.ndarray, local_records: np.ndarray, n_queries: int, group=None) -> Optional[np.ndarray]:
    """Collect per-query records on rank 0 with one ``gather_object`` (tens of bytes per query, off the clock).

    Works with any ``torch.distributed`` backend (NCCL on the GPU box, gloo in the CPU tests)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    payload = (np.asarray(local_idx), np.asarray(local_records))
    out = [None] * world if rank == 0 else None
    dist.gather_object(payload, out, dst=0, group=group)
    if rank != 0:
        return None
    full = np.zeros(n_queries, dtype=local_records.dtype)
    seen = np.zeros(n_queries, dtype=bool)
    for idx, rec in out:
        full[idx] = rec
        seen[idx] = True
    if not seen.all():
        raise RuntimeError("some queries were not planned by any rank")
    return full


def goal_for_query(q: int, env: Environment, radius: float = 1.3, min_dist: float = 4.0, margin: float = 0.4) -> np.ndarray:
    """Deterministic random goal of query q (SURVEY config 5): centre uniform in [1,9]^3 from the GENERIC
    stream of seed q, rejected if within radius+margin of an obstacle (in x-y) or closer than min_dist to the start."""
    from .rng import PHASE_GENERIC, RngStream
    s = RngStream(q, phase=PHASE_GENERIC)
    start = env.start[:3]
    for _ in range(1000):
        c = np.array([s.uniform_in(1.0, 9.0) for _ in range(3)])
        if np.sqrt(((c - start) ** 2).sum()) < min_dist:
            continue
        if env.n_obstacles:
            lo, hi = env.obstacles_min - (radius + margin), env.obstacles_max + (radius + margin)
            if ((c >= lo) & (c <= hi)).all(axis=1).any():
                continue
        return np.array([c[0], c[1], c[2], radius])
    raise ConfigError("could not sample a goal for this scene")


def goals_for_queries(query_ids, env: Environment, radius: float = 1.3, min_dist: float = 4.0, margin: float = 0.4,
                      stream=None) -> np.ndarray:
    """``goal_for_query`` for a whole batch on the device (``kpx_sample_goals``: one thread per query, the same
    GENERIC streams and float64 operations): (Q, 4) goals, bit-identical to the host loop."""
    ids = np.ascontiguousarray([int(q) & 0xFFFFFFFFFFFFFFFF for q in np.asarray(query_ids).ravel()], dtype=np.uint64)
    out = np.zeros((len(ids), 4))
    omin = np.ascontiguousarray(env.obstacles_min, dtype=np.float64)
    omax = np.ascontiguousarray(env.obstacles_max, dtype=np.float64)
    start3 = np.ascontiguousarray(env.start[:3], dtype=np.float64)
    _lib.check(_lib.load().kpx_sample_goals(len(ids), _lib.ptr(ids), env.n_obstacles, _lib.ptr(omin) if env.n_obstacles else None,
                                            _lib.ptr(omax) if env.n_obstacles else None, _lib.ptr(start3), 1.0, 9.0,
                                            float(radius), float(min_dist), float(margin), _lib.ptr(out), stream),
               "kpx_sample_goals")
    return out


class RaceFlags:
    """Stop words of an OR-parallel race across the ranks of one node.

    Each rank owns one 32-bit device word and polls it once per iteration.  The words are
    shared through CUDA IPC handles exchanged with ``all_gather_object``; the winner's kernel
    writes 1 into every peer word directly over NVLink (NVSwitch makes every peer one hop; for
    4 bytes only the ~2 us store latency matters).  With world size 1 it degenerates to a
    private flag, which is what the single-GPU tests exercise.
    """

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.flag = torch.zeros(64, dtype=torch.int32, device="cuda")   # own word (padded to a cache line)
        self.peer_ptrs = []
        self._peer_tensors = []
        if self.world > 1:
            handle = self.flag.untyped_storage()._share_cuda_()
            handles = [None] * self.world
            dist.all_gather_object(handles, (self.rank, handle), group=group)
            for r, h in handles:
                if r == self.rank:
                    continue
                storage = torch.UntypedStorage._new_shared_cuda(*h)
                t = torch.empty(0, dtype=torch.int32, device=storage.device).set_(storage)
                self._peer_tensors.append(t)
                self.peer_ptrs.append(t.data_ptr())

    def clear(self) -> None:
        self.flag.zero_()
        self.torch.cuda.synchronize()

    @property
    def own_ptr(self) -> int:
        return self.flag.data_ptr()

    def fired(self) -> bool:
        return bool(self.flag[0].item())


def race(engine, flags: "RaceFlags", seed: int, t_max: Optional[float] = None):
    """One rank's leg of the race: plan with ``seed`` until solved or a peer's store stops us.

    Returns the ``PlanResult`` of ``KinoPax.solve``: a solved leg has had its trajectory rebuilt and re-validated
    in float64 (a float32 winner's kernel has already stopped the peers by then, so if that check refuses the
    solution this rank plans the query again with the float64 kernels -- unstoppable, the race is over -- and
    still hands back a valid plan).  ``result.device["status_code"]`` tells a stopped leg (5) from a time-out (1)."""
    engine.reset(seed=seed)
    return engine.solve(t_max=t_max, stop_flag=C.c_void_p(flags.own_ptr), peer_flags=[p for p in flags.peer_ptrs])
