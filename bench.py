#!/usr/bin/env python3
"""Benchmark of the B200 Kino-PAX planner on BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload di6_forest] [--impl reference]

Metric: plans/s (whole job) plus, in the same JSON line, the median time-to-solution (ms) and the
success rate over 100 seeds that BASELINE.json quotes.  A *step* is one pass of the hot path over one
batch of synthetic queries: every GPU plans `--queries` independent queries (seeds) of the workload
in ONE persistent kernel launch.  `value` times K such launches with CUDA events, queries already
resident in HBM; `e2e` times the public API call (host buffers in, results + solution chains out)
with the host<->device copies inside the timed region.  Multi-GPU (torchrun, one rank per GPU): each
rank plans its own queries -- independent units, no data-path collective, weak scaling.

`--impl reference` times the reference's own CPU implementation on the host cores: the UNMODIFIED reference
installed under baseline/_ref (baseline/install_ref.sh; it travels to the GPU box), one single-thread process per
core; the pinned C port under oracle/ is timed beside it (and alone when baseline/_ref is absent).
`python bench.py --gpus N` outside torchrun launches the N ranks itself.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (model, scene, flops per RK4 substep [SURVEY 8d], queries per resident team per step).  A step holds
    # several queries per team (592 / 444 / 296 teams of one CTA on a B200) so that teams keep pulling work while the
    # slowest queries finish: with one query per team the tail of the launch idles ~17 % of the GPU (8 instead of 4
    # per team: another +3..5 %).
    "di6_forest": ("di6", "forest", 78, 8),
    "dubins6_building": ("dubins6", "building", 118, 8),
    "quad12_narrow": ("quad12", "narrow", 336, 8),
    "quad12_forest": ("quad12", "forest", 336, 8),
    # BASELINE.json config 4: k stacked 3-D double integrators (only block 1 is workspace position).
    # 12D uses the full-state grid (cells=3).  A full-state grid is not representable for 24D/48D (cells=1 is a
    # single region: no guidance, the planner fills its tree without reaching the goal), so those two run the
    # separately labelled variant whose grid spans block 1 only (position + velocity, cells=4, like di6).
    "di12_forest": ("di12", "forest", 156, 8),
    "di24_forest": ("di24g6", "forest", 312, 8),
    "di48_forest": ("di48g6", "forest", 624, 4),
    # BASELINE.json config 5: 8192 quadcopter queries with per-query random goals, sharded q mod N
    # across the GPUs of the job -- the total is fixed, so this workload reports "strong" scaling
    "quad12_config5": ("quad12", "forest", 336, 0),
}
CONFIG5_QUERIES = 8192


def get_workload_model(dynamics, name):
    """Model of a workload; 'diNNg6' = stacked integrators with the grid on block 1 (6 dims, 4 cells each)."""
    if name.endswith("g6"):
        import dataclasses
        m = dynamics.stacked_double_integrator(int(name[2:-2]) // 6, grid_dims=6)
        return dataclasses.replace(m, default_cells_per_dim=4)
    return dynamics.get_model(name)


def make_env(kp_envgen, kp_core, model, scene):
    """Scene of a workload.  Stacked integrators (config 4) reuse the di6 Trees scene: block 1 starts at the
    scene's start, the other blocks at the centre of their box, at rest."""
    import numpy as np
    if model.name.startswith("di") and model.n > 6:
        base = kp_envgen.gen_environment(scene, "di6", seed=0)
        start = np.tile(np.array([5.0, 5.0, 5.0, 0.0, 0.0, 0.0]), model.n // 6)
        start[:3] = base.start[:3]
        return kp_core.Environment(f"{scene}-{model.name}", base.workspace_lo, base.workspace_hi, base.obstacles_min,
                                   base.obstacles_max, start, base.goal)
    return kp_envgen.gen_environment(scene, model, seed=0)


def workload_config(workload, model, cfg_t_e, t_prop, cells) -> dict:
    """The `config` object of the JSON line: the SAME for the GPU arm and the reference arm (the driver compares
    them); what differs between the arms (queries per step, teams, backend) is reported under `run`."""
    model_name, scene, _, _ = WORKLOADS[workload]
    label = {"di6_forest": "6D double integrator in Trees (BASELINE.json configs[0], the north-star target)",
             "quad12_narrow": "12D quadcopter in Narrow Passage (configs[1])",
             "dubins6_building": "Dubins airplane in Building (configs[2])",
             "quad12_config5": "8192 quadcopter queries with per-query goals (configs[4])"}.get(workload, workload)
    return {"workload": f"{model_name}/{scene} (gen_environment seed 0): {label}; t_e={cfg_t_e}, lambda_max=32, "
                        f"t_prop={t_prop}, cells={cells}, subcells=4, epsilon=0.005, delta=1.0; queries = seeds 0, 1, 2, ...",
            "l2": "inputs larger than L2: the per-step working set (one arena + region state per resident query) far "
                  "exceeds the 126 MB L2"}


def _cfg(kp, model, seed=0, t_max=60.0):
    return kp.PlannerConfig(t_e=model.default_t_e, lambda_max=32, t_prop=model.default_t_prop, epsilon=0.005,
                            delta=1.0, cells_per_dim=model.default_cells_per_dim, subcells_per_dim=4, t_max=t_max,
                            seed=seed)


# --------------------------------------------------------------------------------------- CPU arm

def _cpu_solve(args):
    """Worker (spawned process): one oracle plan.  Returns (seed, status, seconds, items)."""
    workload, seed = args
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    import paper_2409_06807_b200.core as core
    from paper_2409_06807_b200 import dynamics, envgen, problem
    model_name, scene, _, _ = WORKLOADS[workload]
    model = get_workload_model(dynamics, model_name)
    env = make_env(envgen, core, model, scene)
    cfg = core.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop,
                             cells_per_dim=model.default_cells_per_dim, seed=seed, t_max=120.0)
    op = oracle.plan_from_problem(problem.build_problem(cfg, env, model))
    st, el = op.solve(t_max=120.0)
    return seed, op.status, el, int(op.raw.total_items)


def cpu_throughput(workload: str, n_plans: int, procs: int):
    """plans/s of the CPU oracle: `procs` single-thread worker processes over seeds 0..n_plans-1."""
    import multiprocessing as mp
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        recs = pool.map(_cpu_solve, [(workload, s) for s in range(n_plans)], chunksize=1)
    wall = time.perf_counter() - t0
    solved = [r for r in recs if r[1] == "solved"]
    return {"plans_per_s": n_plans / wall, "wall_s": wall, "solved": len(solved), "plans": n_plans,
            "median_plan_s": statistics.median(r[2] for r in recs)}


# --- the UNMODIFIED reference (baseline/_ref, installed by baseline/install_ref.sh; travels to the GPU box) ---

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF_WORKLOADS = {"di6_forest", "dubins6_building", "quad12_narrow", "quad12_forest", "quad12_config5"}


def reference_installed() -> bool:
    import glob
    return os.path.isfile(os.path.join(REF_DIR, "kinopax", "planner.py")) and \
        bool(glob.glob(os.path.join(REF_DIR, "kinopax", "_kernel*.so")))


def _ref_solve(args):
    """Worker (spawned process): one plan through the reference's own public API (kinopax.plan, planner.py:344),
    its stock compiled backend, threads=1.  Nothing of this repository's package is imported here."""
    workload, seed = args
    sys.path.insert(0, REF_DIR)
    import kinopax as K
    import numpy as np
    model_name, scene, _, _ = WORKLOADS[workload]
    model = K.get_model(model_name)
    env = K.gen_environment(scene, model, seed=0)
    if workload == "quad12_config5":       # the query's own goal: the same GENERIC stream the GPU arm draws from
        from kinopax.rng import RngStream
        st, start, r, ok = RngStream(seed, phase=5), env.start[:3], 1.3, False
        while not ok:
            c = np.array([st.uniform_in(1.0, 9.0) for _ in range(3)])
            ok = np.sqrt(((c - start) ** 2).sum()) >= 4.0 and not \
                ((c >= env.obstacles_min - (r + 0.4)) & (c <= env.obstacles_max + (r + 0.4))).all(axis=1).any()
        import dataclasses
        env = dataclasses.replace(env, goal=K.GoalBall(center=c, radius=r))
    cfg = K.PlannerConfig(t_e=model.default_t_e, lambda_max=32, t_prop=model.default_t_prop, epsilon=0.005, delta=1.0,
                          cells_per_dim=model.default_cells_per_dim, subcells_per_dim=4, t_max=120.0, seed=seed, threads=1)
    t0 = time.perf_counter()
    res = K.plan(cfg, env, model, backend="compiled")
    return seed, res.status.value, time.perf_counter() - t0, res.stats.wall_time_ms


def reference_throughput(workload: str, n_plans: int, procs: int):
    """plans/s of the unmodified reference: `procs` single-thread processes (its OpenMP threads anti-scale, SURVEY
    6.2) over seeds 0..n_plans-1.  None when baseline/_ref is absent or the workload is not a reference model."""
    if workload not in _REF_WORKLOADS or not reference_installed():
        return None
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        recs = pool.map(_ref_solve, [(workload, s) for s in range(n_plans)], chunksize=1)
    wall = time.perf_counter() - t0
    return {"plans_per_s": n_plans / wall, "wall_s": wall, "solved": sum(1 for r in recs if r[1] == "solved"),
            "plans": n_plans, "procs": procs, "median_plan_s": statistics.median(r[2] for r in recs),
            "median_wall_time_ms": statistics.median(r[3] for r in recs)}


def _reference_config(workload) -> dict:
    sys.path.insert(0, ROOT)
    from paper_2409_06807_b200 import dynamics
    model = get_workload_model(dynamics, WORKLOADS[workload][0])
    return workload_config(workload, model, model.default_t_e, model.default_t_prop, model.default_cells_per_dim)


def run_reference(args):
    """The reference arm: rank 0 only; each step = one plan per host core.  With baseline/_ref present the plans
    go through the UNMODIFIED reference (kind "reference"); otherwise through the pinned C port (kind "port")."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, 64))
    model_name, scene, _, _ = WORKLOADS[args.workload]
    use_ref = args.workload in _REF_WORKLOADS and reference_installed() and not args.port
    run_step = (lambda: reference_throughput(args.workload, procs, procs)) if use_ref else \
        (lambda: cpu_throughput(args.workload, procs, procs))
    # honour --steps / --warmup as long as the whole run stays within ~2.5 minutes of CPU wall time
    t0 = time.perf_counter()
    first = run_step()
    t_step = max(time.perf_counter() - t0, 1e-3)
    warmup = max(1, min(args.warmup, int(20.0 / t_step) + 1))
    steps = max(1, min(args.steps, int(120.0 / t_step)))
    for _ in range(warmup - 1):
        run_step()
    res = [run_step() for _ in range(steps)]
    del first
    plans = sum(r["plans"] for r in res)
    wall = sum(r["wall_s"] for r in res)
    value = plans / wall
    port = None
    if use_ref:                 # the C port beside it: the stronger CPU baseline (the reference's
        r = cpu_throughput(args.workload, procs, procs)      # Cython helpers re-take the GIL on every call)
        port = {"kind": "port", "value": r["plans_per_s"], "unit": "plans/s", "cores": procs,
                "median_plan_ms": 1e3 * r["median_plan_s"], "solved": r["solved"],
                "sample": f"{r['plans']} plans, one single-thread process per core, C oracle"}
    what = ("the UNMODIFIED reference from baseline/_ref (kinopax.plan, compiled backend, threads=1)" if use_ref else
            "the C oracle (bit-exact restatement of the reference planner)")
    line = {
        "impl": "reference", "metric": "plans_per_sec", "value": value, "unit": "plans/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup, "ms_per_step": 1e3 * wall / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _reference_config(args.workload),
        "run": {"queries_per_step": procs, "what": "one plan per worker process per step"},
        "median_time_to_solution_ms": 1e3 * statistics.median(r["median_plan_s"] for r in res),
        "success_rate": sum(r["solved"] for r in res) / plans,
        "cpu_baseline": {"value": value, "unit": "plans/s", "cores": procs, "kind": "reference" if use_ref else "port",
                         "sample": f"{plans} plans (seeds 0..{procs - 1} per step), {procs} single-thread processes "
                                   f"of {what}; steps / warm-up are cut only if the run would exceed ~2.5 min"},
        "e2e": {"value": value, "unit": "plans/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if port is not None:
        line["cpu_port"] = port
    print(json.dumps(line), flush=True)



# ------------------------------------------------------------ kernel seam (reference kernel vs CUDA)

def _load_reference_kernel():
    """The reference's own compiled propagation kernel (oracle/_ref, built from /root/reference's _kernel.pyx by
    oracle/build_ref.sh; the checker side of the repository -- never used by the product path)."""
    import glob
    import importlib.machinery
    import importlib.util
    hits = sorted(glob.glob(os.path.join(ROOT, "oracle", "_ref", "_kernel*.so")))
    if not hits:
        return None
    loader = importlib.machinery.ExtensionFileLoader("_kernel", hits[0])
    spec = importlib.util.spec_from_file_location("_kernel", hits[0], loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod


def kernel_seam(kp, cfg, env, model, device, target_items=1_000_000):
    """The drop-in boundary itself (`_kernel.propagate_batch`, _kernel.pyx:299-379): one identical batch of
    ~1 M extensions through (i) the reference's compiled kernel on every host thread and (ii)
    `CudaBackend.propagate_batch` with HOST arrays in and out (H2D + kernel + D2H inside the timing).
    Returns items/s for both and the parity of the outputs."""
    import numpy as np
    from paper_2409_06807_b200.backend import PlanContext
    ref = _load_reference_kernel()
    if ref is None:
        return {"unavailable": "oracle/_ref/_kernel*.so not built (oracle/build_ref.sh needs /root/reference)"}
    prob = kp.build_problem(cfg, env, model)
    with kp.KinoPax(cfg.with_seed(3), env, model, backend="cuda", device=device) as eng:   # a real tree to expand
        snap = eng.solve(capture_tree=True).tree_snapshot
    size = int(snap["size"])
    states = np.ascontiguousarray(snap["states"][:size], dtype=np.float64)
    lam = 8
    m = min(size, max(1, target_items // lam))
    e_slots = np.sort(np.random.default_rng(0).choice(size, size=m, replace=False)).astype(np.int64)
    g, ck = prob.grid, prob.checker
    ctx = PlanContext(model=model, seed=11, t_prop=cfg.t_prop, state_lo=ck.state_lo, state_hi=ck.state_hi,
                      obs_min=env.obstacles_min, obs_max=env.obstacles_max, check_res=prob.check_resolution,
                      grid_lo=g.lo, grid_width=g.widths, grid_cells=g.cells, grid_strides=g.strides,
                      subcells=cfg.subcells_per_dim)
    threads = max(1, min(os.cpu_count() or 1, 64))
    i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)

    def run_ref(slots, nthreads):
        return ref.propagate_batch(states, slots, lam, 11, 5, model.kernel_id, f64(model.control_lo),
                                   f64(model.control_hi), float(cfg.t_prop), f64(ck.state_lo), f64(ck.state_hi),
                                   f64(env.obstacles_min).reshape(-1, 3), f64(env.obstacles_max).reshape(-1, 3),
                                   float(prob.check_resolution), f64(g.lo), f64(g.widths), i64(g.cells), i64(g.strides),
                                   int(cfg.subcells_per_dim), nthreads)

    def best(fn, reps=3):
        out, t = None, float("inf")
        for _ in range(reps):
            t0 = time.perf_counter(); out = fn(); t = min(t, time.perf_counter() - t0)
        return out, t

    # whole batch single-threaded (also the parity reference); a bounded sample on every host thread -- the
    # reference's helpers re-check the GIL on each call, so more OpenMP threads make it slower
    r, t_ref = best(lambda: run_ref(e_slots, 1), reps=1)
    sample = e_slots[:max(1, 16384 // lam)]
    _, t_mt = best(lambda: run_ref(sample, threads), reps=1)
    r_valid, r_region, r_sub, r_end = (np.asarray(r[k]) for k in ("valid", "region", "sub", "end"))
    items = m * lam
    ips_1, ips_mt = items / t_ref, len(sample) * lam / t_mt
    res = {"items": items, "lam": lam, "parents": m, "reference_items_per_s": max(ips_1, ips_mt),
           "reference_items_per_s_1_thread": ips_1, f"reference_items_per_s_{threads}_threads": ips_mt,
           "reference_threads": 1 if ips_1 >= ips_mt else threads,
           "reference": "oracle/_ref: the reference's own _kernel.pyx compiled with its flags (-O3 -fopenmp "
                        "-ffp-contract=off); whole batch on 1 thread, 16 k-item sample on all threads, best reported"}
    for name in ("cuda", "cuda-f32"):
        be = kp.get_backend(name)
        be.propagate_batch(ctx, states, e_slots[:64], lam, 5)          # context / module warm-up
        b, t = best(lambda: be.propagate_batch(ctx, states, e_slots, lam, 5))
        key = "cuda_f64" if name == "cuda" else "cuda_f32"
        res[key + "_items_per_s"] = items / t
        res[key + "_kernel_only_items_per_s"] = items / (b.kernel_ms * 1e-3) if b.kernel_ms else None
        same = bool(np.array_equal(b.valid, r_valid) and np.array_equal(b.region, r_region)
                    and np.array_equal(b.sub[b.valid == 1], r_sub[r_valid == 1]))
        if name == "cuda":
            err = float(np.max(np.abs(b.end - r_end))) if items else 0.0
            res["parity_f64"] = {"valid_region_sub_identical": same, "max_abs_end_diff": err}
        else:
            keep = (b.valid == 1) & (r_valid == 1)
            rel = float(np.max(np.abs(b.end[keep] - r_end[keep]) / np.maximum(np.abs(r_end[keep]), 1.0))) if keep.any() else 0.0
            res["parity_f32"] = {"verdicts_agree_frac": float(np.mean(b.valid == r_valid)), "max_rel_end_diff_valid": rel}
    return res

# --------------------------------------------------------------------------------------- GPU arm

class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc, self.lines = device, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None

    def _pump(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


class _Ctx:
    """What every leg of the GPU arm needs: the package, the rank layout, the launching stream, the barrier."""

    def __init__(self, args):
        import numpy as np
        import torch
        self.np, self.torch, self.args = np, torch, args
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # test hooks (a one-GPU box cannot host two NCCL ranks): KPX_BENCH_DIST_BACKEND=gloo KPX_BENCH_DEVICE=0 run
        # the multi-rank code path with every rank on one device
        self.dist_backend = os.environ.get("KPX_BENCH_DIST_BACKEND", "nccl")
        if "KPX_BENCH_DEVICE" in os.environ:
            self.local = int(os.environ["KPX_BENCH_DEVICE"])
        self.red_dev = "cuda" if self.dist_backend == "nccl" else "cpu"

    def init_device(self):
        torch = self.torch
        torch.cuda.set_device(self.local)
        if self.world > 1:
            import torch.distributed as dist
            if self.dist_backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.dist_backend)
        import paper_2409_06807_b200 as kp
        from paper_2409_06807_b200 import _lib, core, dynamics, envgen
        self.kp, self._lib, self.core, self.dynamics, self.envgen = kp, _lib, core, dynamics, envgen
        self.L = _lib.load()
        self.sptr = _lib.C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def barrier(self):
        if self.world > 1:
            self.torch.distributed.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], device=self.red_dev, dtype=self.torch.float64)
        self.torch.distributed.all_reduce(t, op=self.torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], device=self.red_dev, dtype=self.torch.float64)
        self.torch.distributed.all_reduce(t, op=self.torch.distributed.ReduceOp.SUM)
        return float(t.item())

    def scene(self, workload):
        model_name, scene, f_step, q_per_team = WORKLOADS[workload]
        model = get_workload_model(self.dynamics, model_name)
        env = make_env(self.envgen, self.core, model, scene)
        return model, env, _cfg(self.kp, model), f_step, q_per_team


def latency_leg(ctx, workload, backend, n_seeds, fine_check=True):
    """One query at a time on the whole GPU, seeds 0..n_seeds-1 through KinoPax.solve (BASELINE.json's
    time-to-solution): wall clock per solve incl. the host's float64 trajectory rebuild and re-validation."""
    kp, np = ctx.kp, ctx.np
    model, env, cfg, _, _ = ctx.scene(workload)
    t_setup = time.perf_counter()
    eng = kp.KinoPax(cfg, env, model, backend=backend, device=ctx.local)      # allocation, uploads, module load
    setup_ms = (time.perf_counter() - t_setup) * 1e3
    t_first = time.perf_counter()
    eng.reset(seed=10_000)
    eng.solve()
    first_solve_ms = (time.perf_counter() - t_first) * 1e3                     # first launch of the kernel
    for w in range(1, 3):
        eng.reset(seed=10_000 + w)
        eng.solve()
    dev_ms, wall_ms, ok, reval, reval_fine, iters, trees = [], [], 0, 0, 0, [], []
    fine = kp.ValidityChecker(env, model, 0.005)
    coarse = kp.ValidityChecker(env, model, 0.05)
    for seed in range(n_seeds):
        eng.reset(seed=seed)
        res = eng.solve()
        if res.solved:
            ok += 1
            dev_ms.append(res.device["device_ms"]); wall_ms.append(res.stats.wall_time_ms)
            iters.append(res.stats.iterations); trees.append(res.stats.tree_size)
            reval += bool(coarse.trajectory_valid(res.trajectory, start=env.start))
            if fine_check:
                reval_fine += bool(fine.trajectory_valid(res.trajectory, start=env.start))
    eng.close()
    ref_rate = None
    gold = os.path.join(ROOT, "tests", "golden", f"outcomes_{workload}.json")
    if os.path.isfile(gold):
        g = json.load(open(gold))
        n = min(n_seeds, g["seeds"])
        ref_rate = sum(1 for r in g["records"] if r["seed"] < n and r["status"] == "solved") / n
    return {"seeds": n_seeds, "solved": ok, "success_rate": ok / n_seeds,
            "reference_success_rate_same_seeds": ref_rate,
            "median_device_ms": statistics.median(dev_ms) if dev_ms else None,
            "median_wall_ms": statistics.median(wall_ms) if wall_ms else None,
            "p90_wall_ms": float(np.percentile(wall_ms, 90)) if wall_ms else None,
            "median_iterations": statistics.median(iters) if iters else None,
            "median_tree_size": statistics.median(trees) if trees else None,
            "revalidated_at_check_resolution": reval,
            "revalidated_at_fine_resolution": reval_fine if fine_check else None,
            # the reference excludes construction from wall_time_ms (planner.py:274, 316);
            # reported here as well: one-off engine construction and the first (cold) solve
            "setup_ms_once": setup_ms, "first_solve_ms_cold": first_solve_ms}


def throughput_leg(ctx, workload, backend, steps, warmup, queries=0, team_ctas=1, e2e_steps=0, clocks=False,
                   peaks=None):
    """plans/s of one workload: every rank plans its queries in ONE persistent kernel launch per step (+ the float64
    re-validation kernel), queries resident in HBM, CUDA events on the launching stream, max over ranks.  With
    e2e_steps the public BatchPlanner.run call is timed too (host buffers in and out)."""
    kp, np, torch, args = ctx.kp, ctx.np, ctx.torch, ctx.args
    model, env, cfg, f_step, q_per_team = ctx.scene(workload)
    rank, world = ctx.rank, ctx.world
    bp = kp.BatchPlanner(cfg, env, model, backend=backend, team_ctas=team_ctas, device=ctx.local)
    goals = None
    if workload == "quad12_config5":
        idx = kp.shard_queries(queries or CONFIG5_QUERIES, rank, world)      # q mod world == rank
        seeds, q_here = idx.astype(np.int64), len(idx)
        goals = kp.goals_for_queries(idx, env)
        q_total = queries or CONFIG5_QUERIES
    else:
        q_here = queries or q_per_team * bp.n_teams
        seeds = np.arange(q_here, dtype=np.int64) + rank * q_here
        q_total = q_here * world
    bp.upload(seeds, goals=goals, want_chains=True, stream=ctx.sptr)
    for _ in range(warmup):
        bp.launch(stream=ctx.sptr)
        bp.validate(stream=ctx.sptr)
    torch.cuda.synchronize()
    sampler = ClockSampler(ctx.local) if (clocks and rank == 0) else None
    ctx.barrier()
    if sampler:
        sampler.start()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ctx.barrier()
    ev[0].record()
    for i in range(steps):
        bp.launch(stream=ctx.sptr)          # the whole planning loop of every query: one persistent kernel
        bp.validate(stream=ctx.sptr)        # float64 re-validation of every solution (reference checker rules)
        ev[i + 1].record()
    ctx.barrier()
    clk = sampler.stop() if sampler else None
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    total_ms = ctx.max_over_ranks(ev[0].elapsed_time(ev[-1]))
    res = bp.download(stream=ctx.sptr)
    rec = res.records
    n, nu = model.n, model.control_dim
    out = {"workload": workload, "backend": backend, "model": model, "env": env, "cfg": cfg, "rec": rec,
           "q_here": q_here, "q_total": q_total, "steps": steps, "warmup": warmup, "total_ms": total_ms,
           "step_ms": step_ms, "value": q_total * steps / (total_ms * 1e-3), "teams": bp.n_teams,
           "team_ctas": bp.team_ctas, "clocks": clk, "max_chain": bp.max_chain}
    # algorithmic work of one launch, counted exactly on the device
    flops = float(rec["substeps"].sum()) * f_step + float(rec["boxsteps"].sum()) * 2 * n + \
        float(rec["points"].sum()) * (6 + 6 * env.n_obstacles)
    kern_ms = statistics.mean(step_ms)
    out["flops"], out["kern_ms"] = flops, kern_ms
    out["achieved_tflops"] = flops / (kern_ms * 1e-3) / 1e12
    if peaks:
        peak = peaks["f32"] if "f32" in backend else peaks["f64"]
        out["peak_tflops"], out["frac"] = peak, (out["achieved_tflops"] / peak if peak else None)
    if e2e_steps:
        # the public call with host buffers, copies inside the timed region
        ctx.barrier()
        bp.run(seeds, goals=goals, want_chains=True, stream=ctx.sptr)           # warm the pinned paths
        ctx.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            r2 = bp.run(seeds, goals=goals, want_chains=True, stream=ctx.sptr)
        torch.cuda.synchronize()
        e2e_s = ctx.max_over_ranks(time.perf_counter() - t0)
        chain_rows = int(r2.records["chain_len"].clip(min=0).sum())
        out["e2e"] = {"value": q_total * e2e_steps / e2e_s, "unit": "plans/s",
                      "h2d_bytes_per_step": q_here * (8 + 8 * n + 32),
                      "d2h_bytes_per_step": int(q_here * rec.dtype.itemsize + 8 * chain_rows * (n + nu + 1)),
                      "steps": e2e_steps}
        # re-validate a sample of batch solutions on the host (float64 rebuild + reference checker rules)
        checked = okc = agree = 0
        for q in range(0, q_here, max(1, q_here // 64)):
            if r2.status(q) is kp.PlanStatus.SOLVED:
                _, ok = bp.trajectory(r2, q)
                checked += 1
                okc += bool(ok)
                agree += bool(ok) == bool(r2.records["checked"][q] == 1)
        out["host_check"] = (okc, agree, checked)
    bp.close()
    return out


def _traffic(workload, q_here, kern_ms):
    """DRAM bytes of one launch of the dominant kernel: measured once per round with `ncu --set full`
    (dram__bytes_read.sum + dram__bytes_write.sum, profiles/traffic.json), scaled to this run's queries per launch."""
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.isfile(prof):
        return None, None, None
    tj = json.load(open(prof)).get(workload)
    if not tj or not tj.get("queries_per_launch"):
        return None, None, None
    traffic = float(tj["dram_bytes_per_launch"]) * q_here / float(tj["queries_per_launch"])
    src = f"profiles/{tj['source']}: {tj['dram_bytes_per_launch'] / tj['queries_per_launch'] / 1e6:.1f} MB per query"
    hbm = {"dram_gbs": traffic / (kern_ms * 1e-3) / 1e9, "peak_gbs": _measured_hbm(),
           "frac": traffic / (kern_ms * 1e-3) / 1e9 / _measured_hbm()}
    return traffic, src, hbm


# BASELINE.json's other configurations, each as a short leg of the default run (bounded: ~1 warm-up + 1-2 timed
# launches) so that their numbers are measured by whoever runs bench.py, not only claimed in DESIGN.md
CONFIG_LEGS = [
    # (workload, backend, timed steps, warm-up steps, latency seeds)
    ("quad12_narrow", "cuda-f32", 2, 1, 20),        # configs[1]
    ("dubins6_building", "cuda-f32", 2, 1, 20),     # configs[2]
    ("di12_forest", "cuda-f32", 2, 1, 20),          # configs[3]
    ("di24_forest", "cuda-f32", 2, 1, 20),          # configs[3]
    ("quad12_config5", "cuda-f32", 1, 1, 0),        # configs[4]: 8192 queries with per-query goals
    ("di6_forest", "cuda", 2, 1, 20),               # the float64 (bit-parity) kernels on the headline workload
    ("di6_forest", "cuda-f32-philox", 2, 1, 20),    # the production Philox4x32-10 stream on the headline workload
]


def config_leg(ctx, workload, backend, steps, warmup, lat_seeds, peaks):
    np = ctx.np
    t = throughput_leg(ctx, workload, backend, steps, warmup, peaks=peaks)
    rec = t["rec"]
    ent = {"workload": workload, "backend": backend, "plans_per_s": t["value"], "steps": steps, "warmup": warmup,
           "queries_per_step": t["q_total"], "ms_per_step": t["total_ms"] / steps,
           "batch_solved": int((rec["status"] == 0).sum()), "batch_queries": int(len(rec)),
           "batch_revalidated_f64": int((rec["checked"] == 1).sum()),
           "roofline": {"bound": "fp32" if "f32" in backend else "fp64", "achieved": t["achieved_tflops"],
                        "peak": t.get("peak_tflops"), "unit": "TFLOP/s", "frac": t.get("frac")}}
    traffic, traffic_src, hbm = _traffic(workload, t["q_here"], t["kern_ms"])
    if traffic is not None:
        ent["roofline"].update({"traffic": traffic, "traffic_source": traffic_src, "hbm": hbm})
    gold = os.path.join(ROOT, "tests", "golden", f"outcomes_{workload}.json")
    if os.path.isfile(gold) and ctx.world == 1 and len(rec) >= 100:
        g = json.load(open(gold))                          # the batch's first 100 queries are seeds 0..99
        ent["success_100_seeds"] = int((rec["status"][:100] == 0).sum())
        ent["reference_success_100_seeds"] = sum(1 for r in g["records"] if r["seed"] < 100 and r["status"] == "solved")
    if lat_seeds and ctx.rank == 0:
        lat = latency_leg(ctx, workload, backend, lat_seeds, fine_check=False)
        ent["median_time_to_solution_ms"] = lat["median_wall_ms"]
        ent["median_device_ms"] = lat["median_device_ms"]
        ent["latency_seeds_solved"] = f"{lat['solved']}/{lat['seeds']}"
    return ent


def run_gpu(args):
    ctx = _Ctx(args)
    rank, world = ctx.rank, ctx.world
    model_name, scene, f_step, q_per_team = WORKLOADS[args.workload]

    # CPU baselines first (rank 0, N=1 only), before this process touches CUDA: bounded samples, one plan per core
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = max(1, min(os.cpu_count() or 1, 64))
        r = cpu_throughput(args.workload, cores, cores)
        cpu = {"value": r["plans_per_s"], "unit": "plans/s", "cores": cores, "kind": "port",
               "sample": f"{r['plans']} plans (seeds 0..{cores - 1}), one single-thread process per core, C oracle "
                         f"(bit-exact restatement of the reference planner), {r['wall_s']:.1f} s wall, "
                         f"median {1e3 * r['median_plan_s']:.0f} ms per plan, {r['solved']} solved"}
        ref = reference_throughput(args.workload, min(cores, 8), min(cores, 8))
        if ref is not None:      # the UNMODIFIED reference's own plan(), threads=1, one process per plan
            cpu["reference_unmodified"] = {
                "kind": "reference", "value": ref["plans_per_s"], "unit": "plans/s", "cores": ref["procs"],
                "median_wall_time_ms": 1e3 * ref["median_plan_s"], "solved": ref["solved"],
                "sample": f"{ref['plans']} plans (seeds 0..{ref['plans'] - 1}) through baseline/_ref "
                          f"(kinopax.plan, compiled backend, threads=1), one process per plan, {ref['wall_s']:.1f} s wall"}

    ctx.init_device()
    kp, _lib, np, torch = ctx.kp, ctx._lib, ctx.np, ctx.torch
    model, env, cfg, _, _ = ctx.scene(args.workload)

    # ---- latency leg: one query at a time on the whole GPU, seeds 0..99 (BASELINE.json's time-to-solution)
    lat = None
    if rank == 0 and not args.no_latency:
        lat = latency_leg(ctx, args.workload, args.backend, args.latency_seeds)

    # ---- kernel seam leg (rank 0, N = 1): the reference's compiled kernel beside the CUDA backend
    seam = None
    if rank == 0 and world == 1 and not args.no_kernel_seam:
        try:
            seam = kernel_seam(kp, cfg, env, model, ctx.local)
        except Exception as exc:                     # the seam leg must never take the headline down with it
            seam = {"error": f"{type(exc).__name__}: {exc}"}

    # non-tensor compute peak measured in this run (MEASURED_PEAKS.json holds only HBM / bf16 numbers)
    fp32_peak, fp64_peak = _lib.C.c_double(0), _lib.C.c_double(0)
    if rank == 0:
        _lib.check(ctx.L.kpx_fma_peak(ctx.local, 30.0, _lib.C.byref(fp32_peak), _lib.C.byref(fp64_peak)), "kpx_fma_peak")
    peaks = {"f32": fp32_peak.value, "f64": fp64_peak.value}

    # ---- throughput leg (the headline `value`) and the end-to-end leg
    head = throughput_leg(ctx, args.workload, args.backend, args.steps, args.warmup, queries=args.queries,
                          team_ctas=args.team_ctas, e2e_steps=max(1, min(args.steps, 5)), clocks=True, peaks=peaks)
    rec = head["rec"]

    # ---- BASELINE.json's other configurations (bounded legs); config 5 also under multi-GPU runs (it is the
    # configuration that is sharded q mod N), the rest at N = 1
    configs = []
    if not args.no_configs:
        for wl, be, st, wu, ls in CONFIG_LEGS:
            if (wl, be) == (args.workload, args.backend) or (world > 1 and wl != "quad12_config5"):
                continue
            try:
                ent = config_leg(ctx, wl, be, st, wu, ls, peaks)
            except Exception as exc:
                ent = {"workload": wl, "backend": be, "error": f"{type(exc).__name__}: {exc}"}
            configs.append(ent)

    if rank != 0:
        return
    okc, agree, checked = head["host_check"]
    traffic, traffic_src, hbm = _traffic(args.workload, head["q_here"], head["kern_ms"])
    line = {
        "metric": "plans_per_sec", "value": head["value"], "unit": "plans/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["total_ms"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.workload == "quad12_config5" else "weak",
        "vs_baseline": None, "dtype": "f32" if "f32" in args.backend else "f64", "data": "synthetic",
        "config": workload_config(args.workload, model, cfg.t_e, cfg.t_prop, cfg.cells_per_dim),
        "run": {"queries_per_gpu_per_step": head["q_here"], "team_ctas": head["team_ctas"], "teams": head["teams"],
                "backend": args.backend},
        "median_time_to_solution_ms": lat["median_wall_ms"] if lat else None,
        "success_rate": lat["success_rate"] if lat else float((rec["status"] == 0).mean()),
        "time_to_solution": lat,
        "batch": {"solved": int((rec["status"] == 0).sum()), "queries": int(len(rec)),
                  "revalidated_f64_on_device": int((rec["checked"] == 1).sum()),
                  "rejected_by_revalidation": int((rec["checked"] == -1).sum()),
                  "query_device_ms": {"median": float(np.median(rec["device_ms"])),
                                      "p90": float(np.percentile(rec["device_ms"], 90)),
                                      "max": float(rec["device_ms"].max())},
                  "median_iterations": float(np.median(rec["iterations"])),
                  "median_tree_size": float(np.median(rec["tree_size"])), "host_checker_sample": f"{okc}/{checked}",
                  "host_and_device_verdicts_agree": f"{agree}/{checked}"},
        "e2e": head["e2e"],
        # per step: plan_kernel, the six hand-off stages (a small kernel that clears the suspended queries' stop words
        # + plan_kernel on teams of 2 / 4 / 8 / 16 / 64 / all CTAs, each), validate_kernel
        "gpu_launches": 14 * args.steps,
        "roofline": {"bound": "fp32" if "f32" in args.backend else "fp64", "achieved": head["achieved_tflops"],
                     "peak": head["peak_tflops"], "unit": "TFLOP/s", "frac": head["frac"], "traffic": traffic,
                     "traffic_source": traffic_src, "hbm": hbm,
                     "kernel": "kpx::plan_kernel (one persistent launch per step + six short follow-up launches that finish "
                               "the last queries on wider and wider teams; the validate kernel after them is < 1 % of the step)", "kernel_ms": head["kern_ms"],
                     "algorithmic_flops_per_launch": head["flops"],
                     "note": "non-tensor compute bound (no dense contraction): peak = FMA micro-benchmark measured "
                             "in this run (MEASURED_PEAKS.json holds only HBM / bf16 numbers); achieved counts "
                             "SURVEY 8(d) algorithmic ops: substeps*F_step + box tests*2n + collision points*(6+6*n_obs)",
                     "hbm_gbs_measured_peak": _measured_hbm()},
        "clocks": head["clocks"],
    }
    if configs:
        line["configs"] = configs
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if seam is not None:
        line["kernel_seam"] = seam
    print(json.dumps(line), flush=True)


def _measured_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.isfile(p):
        return json.load(open(p)).get("hbm_gbs")
    return 6650.0


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_spawn(args) -> int:
    """`python bench.py --gpus N` outside torchrun: launch the N ranks ourselves, exactly as the driver would
    (one process per GPU, NCCL), and pass the ranks' output through."""
    if "KPX_BENCH_DEVICE" not in os.environ:       # (the test hook that puts every rank on one GPU)
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py --gpus {args.gpus}: one rank per GPU, but only {have} GPU(s) are visible\n")
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="di6_forest", choices=sorted(WORKLOADS))
    ap.add_argument("--backend", default="cuda-f32", choices=["cuda", "cuda-f32", "cuda-philox", "cuda-f32-philox"])
    ap.add_argument("--queries", type=int, default=0, help="queries per GPU per step (default per workload)")
    ap.add_argument("--team-ctas", type=int, default=1)
    ap.add_argument("--latency-seeds", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-kernel-seam", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the bounded legs of BASELINE.json's other configurations")
    ap.add_argument("--port", action="store_true", help="--impl reference: time the C port even when baseline/_ref is installed")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(self_spawn(args))
    else:
        if "RANK" in os.environ and int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")
        run_gpu(args)


if __name__ == "__main__":
    main()
