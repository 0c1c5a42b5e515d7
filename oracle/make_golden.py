#!/usr/bin/env python3
"""TEST INFRASTRUCTURE ONLY -- generate golden vectors from the UNMODIFIED reference.

Run in the build container (needs /root/reference; uses the reference's compiled
kernel from oracle/_ref when built, else its Python backend):

    python oracle/make_golden.py small      # seconds: rng, scenes, batches, plan digests
    python oracle/make_golden.py runner     # ~a minute: the files the reference's bench harness writes (records / summary / csv)
    python oracle/make_golden.py stacked    # ~a minute: stacked integrators (12D/24D) through the Python backend
    python oracle/make_golden.py outcomes   # minutes: full-size solves, seeds 0..N-1

Outputs go to tests/golden/.  Nothing here imports the product package: every
number is produced by the reference's own code.
"""
from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, HERE)
import ref_loader  # noqa: E402


def _digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def _cfg(K, model, t_e, seed, **kw):
    return K.PlannerConfig(t_e=t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim,
                           seed=seed, **kw)


def gen_rng(K):
    from kinopax import rng
    cases = []
    for seed, it, slot, ext, phase in [(0, 1, 0, 0, 1), (99, 4, 0, 2, 1), (-1, 0, 0, 0, 1), (123, 5, 17, 3, 2),
                                       (2 ** 63 + 5, 2 ** 32, 2 ** 20, 63, 3), (7, 11, 199999, 31, 4)]:
        key = rng.stream_key(seed, it, slot, ext, phase)
        draws = [rng.draw_u64(key, i) for i in range(6)]
        cases.append({"seed": seed, "iteration": it, "slot": slot, "ext": ext, "phase": phase,
                      "key": str(key), "draws": [str(d) for d in draws],
                      "units": [rng.u64_to_unit(d).hex() for d in draws]})
    mixes = [{"z": str(z), "mix": str(rng.mix64(z))} for z in (0, 1, 2 ** 64 - 1, 0x9E3779B97F4A7C15, 123456789)]
    json.dump({"stream_cases": cases, "mix64": mixes}, open(os.path.join(GOLD, "rng.json"), "w"), indent=1)


def gen_scenes(K):
    out = {}
    for kind in ("forest", "narrow", "building"):
        for model in ("di6", "dubins6", "quad12"):
            for seed in (0, 1, 5):
                env = K.gen_environment(kind, model, seed=seed)
                out[f"{kind}/{model}/{seed}"] = {
                    "name": env.name, "obs_min": env.obstacles_min.tolist(), "obs_max": env.obstacles_max.tolist(),
                    "start": env.start.tolist(), "goal": env.goal.center.tolist() + [env.goal.radius]}
    json.dump(out, open(os.path.join(GOLD, "scenes.json"), "w"))


def _grown(K, model_name, t_e, iters, seed, lam_cap=8):
    """The reference tests' canonical way to get a realistic batch (tests/test_backends.py:21-34)."""
    from kinopax.planner import TAG_EXPAND, KinoPax
    model = K.get_model(model_name)
    env = K.gen_environment("forest", model, seed=0)
    eng = KinoPax(_cfg(K, model, t_e, seed), env, model)
    for _ in range(iters):
        eng.iteration += 1
        ve = len(eng.arena.slots_with_tag(TAG_EXPAND))
        staged = eng.propagate_pass(min(lam_cap, max(1, (t_e - eng.arena.size) // ve)))
        eng.update_estimates_pass()
        eng.update_node_sets_pass(staged)
    return eng


def gen_batches(K):
    from kinopax.backend import CompiledBackend, PythonBackend, compiled_available
    from kinopax.planner import TAG_EXPAND
    for model_name in ("di6", "dubins6", "quad12"):
        eng = _grown(K, model_name, t_e=2500, iters=5, seed=0)
        e_slots = eng.arena.slots_with_tag(TAG_EXPAND)[:400]
        it = eng.iteration + 1
        py = PythonBackend().propagate_batch(eng.ctx, eng.arena.states, e_slots, 4, it)
        backend = "python"
        if compiled_available():
            cc = CompiledBackend().propagate_batch(eng.ctx, eng.arena.states, e_slots, 4, it)
            for f in ("control", "dt", "accept_u", "valid", "region", "sub"):
                assert np.array_equal(getattr(cc, f), getattr(py, f)), f
            assert np.max(np.abs(cc.end - py.end)) < 1e-12
            py, backend = cc, "compiled"
        c = eng.ctx
        np.savez_compressed(
            os.path.join(GOLD, f"batch_{model_name}.npz"),
            states=eng.arena.states[: eng.arena.size], e_slots=e_slots, lam=4, iteration=it, seed=c.seed,
            t_prop=c.t_prop, state_lo=c.state_lo, state_hi=c.state_hi, obs_min=c.obs_min, obs_max=c.obs_max,
            check_res=c.check_res, grid_lo=c.grid_lo, grid_width=c.grid_width, grid_cells=c.grid_cells,
            grid_strides=c.grid_strides, subcells=c.subcells, backend=backend,
            valid=py.valid, region=py.region, sub=py.sub, end=py.end, control=py.control, dt=py.dt,
            accept_u=py.accept_u)
        print("batch", model_name, "items", py.items, "valid", int(py.valid.sum()), backend)


def _step_digest(eng):
    a, d = eng.arena, eng.decomp
    s = a.size
    return {
        "tree": _digest(a.states[:s], a.parent[:s], a.control[:s], a.dt[:s], a.tag[:s], a.region[:s]),
        "tree_int": _digest(a.parent[:s], a.tag[:s], a.region[:s]),
        "counters": _digest(d.n_valid, d.n_invalid, d.cov, d.visited, d.avail_mask.astype(np.uint8)),
        "estimates": _digest(d.free_vol, d.score, d.p_accept),
    }


def gen_plans(K):
    """Per-iteration digests of complete small plans + the final tree of one of them."""
    from kinopax.planner import TAG_EXPAND, TAG_OPEN, KinoPax, compute_branching_factor
    cases = [("di6", "forest", 6000, 1), ("di6", "narrow", 3000, 2), ("dubins6", "building", 5000, 2),
             ("quad12", "narrow", 8000, 3), ("di6", "building", 20000, 4), ("quad12", "forest", 12000, 5)]
    out = []
    for model_name, kind, t_e, seed in cases:
        model = K.get_model(model_name)
        env = K.gen_environment(kind, model, seed=0)
        cfg = _cfg(K, model, t_e, seed)
        eng = KinoPax(cfg, env, model)
        iters = []
        status = "running"
        while status == "running" and eng.iteration < 80:
            eng.iteration += 1
            ve = len(eng.arena.slots_with_tag(TAG_EXPAND))
            lam = compute_branching_factor(cfg.t_e, eng.arena.size, ve, cfg.lambda_max)
            staged = eng.propagate_pass(lam)
            eng.update_estimates_pass()
            slot, exhausted, appended = eng.update_node_sets_pass(staged)
            rec = {"iteration": eng.iteration, "branching": lam, "ve_size": ve,
                   "vo_size": int(len(eng.arena.slots_with_tag(TAG_OPEN))), "attempted": staged.attempted,
                   "valid": staged.valid_count, "staged": len(staged), "appended": appended,
                   "tree_size": eng.arena.size}
            rec.update(_step_digest(eng))
            iters.append(rec)
            if slot is not None:
                status = "solved"
            elif exhausted:
                status = "capacity_exhausted"
        case = {"model": model_name, "scene": kind, "t_e": t_e, "seed": seed, "status": status,
                "solution_slot": None if status != "solved" else int(slot), "iterations": iters}
        out.append(case)
        print("plan", model_name, kind, t_e, seed, status, "iters", len(iters), "size", eng.arena.size)
        if (model_name, kind) == ("di6", "forest"):
            s = eng.arena.snapshot()
            np.savez_compressed(os.path.join(GOLD, "tree_di6_forest_te6000_s1.npz"),
                                **{k: v for k, v in s.items() if k != "size"}, size=s["size"],
                                p_accept=eng.decomp.p_accept, n_valid=eng.decomp.n_valid,
                                n_invalid=eng.decomp.n_invalid, cov=eng.decomp.cov)
    json.dump(out, open(os.path.join(GOLD, "plans.json"), "w"), indent=1)


def gen_checker(K):
    """Known answers of the reference checker (validity.py) on solved trajectories."""
    out = []
    for model_name, kind, t_e, seed in [("di6", "forest", 30000, 0), ("dubins6", "forest", 30000, 1),
                                        ("quad12", "forest", 60000, 0)]:
        model = K.get_model(model_name)
        env = K.gen_environment(kind, model, seed=0)
        res = K.plan(_cfg(K, model, t_e, seed), env, model)
        if not res.solved:
            print("checker case not solved", model_name)
            continue
        segs = res.trajectory
        rec = {"model": model_name, "scene": kind, "t_e": t_e, "seed": seed,
               "seg_start": [s.start_state.tolist() for s in segs], "seg_control": [s.control.tolist() for s in segs],
               "seg_dt": [s.dt for s in segs], "end_state": segs[-1].end_state.tolist(), "valid": {}}
        for r in (0.05, 0.005):
            rec["valid"][str(r)] = bool(K.ValidityChecker(env, model, r).trajectory_valid(segs, start=env.start))
        # a deliberately broken copy: shift the first control -> chain/goal must fail
        out.append(rec)
        print("checker", model_name, len(segs), rec["valid"])
    json.dump(out, open(os.path.join(GOLD, "checker.json"), "w"))


def stacked_reference_model(K, blocks):
    """BASELINE.json config 4 as the REFERENCE sees it: `blocks` stacked 3-D double integrators as a
    custom DynamicsModel with kernel_id=None, which the reference runs through its Python backend (_purepy.py).
    Built from the reference's own dataclass; nothing of the product package is involved."""
    from kinopax.dynamics import DynamicsModel
    n = 6 * blocks

    def f(x, u, out):
        for b in range(blocks):
            out[6 * b:6 * b + 3] = x[6 * b + 3:6 * b + 6]
            out[6 * b + 3:6 * b + 6] = u[3 * b:3 * b + 3]

    lo = np.tile(np.array([0.0] * 3 + [-5.0] * 3), blocks)
    hi = np.tile(np.array([10.0] * 3 + [5.0] * 3), blocks)
    lo[:3] = np.nan
    hi[:3] = np.nan
    return DynamicsModel(name=f"di{n}", n=n, control_dim=3 * blocks, control_lo=np.full(3 * blocks, -2.0),
                         control_hi=np.full(3 * blocks, 2.0), nonposition_lo=lo, nonposition_hi=hi, deriv_fn=f,
                         wrap_dims=(), dim_kinds=np.tile(np.array([0, 0, 0, 1, 1, 1]), blocks), kernel_id=None,
                         default_t_e=200_000, default_cells_per_dim={1: 4, 2: 3}.get(blocks, 1), default_t_prop=1.0)


def stacked_reference_env(K, model):
    """The di6 Trees scene with block 1 at the scene's start and the other blocks at the centre of their box, at rest."""
    base = K.gen_environment("forest", "di6", seed=0)
    start = np.tile(np.array([5.0, 5.0, 5.0, 0.0, 0.0, 0.0]), model.n // 6)
    start[:3] = base.start[:3]
    return K.Environment(name=f"forest-{model.name}", workspace_lo=base.workspace_lo, workspace_hi=base.workspace_hi,
                         obstacles_min=base.obstacles_min, obstacles_max=base.obstacles_max, start=start, goal=base.goal)


STACKED_CASES = [(2, 1200, 3, 7), (4, 900, 5, 6)]      # (blocks, t_e, seed, iterations)


def gen_stacked(K):
    """Pins oracle model id 3 (stacked integrators, 12D and 24D) to the reference's Python backend: per-iteration
    digests of the tree, the counters and the estimates, plus the last iteration's whole Batch."""
    from kinopax.planner import TAG_EXPAND, TAG_OPEN, KinoPax, compute_branching_factor
    out = []
    for blocks, t_e, seed, n_iter in STACKED_CASES:
        model = stacked_reference_model(K, blocks)
        env = stacked_reference_env(K, model)
        cfg = _cfg(K, model, t_e, seed)
        eng = KinoPax(cfg, env, model)
        assert eng.backend.name == "python", eng.backend.name
        iters = []
        t0 = time.perf_counter()
        for _ in range(n_iter):
            eng.iteration += 1
            e_slots = eng.arena.slots_with_tag(TAG_EXPAND)
            lam = compute_branching_factor(cfg.t_e, eng.arena.size, len(e_slots), cfg.lambda_max)
            batch = eng.backend.propagate_batch(eng.ctx, eng.arena.states, e_slots, lam, eng.iteration)
            staged = eng.propagate_pass(lam)
            eng.update_estimates_pass()
            slot, exhausted, appended = eng.update_node_sets_pass(staged)
            rec = {"iteration": eng.iteration, "branching": lam, "ve_size": int(len(e_slots)),
                   "vo_size": int(len(eng.arena.slots_with_tag(TAG_OPEN))), "attempted": staged.attempted,
                   "valid": staged.valid_count, "staged": len(staged), "appended": appended,
                   "tree_size": eng.arena.size,
                   "batch": _digest(batch.valid, batch.region, batch.sub, batch.end, batch.control, batch.dt, batch.accept_u)}
            rec.update(_step_digest(eng))
            iters.append(rec)
            if slot is not None or exhausted:
                break
        out.append({"blocks": blocks, "t_e": t_e, "seed": seed, "cells": model.default_cells_per_dim, "iterations": iters})
        print("stacked", model.name, "iters", len(iters), "size", eng.arena.size, f"{time.perf_counter() - t0:.1f} s")
    json.dump(out, open(os.path.join(GOLD, "plans_stacked.json"), "w"), indent=1)


RUNNER_CASES = [("di6", "forest", 6000, 1, 8), ("dubins6", "building", 20000, 2, 4)]   # model, scene, t_e, first seed, trials
RUNNER_SWEEP = ("di6", "forest", [1500, 3000, 6000], 3, 6)                              # model, scene, t_e values, first seed, trials


def gen_runner(K):
    """The files the reference's own harness writes (bench.py:106-257: records.jsonl, summary.json, trajectory.csv +
    sidecar, regions_trialNNN.csv, sweep.jsonl) on small configurations: the fixtures the product's runner is
    diffed against (tests/test_runner_gpu.py)."""
    import shutil
    from kinopax import bench
    for model_name, kind, t_e, seed, trials in RUNNER_CASES:
        model = K.get_model(model_name)
        env = K.gen_environment(kind, model, seed=0)
        out = os.path.join(GOLD, f"runner_{model_name}_{kind}")
        shutil.rmtree(out, ignore_errors=True)
        table, _ = bench.run_trials(_cfg(K, model, t_e, seed), env, model, "kinopax", trials, out_dir=out,
                                    dump_regions_dir=out)
        print("runner", model_name, kind, "solved", table.solved, "/", table.trials, "reval failures", table.revalidation_failures)
    model_name, kind, tes, seed, trials = RUNNER_SWEEP
    model = K.get_model(model_name)
    out = os.path.join(GOLD, f"runner_sweep_{model_name}_{kind}")
    shutil.rmtree(out, ignore_errors=True)
    rows = bench.sweep_te(_cfg(K, model, tes[0], seed), K.gen_environment(kind, model, seed=0), model, tes, trials, out_dir=out)
    print("sweep", [(r["t_e"], r["failures"]) for r in rows])


# ------------------------------------------------------------------ full-size outcomes

CONFIGS = {
    "di6_forest": ("di6", "forest"), "quad12_narrow": ("quad12", "narrow"), "dubins6_building": ("dubins6", "building"),
    "quad12_forest": ("quad12", "forest"),
}


def _solve_one(args):
    name, seed = args
    K = ref_loader.load_reference()
    model_name, kind = CONFIGS[name]
    model = K.get_model(model_name)
    env = K.gen_environment(kind, model, seed=0)
    cfg = _cfg(K, model, model.default_t_e, seed, t_max=120.0)
    t0 = time.perf_counter()
    res = K.plan(cfg, env, model)
    rec = {"seed": seed, "status": res.status.value, "iterations": res.stats.iterations,
           "tree_size": res.stats.tree_size, "wall_time_ms": res.stats.wall_time_ms,
           "solution_duration_s": res.stats.solution_duration_s, "segments": len(res.trajectory)}
    if res.solved:
        rec["reval_res"] = bool(K.ValidityChecker(env, model, 0.05).trajectory_valid(res.trajectory, start=env.start))
        rec["reval_fine"] = bool(K.ValidityChecker(env, model, 0.005).trajectory_valid(res.trajectory, start=env.start))
    rec["total_s"] = time.perf_counter() - t0
    return name, rec


def gen_outcomes(names, n_seeds, procs):
    jobs = [(n, s) for n in names for s in range(n_seeds)]
    out = {n: [] for n in names}
    with mp.Pool(procs) as pool:
        for name, rec in pool.imap_unordered(_solve_one, jobs):
            out[name].append(rec)
            print(name, rec["seed"], rec["status"], f"{rec['wall_time_ms']:.0f} ms", flush=True)
    for n in names:
        recs = sorted(out[n], key=lambda r: r["seed"])
        solved = [r for r in recs if r["status"] == "solved"]
        summary = {"config": n, "model": CONFIGS[n][0], "scene": CONFIGS[n][1], "seeds": n_seeds,
                   "solved": len(solved),
                   "median_ms_solved": float(np.median([r["wall_time_ms"] for r in solved])) if solved else None,
                   "reval_res_fail": sum(1 for r in solved if not r["reval_res"]),
                   "reval_fine_fail": sum(1 for r in solved if not r["reval_fine"]),
                   "host": f"{os.cpu_count()} vCPU build container, compiled backend threads=1, {procs} procs",
                   "records": recs}
        json.dump(summary, open(os.path.join(GOLD, f"outcomes_{n}.json"), "w"), indent=1)
        print("outcomes", n, "solved", len(solved), "/", n_seeds, "median ms", summary["median_ms_solved"])


def main():
    os.makedirs(GOLD, exist_ok=True)
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    K = ref_loader.load_reference()
    print("reference backends:", K.available_backends())
    if what == "small":
        gen_rng(K)
        gen_scenes(K)
        gen_batches(K)
        gen_plans(K)
        gen_checker(K)
    elif what == "runner":
        gen_runner(K)
    elif what == "stacked":
        gen_stacked(K)
    elif what == "outcomes":
        names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["di6_forest"]
        n_seeds = int(sys.argv[3]) if len(sys.argv) > 3 else 100
        procs = int(sys.argv[4]) if len(sys.argv) > 4 else os.cpu_count()
        gen_outcomes(names, n_seeds, procs)
    else:
        raise SystemExit(f"unknown target {what}")


if __name__ == "__main__":
    main()
