"""GPU parity tests proper: the CUDA path (through the C ABI) against the CPU oracle and the
golden vectors recorded from the unmodified reference.

Bars (BASELINE.json north_star): RNG draws, controls, durations, collision verdicts, region /
sub-region indices, region counters, first-visit winners and compaction slots are BIT-EXACT;
float64 end states are bit-exact for the double integrator and within 1e-12 for the trig models
(CUDA libm vs glibc, the tolerance the reference uses between its own two backends,
tests/test_backends.py:44-53); float32 end states agree within 1e-5 relative.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, make_empty_env, small_cfg

pytestmark = pytest.mark.gpu

F32_RTOL = 1e-5      # north_star: "propagated states agree within 1e-5 relative (FP32 vs float64)"
TRIG_ATOL = 1e-12    # reference's own cross-backend tolerance for trig models


def _ctx_from_golden(kp, g, model):
    from paper_2409_06807_b200.backend import PlanContext
    return PlanContext(model=model, seed=int(g["seed"]), t_prop=float(g["t_prop"]), state_lo=g["state_lo"],
                       state_hi=g["state_hi"], obs_min=g["obs_min"], obs_max=g["obs_max"],
                       check_res=float(g["check_res"]), grid_lo=g["grid_lo"], grid_width=g["grid_width"],
                       grid_cells=g["grid_cells"], grid_strides=g["grid_strides"], subcells=int(g["subcells"]))


def _wrap_diff(a, b, wrap_dims):
    d = np.abs(a - b)
    for w in wrap_dims:
        d[:, w] = np.minimum(d[:, w], np.abs(2 * np.pi - d[:, w]))
    return d


@pytest.mark.parametrize("model_name", ["di6", "dubins6", "quad12"])
def test_batch_parity_f64_vs_reference_golden(kp, model_name):
    """tests/test_backends.py:37-54 with the CUDA backend in the compiled backend's place."""
    g = np.load(os.path.join(GOLDEN, f"batch_{model_name}.npz"))
    model = kp.get_model(model_name)
    b = kp.get_backend("cuda").propagate_batch(_ctx_from_golden(kp, g, model), g["states"], g["e_slots"],
                                               int(g["lam"]), int(g["iteration"]))
    assert np.array_equal(b.control, g["control"])
    assert np.array_equal(b.dt, g["dt"])
    assert np.array_equal(b.accept_u, g["accept_u"])
    assert np.array_equal(b.valid, g["valid"])
    assert np.array_equal(b.region, g["region"])
    assert np.array_equal(b.sub, g["sub"])
    if model_name == "di6":
        assert np.array_equal(b.end, g["end"])
    else:
        assert np.max(_wrap_diff(b.end, g["end"], model.wrap_dims)) < TRIG_ATOL


@pytest.mark.parametrize("model_name", ["di6", "dubins6", "quad12"])
def test_batch_parity_f32_tolerance(kp, model_name):
    g = np.load(os.path.join(GOLDEN, f"batch_{model_name}.npz"))
    model = kp.get_model(model_name)
    b = kp.get_backend("cuda-f32").propagate_batch(_ctx_from_golden(kp, g, model), g["states"], g["e_slots"],
                                                   int(g["lam"]), int(g["iteration"]))
    # sampling is done in float64 on the device even in the float32 build: bit-exact
    assert np.array_equal(b.control, g["control"]) and np.array_equal(b.dt, g["dt"])
    assert np.array_equal(b.accept_u, g["accept_u"])
    # tolerance is stated on the states that can enter the tree (valid in both); an invalid quadcopter item
    # keeps integrating after leaving the box (reference rule 11) and may pass the tan(pitch) singularity,
    # where float32 and float64 trajectories legitimately diverge
    both_valid = (b.valid == 1) & (g["valid"] == 1)
    assert both_valid.sum() > 0.9 * g["valid"].sum()
    scale = np.maximum(np.abs(g["end"]), 1.0)
    rel = (_wrap_diff(b.end, g["end"], model.wrap_dims) / scale)[both_valid]
    assert np.max(rel) < F32_RTOL, np.max(rel)
    # Verdicts / cells may flip only for items that sit within float32 rounding of a boundary.  Measured on B200:
    # no flip at all on these batches (1200-1600 items); the bar leaves room for one such item per thousand, and
    # every flip must be explained by a boundary within a few float32 ulps of the float64 end state.
    agree = (b.valid == g["valid"]) & (b.region == g["region"])
    both = (b.valid == 1) & (g["valid"] == 1) & (b.region == g["region"])
    sub_ok = b.sub[both] == g["sub"][both]
    assert agree.mean() >= 0.999, agree.mean()
    assert sub_ok.mean() >= 0.999, sub_ok.mean()
    flipped = np.flatnonzero((b.region != g["region"]) & (b.valid == 1) & (g["valid"] == 1))
    ulp = 8 * np.finfo(np.float32).eps
    for w in flipped:        # a cell flip: some grid coordinate of the float64 end state is within ulps of a cell edge
        rel = (g["end"][w] - g["grid_lo"]) / g["grid_width"]
        assert np.min(np.abs(rel - np.round(rel))) <= ulp * np.max(np.abs(g["end"][w]) / g["grid_width"] + 1), w
    for w in np.flatnonzero(both)[~sub_ok]:
        rel = (g["end"][w][:3] - g["grid_lo"][:3]) / g["grid_width"][:3] * int(g["subcells"])
        assert np.min(np.abs(rel - np.round(rel))) <= ulp * int(g["subcells"]) * np.max(np.abs(g["end"][w][:3]) / g["grid_width"][:3] + 1), w


def test_kernel_rng_matches_stream(kp):
    """tests/test_rng.py:70-102: one item's controls / duration / gate draw equal the scalar stream."""
    from paper_2409_06807_b200.backend import PlanContext
    from paper_2409_06807_b200.rng import PHASE_ACCEPT, PHASE_SAMPLE, RngStream
    model = kp.get_model("di6")
    ctx = PlanContext(model=model, seed=99, t_prop=1.0, state_lo=np.array([0, 0, 0, -5, -5, -5.0]),
                      state_hi=np.array([10, 10, 10, 5, 5, 5.0]), obs_min=np.zeros((0, 3)), obs_max=np.zeros((0, 3)),
                      check_res=0.05, grid_lo=np.array([0, 0, 0, -5, -5, -5.0]), grid_width=np.full(6, 2.5),
                      grid_cells=np.full(6, 4, dtype=np.int64),
                      grid_strides=np.array([1024, 256, 64, 16, 4, 1], dtype=np.int64), subcells=4)
    states = np.array([[1, 1, 1, 0, 0, 0.0]])
    for name in ("cuda", "cuda-f32"):
        batch = kp.get_backend(name).propagate_batch(ctx, states, np.array([0], dtype=np.int64), 3, iteration=4)
        for ext in range(3):
            s = RngStream(seed=99, iteration=4, slot=0, extension=ext, phase=PHASE_SAMPLE)
            assert batch.control[ext].tolist() == [s.uniform_in(model.control_lo[j], model.control_hi[j])
                                                   for j in range(3)]
            assert batch.dt[ext] == s.duration(1.0)
            assert batch.accept_u[ext] == RngStream(seed=99, iteration=4, slot=0, extension=ext,
                                                    phase=PHASE_ACCEPT).uniform()


def test_batch_edge_cases(kp, orc):
    """Empty batch, single item, no obstacles, ragged (non multiple of the block) sizes, dimension limits."""
    from paper_2409_06807_b200.backend import PlanContext
    model = kp.get_model("di6")
    env = make_empty_env(kp)
    prob = kp.build_problem(small_cfg(kp, model, t_e=100), env, model)
    ctx = PlanContext(model=model, seed=5, t_prop=1.0, state_lo=prob.state_lo, state_hi=prob.state_hi,
                      obs_min=env.obstacles_min, obs_max=env.obstacles_max, check_res=0.05, grid_lo=prob.grid.lo,
                      grid_width=prob.grid.widths, grid_cells=prob.grid.cells, grid_strides=prob.grid.strides,
                      subcells=4)
    be = kp.get_backend("cuda")
    states = np.tile(env.start, (7, 1))
    empty = be.propagate_batch(ctx, states, np.zeros(0, dtype=np.int64), 4, 1)
    assert empty.items == 0 and empty.end.shape == (0, 6)
    octx, keep = orc.ctx_from_problem(prob)
    for m, lam in ((1, 1), (7, 3), (5, 32)):
        slots = np.arange(m, dtype=np.int64)
        a = be.propagate_batch(ctx, states, slots, lam, 2)
        o = orc.propagate_batch(octx, states, slots, lam, 5, 2)
        for f in ("valid", "region", "sub", "end", "control", "dt", "accept_u"):
            assert np.array_equal(getattr(a, f), o[f]), (m, lam, f)
    with pytest.raises(kp.ConfigError):
        be.propagate_batch(ctx, states, np.array([9], dtype=np.int64), 1, 1)       # slot outside states


def _step_compare(kp, orc, model_name, scene, t_e, seed, backend, max_iters=60, env=None):
    model = kp.get_model(model_name) if isinstance(model_name, str) else model_name
    model_name = model.name
    env = kp.gen_environment(scene, model, seed=0) if env is None else env
    cfg = small_cfg(kp, model, t_e=t_e, seed=seed)
    op = orc.plan_from_problem(kp.build_problem(cfg, env, model))
    exact = model_name.startswith("di")
    with kp.KinoPax(cfg, env, model, backend=backend) as eng:
        for it in range(1, max_iters + 1):
            st = eng.step()
            op.step()
            a, b = eng.snapshot(), op.snapshot()
            assert a["size"] == b["size"], (it, a["size"], b["size"])
            for k in ("parent", "tag", "region", "control", "dt"):
                assert np.array_equal(a[k], b[k]), (it, k)
            if exact:
                assert np.array_equal(a["states"], b["states"]), it
            else:
                assert np.max(_wrap_diff(a["states"], b["states"], model.wrap_dims)) < 1e-9, it
            ra, rb = eng.region_state(), op.decomposition()
            for k in ("n_valid", "n_invalid", "cov", "visited"):
                assert np.array_equal(getattr(ra, k), rb[k]), (it, k)
            assert np.array_equal(ra.avail_mask, rb["avail"].astype(bool)), it
            # scores use the reference's expression order; the total is summed in NumPy's pairwise order on the
            # device (decomposition.py:199), so the estimates are bit-identical
            assert np.array_equal(ra.score, rb["score"]), it
            assert np.array_equal(ra.p_accept, rb["p_accept"]), it
            tr, orc_tr = eng.traces()[-1], op.trace()
            for k in ("iteration", "branching", "ve_size", "vo_size", "attempted", "valid", "staged", "appended",
                      "tree_size"):
                assert getattr(tr, k) == orc_tr[k], (it, k)
            # the kernel's per-item results (valid / region / sub / keep / end) of this iteration
            items, ob = eng.last_items(), op.last_batch()
            assert np.array_equal(items["valid"], ob["valid"]), it
            v = ob["valid"].astype(bool)
            # regions of ALL items (an invalid item still counts towards its end state's region; -1 = non-finite)
            assert np.array_equal(items["region"], ob["region"]) and np.array_equal(items["sub"][v], ob["sub"][v])
            keep = np.zeros(len(v), np.uint8)
            keep[ob["staged_idx"]] = 1
            assert np.array_equal(items["keep"], keep), it
            if st.status != 4:
                break
        assert {0: "solved", 1: "timeout", 2: "capacity_exhausted", 4: "running"}[st.status] == op.status
        if st.status == 0:
            assert int(st.solution_slot) == int(op.raw.solution_slot)
        return it


@pytest.mark.parametrize("model_name,scene,t_e,seed", [("di6", "forest", 6000, 1), ("di6", "narrow", 3000, 2),
                                                       ("dubins6", "building", 5000, 2), ("quad12", "narrow", 8000, 3)])
def test_plan_matches_oracle_every_iteration_f64(kp, orc, model_name, scene, t_e, seed):
    """Whole-state parity after every iteration: tree, tags, counters, visited bits, scores, p_accept,
    trace counters, per-item verdicts and the kept set (compaction input) -- the device-side twin of
    tests/test_backends.py:73-85 (tree_snapshot identical across backends)."""
    _step_compare(kp, orc, model_name, scene, t_e, seed, "cuda")


def test_plan_matches_reference_golden_tree(kp):
    """Single-launch solve (no stepping) reproduces the tree the reference itself produced."""
    g = np.load(os.path.join(GOLDEN, "tree_di6_forest_te6000_s1.npz"))
    model = kp.get_model("di6")
    res = kp.plan(small_cfg(kp, model, t_e=6000, seed=1), kp.gen_environment("forest", model, 0), model,
                  backend="cuda", capture_tree=True)
    s = res.tree_snapshot
    assert res.solved and s["size"] == int(g["size"])
    for k in ("states", "parent", "control", "dt", "tag", "region"):
        assert np.array_equal(s[k], g[k]), k
    cases = {(c["model"], c["scene"], c["t_e"], c["seed"]): c for c in json.load(open(os.path.join(GOLDEN, "plans.json")))}
    c = cases[("di6", "forest", 6000, 1)]
    assert res.stats.iterations == len(c["iterations"]) and res.stats.tree_size == c["iterations"][-1]["tree_size"]


def test_team_size_does_not_change_the_tree(kp):
    """Determinism by construction (reference: thread-count invariance, tests/test_backends.py:88-97)."""
    model = kp.get_model("di6")
    env = kp.gen_environment("narrow", model, seed=0)
    cfg = small_cfg(kp, model, t_e=3000, seed=2)
    snaps, regs = [], []
    for team in (0, 1, 3, 16):
        with kp.KinoPax(cfg, env, model, backend="cuda", team_ctas=team) as eng:
            snaps.append(eng.solve(capture_tree=True).tree_snapshot)
            regs.append(eng.region_state())
    for s, r in zip(snaps[1:], regs[1:]):
        assert s["size"] == snaps[0]["size"]
        for k in ("states", "parent", "tag", "region", "dt"):
            assert np.array_equal(s[k], snaps[0][k]), k
        # the score total is summed in one fixed (NumPy pairwise) order whatever the team size
        for k in ("n_valid", "n_invalid", "cov", "visited", "score", "p_accept"):
            assert np.array_equal(getattr(r, k), getattr(regs[0], k)), k


def test_capacity_exhaustion_start_in_goal_and_enclosed_goal(kp, orc):
    model = kp.get_model("di6")
    env = make_empty_env(kp, goal_center=(9.0, 9.0, 9.0))
    res = kp.plan(small_cfg(kp, model, t_e=40, seed=0), env, model)
    assert res.status is kp.PlanStatus.CAPACITY_EXHAUSTED and res.stats.tree_size == 40      # tests/test_planner.py:145
    here = make_empty_env(kp, goal_center=(1.0, 1.0, 1.0))
    res = kp.plan(small_cfg(kp, model, t_e=100), here, model)
    assert res.solved and res.stats.iterations == 0 and res.trajectory == []                  # tests/test_planner.py:153
    # goal sealed inside a box: the run must end by timeout, never claim success
    sealed = kp.Environment("sealed", np.zeros(3), np.full(3, 10.0), np.array([[7.0, 7, 7]]), np.array([[10.0, 10, 10]]),
                            env.start, kp.GoalBall(np.array([8.5, 8.5, 8.5]), 0.5))
    res = kp.plan(small_cfg(kp, model, t_e=3000, t_max=0.05), sealed, model)
    assert res.status in (kp.PlanStatus.TIMEOUT, kp.PlanStatus.CAPACITY_EXHAUSTED)


def test_rescue_rule_matches_oracle(kp, orc):
    """Tiny epsilon-driven demotion empties V_E quickly; the forced promotion must pick the same slot
    (tests/test_planner.py:208)."""
    model = kp.get_model("di6")
    env = kp.gen_environment("building", model, seed=0)
    cfg = kp.PlannerConfig(t_e=400, t_prop=1.0, cells_per_dim=2, epsilon=1e-6, seed=11)
    op = orc.plan_from_problem(kp.build_problem(cfg, env, model))
    with kp.KinoPax(cfg, env, model, backend="cuda") as eng:
        for it in range(40):
            st = eng.step()
            op.step()
            a, b = eng.snapshot(), op.snapshot()
            assert a["size"] == b["size"] and np.array_equal(a["tag"], b["tag"]), it
            assert (a["tag"] == 1).sum() >= 1
            if st.status != 4:
                break


@pytest.mark.parametrize("model_name,scene", [("di6", "forest"), ("dubins6", "building"), ("quad12", "forest")])
def test_solutions_revalidate_f32_and_f64(kp, orc, model_name, scene):
    """Every returned solution is re-validated (dynamically feasible, collision-free, ends in goal) by the
    host checker AND by the oracle's restatement of the reference checker, at the planning resolution."""
    model = kp.get_model(model_name)
    env = kp.gen_environment(scene, model, seed=0)
    t_e = 60000 if model_name != "quad12" else 120000
    for backend in ("cuda", "cuda-f32"):
        solved = 0
        for seed in range(4):
            cfg = small_cfg(kp, model, t_e=t_e, seed=seed)
            res = kp.plan(cfg, env, model, backend=backend)
            if not res.solved:
                continue
            solved += 1
            assert kp.ValidityChecker(env, model, 0.05).trajectory_valid(res.trajectory, start=env.start)
            prob = kp.build_problem(cfg, env, model)
            ctx, keep = orc.ctx_from_problem(prob)
            ok, code = orc.trajectory_valid(ctx, [s.start_state for s in res.trajectory],
                                            [s.control for s in res.trajectory], [s.dt for s in res.trajectory],
                                            env.start, prob.goal4, 0.05)
            assert ok, (backend, seed, code)
        assert solved >= 3, (backend, solved)


def test_load_state_resume_equals_uninterrupted(kp, orc):
    """Checkpoint/resume: load the oracle's state after k iterations, continue on the device, and land on the
    same tree as an uninterrupted device run."""
    model = kp.get_model("di6")
    env = kp.gen_environment("forest", model, seed=0)
    cfg = small_cfg(kp, model, t_e=6000, seed=1)
    op = orc.plan_from_problem(kp.build_problem(cfg, env, model))
    for _ in range(4):
        op.step()
    with kp.KinoPax(cfg, env, model, backend="cuda") as eng:
        eng.load_state(op.snapshot(), op.decomposition(), iteration=4)
        st = eng._run(60.0)
        resumed = eng.snapshot()
    full = kp.plan(cfg, env, model, backend="cuda", capture_tree=True).tree_snapshot
    assert st.status == 0 and resumed["size"] == full["size"]
    for k in ("states", "parent", "tag", "region"):
        assert np.array_equal(resumed[k], full[k]), k


def test_high_dimensional_stacked_integrators(kp, orc):
    """Config 4 (12D/24D/48D): device vs oracle, every iteration, float64."""
    for blocks, t_e in ((2, 3000), (4, 2500), (8, 2000)):
        model = kp.stacked_double_integrator(blocks)
        base = kp.gen_environment("forest", "di6", seed=0)
        start = np.tile(np.array([5.0, 5, 5, 0, 0, 0]), blocks)
        start[:3] = base.start[:3]
        env = kp.Environment(f"forest-{model.name}", base.workspace_lo, base.workspace_hi, base.obstacles_min,
                             base.obstacles_max, start, base.goal)
        _step_compare(kp, orc, model.name, "forest", t_e, 3, "cuda", max_iters=12, env=env)


def test_stacked_integrators_with_block1_grid(kp, orc):
    """Config 4 variant for 24D/48D: the grid spans block 1 only (6 of n dims); device vs oracle, every iteration."""
    import dataclasses
    for blocks, t_e in ((4, 3000), (8, 2500)):
        model = dataclasses.replace(kp.stacked_double_integrator(blocks, grid_dims=6), default_cells_per_dim=4)
        base = kp.gen_environment("forest", "di6", seed=0)
        start = np.tile(np.array([5.0, 5, 5, 0, 0, 0]), blocks)
        start[:3] = base.start[:3]
        env = kp.Environment(f"forest-{model.name}-g6", base.workspace_lo, base.workspace_hi, base.obstacles_min,
                             base.obstacles_max, start, base.goal)
        _step_compare(kp, orc, model, "forest", t_e, 5, "cuda", max_iters=12, env=env)


def test_claim_epochs_run_out_and_wrap(kp):
    """The first-visit table is epoch-tagged (no reset between queries) and refilled only when the epochs run out.
    Crossing that boundary -- last epochs 1 and 0, then the dense refill -- must not change a single plan."""
    from paper_2409_06807_b200 import _lib
    model = kp.get_model("di6")
    env = kp.gen_environment("forest", model, seed=0)
    cfg = small_cfg(kp, model, t_e=6000, seed=4)
    for backend in ("cuda", "cuda-f32"):
        with kp.KinoPax(cfg, env, model, backend=backend) as eng:
            ref = eng.solve(capture_tree=True)
            _lib.check(eng._lib.kpx_plan_set_epoch(eng._handle, 2), "kpx_plan_set_epoch")
            for _ in range(5):                      # epochs 1, 0, refill -> e_max, e_max - 1, ...
                eng.reset(seed=4)
                again = eng.solve(capture_tree=True)
                assert again.status is ref.status and again.stats.iterations == ref.stats.iterations
                assert again.stats.tree_size == ref.stats.tree_size
                for k in ("parent", "tag", "region", "states"):
                    assert np.array_equal(again.tree_snapshot[k], ref.tree_snapshot[k]), k
                ra, rb = eng.region_state(), None
                assert ra.visited.sum() > 0


@pytest.mark.parametrize("backend", ["cuda", "cuda-f32"])
def test_fused_trajectory_call_equals_the_separate_entry_points(kp, backend):
    """kpx_plan_trajectory (one host call) returns exactly what kpx_plan_solution + kpx_trajectory +
    kpx_trajectory_valid return together, for both tree precisions (and hence propagate_ode's samples,
    test_native_trajectory_rebuild_and_check)."""
    for model_name, scene, t_e in (("di6", "forest", 20000), ("quad12", "forest", 60000)):
        model = kp.get_model(model_name)
        env = kp.gen_environment(scene, model, seed=0)
        cfg = small_cfg(kp, model, t_e=t_e, seed=0)
        with kp.KinoPax(cfg, env, model, backend=backend) as eng:
            for seed in range(8):                       # the first seed this small tree solves
                eng.reset(seed=seed)
                res = eng.solve()
                if res.solved and len(res.trajectory) > 0:
                    break
            assert res.solved
            a, ok_a = eng._trajectory()
            b, ok_b = eng._trajectory_general()
            assert ok_a == ok_b and len(a) == len(b) == len(res.trajectory) > 0
            for x, y in zip(a, b):
                assert x.dt == y.dt and np.array_equal(x.control, y.control)
                assert np.array_equal(x.sampled_states, y.sampled_states) and np.array_equal(x.end_state, y.end_state)
            assert kp.ValidityChecker(env, model, 0.05).trajectory_valid(a, start=env.start)


# ---------------------------------------------------------------------------------------------------------------
# float32 production loop: integer bookkeeping held to the reference's rules GIVEN ITS OWN SEGMENTS

@pytest.mark.parametrize("model_name,scene,t_e,seed,team", [("di6", "forest", 6000, 1, 0), ("di6", "forest", 20000, 2, 1),
                                                            ("dubins6", "building", 5000, 2, 0),
                                                            ("quad12", "narrow", 8000, 3, 0), ("quad12", "forest", 30000, 5, 1)])
def test_f32_bookkeeping_is_exact_given_its_own_items(kp, orc, model_name, scene, t_e, seed, team):
    """north_star: "collision verdicts, region counts and compaction indices are bit-exact for the same segments".
    The float32 engine is stepped; after every iteration its own per-item results (valid, region, sub, end state,
    goal test) are handed to the oracle's bookkeeping (kpo_plan_step_given = planner.py:185-265 on a supplied
    Batch).  Region counters, first-visit winners (visited / cov), the kept set, the appended slots (parent,
    region, states), the demote / promote tags, the estimates and the trace counters must then be IDENTICAL --
    for the whole-GPU team (latency build, global sort) and the one-CTA team (throughput build, tile sort)."""
    model = kp.get_model(model_name)
    env = kp.gen_environment(scene, model, seed=0)
    cfg = small_cfg(kp, model, t_e=t_e, seed=seed)
    op = orc.plan_from_problem(kp.build_problem(cfg, env, model))
    f32 = lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)   # noqa: E731
    worst_end = 0.0
    with kp.KinoPax(cfg, env, model, backend="cuda-f32", team_ctas=team) as eng:
        for it in range(1, 80):
            before = op.snapshot()["states"]                                      # == the device tree (float32 values)
            st = eng.step()
            items = eng.last_items()
            ost = op.step_given(items["valid"], items["region"], items["sub"], items["end"], goal_hit=items["goal_hit"])
            ob = op.last_batch()
            # the loop's own end states (the closed-form paths included) against the float64 RK4 of the reference on
            # the same (parent state, control, duration): north_star's 1e-5 relative
            vi = np.flatnonzero(items["valid"])
            for w in vi[:: max(1, len(vi) // 400)]:
                ref = orc.propagate_ode(model.kernel_id, before[items["parent_slot"][w]], f32(ob["control"][w]), float(f32(ob["dt"][w])))[-1]
                err = _wrap_diff(items["end"][w][None, :], ref[None, :], model.wrap_dims)[0] / np.maximum(np.abs(ref), 1.0)
                worst_end = max(worst_end, float(err.max()))
            # the kernel's parent slots are the oracle's e_slots repeated lambda times (ascending V_E order)
            lam = len(items["valid"]) // len(ob["e_slots"])
            assert np.array_equal(items["parent_slot"], np.repeat(ob["e_slots"], lam)), it
            keep = np.zeros(len(items["valid"]), np.uint8)
            keep[ob["staged_idx"]] = 1
            assert np.array_equal(items["keep"], keep), it                       # the kept set (compaction input)
            a, b = eng.snapshot(), op.snapshot()
            assert a["size"] == b["size"], (it, a["size"], b["size"])
            for k in ("parent", "tag", "region"):                                 # appended slots, demote / promote
                assert np.array_equal(a[k], b[k]), (it, k)
            assert np.array_equal(a["states"][1:], b["states"][1:]), it           # the float32 end states, where appended
            assert np.array_equal(a["states"][0], f32(env.start))                 # the root is the start rounded once
            assert np.array_equal(a["control"], f32(b["control"])) and np.array_equal(a["dt"], f32(b["dt"])), it
            ra, rb = eng.region_state(), op.decomposition()
            for k in ("n_valid", "n_invalid", "cov", "visited", "score", "p_accept"):
                assert np.array_equal(getattr(ra, k), rb[k]), (it, k)
            assert np.array_equal(ra.avail_mask, rb["avail"].astype(bool)), it
            tr, otr = eng.traces()[-1], op.trace()
            for k in ("iteration", "branching", "ve_size", "vo_size", "attempted", "valid", "staged", "appended", "tree_size"):
                assert getattr(tr, k) == otr[k], (it, k)
            assert {0: 0, 2: 2, 4: 4}[st.status] == ost, (it, st.status, ost)
            if st.status != 4:
                break
        if st.status == 0:
            assert int(st.solution_slot) == int(op.raw.solution_slot)
        assert it >= 4
    assert worst_end < F32_RTOL, worst_end


def test_time_budget_rules(kp):
    """planner.py:282: the clock is tested BEFORE each iteration -- t_max = 0 runs no iteration at all and reports
    TIMEOUT; a stepped run only counts the time its launches were running, not the host's pauses between them."""
    import time
    model = kp.get_model("di6")
    env = kp.gen_environment("forest", model, seed=0)
    res = kp.plan(small_cfg(kp, model, t_e=6000, seed=1, t_max=0.0), env, model, backend="cuda")
    assert res.status is kp.PlanStatus.TIMEOUT and res.stats.iterations == 0 and res.stats.tree_size == 1
    cfg = small_cfg(kp, model, t_e=6000, seed=1, t_max=0.25)
    with kp.KinoPax(cfg, env, model, backend="cuda") as eng:
        st = eng.step()
        assert st.status == 4 and st.iterations == 1
        time.sleep(0.6)                                  # longer than t_max: must not count
        st = eng.step()
        assert st.status == 4 and st.iterations == 2, (st.status, st.iterations)
        assert st.device_ms < 250.0
        full = eng._run(60.0)
        assert full.status == 0
    ref = kp.plan(small_cfg(kp, model, t_e=6000, seed=1), env, model, backend="cuda")
    assert ref.stats.iterations == full.iterations and ref.stats.tree_size == full.tree_size
    # a run that timed out can be continued with a larger budget
    sealed = kp.Environment("sealed", np.zeros(3), np.full(3, 10.0), np.array([[7.0, 7, 7]]), np.array([[10.0, 10, 10]]),
                            env.start, kp.GoalBall(np.array([8.5, 8.5, 8.5]), 0.5))
    with kp.KinoPax(small_cfg(kp, model, t_e=200000, seed=0, t_max=0.0003), sealed, model, backend="cuda-f32") as eng:
        a = eng._run(0.0003)
        assert a.status == 1 and a.iterations >= 1
        b = eng._run(0.0008)
        assert b.status in (1, 2) and b.iterations > a.iterations


def test_set_obstacles_capacity(kp):
    """kpx_plan_set_obstacles: a plan created without obstacles has no room for one (error, no write); a plan
    created with k obstacles accepts up to k and plans against the new set."""
    from paper_2409_06807_b200 import _lib
    model = kp.get_model("di6")
    cfg = small_cfg(kp, model, t_e=3000, seed=2)
    one_min, one_max = np.array([[4.0, 0.0, 0.0]]), np.array([[6.0, 10.0, 10.0]])          # a wall across the cube
    with kp.KinoPax(cfg, make_empty_env(kp), model, backend="cuda") as eng:
        rc = eng._lib.kpx_plan_set_obstacles(eng._handle, 1, _lib.ptr(one_min), _lib.ptr(one_max))
        assert rc == _lib.E_ARG
        assert eng.solve().solved                        # untouched: still the empty scene
    env = kp.gen_environment("narrow", model, seed=0)
    with kp.KinoPax(cfg, env, model, backend="cuda") as eng:
        rc = eng._lib.kpx_plan_set_obstacles(eng._handle, 3, _lib.ptr(np.zeros((3, 3))), _lib.ptr(np.ones((3, 3))))
        assert rc == _lib.E_ARG                          # created with 2
        _lib.check(eng._lib.kpx_plan_set_obstacles(eng._handle, 1, _lib.ptr(one_min), _lib.ptr(one_max)), "set")
        res = eng.solve()
        assert res.status is not kp.PlanStatus.SOLVED    # the wall seals the goal side off
        _lib.check(eng._lib.kpx_plan_set_obstacles(eng._handle, 0, None, None), "set")
        eng.reset()
        assert eng.solve().solved


# ---------------------------------------------------------------------------------------------------------------
# Philox4x32-10 production stream (north_star: "draws controls from a counter-based Philox stream")

def test_philox_known_answers_on_device(kp):
    from test_host import PHILOX_KAT
    from paper_2409_06807_b200 import _lib
    lib = _lib.load()
    for ctr, key, want in PHILOX_KAT:
        c, k = np.array(ctr, np.uint32), np.array(key, np.uint32)
        host, dev = np.zeros(4, np.uint32), np.zeros(4, np.uint32)
        _lib.check(lib.kpx_philox4x32(_lib.ptr(c), _lib.ptr(k), _lib.ptr(host), _lib.ptr(dev)), "kpx_philox4x32")
        assert tuple(int(x) for x in dev) == want and np.array_equal(host, dev)


@pytest.mark.parametrize("model_name", ["di6", "quad12"])
def test_philox_kernel_draws_match_the_host_stream(kp, model_name):
    """The kernel seam with the Philox backends: every item's controls, duration and gate uniform are the draws of
    the host twin's stream (seed, iteration, slot, extension, phase) -- tests/test_rng.py:70-102 for the production
    generator -- for both precisions; and the integration that follows is the same code as in the parity mode."""
    from paper_2409_06807_b200.rng import PHASE_ACCEPT, PHASE_SAMPLE, PhiloxStream
    g = np.load(os.path.join(GOLDEN, f"batch_{model_name}.npz"))
    model = kp.get_model(model_name)
    ctx = _ctx_from_golden(kp, g, model)
    lam, it = int(g["lam"]), int(g["iteration"])
    slots = g["e_slots"][:40]
    out = {name: kp.get_backend(name).propagate_batch(ctx, g["states"], slots, lam, it) for name in ("cuda-philox", "cuda-f32-philox")}
    for b in out.values():
        for i, slot in enumerate(slots):
            for ext in range(lam):
                w = i * lam + ext
                s = PhiloxStream(int(g["seed"]), it, int(slot), ext, PHASE_SAMPLE)
                assert b.control[w].tolist() == [s.uniform_in(model.control_lo[j], model.control_hi[j]) for j in range(model.control_dim)]
                assert b.dt[w] == s.duration(float(g["t_prop"]))
                assert b.accept_u[w] == PhiloxStream(int(g["seed"]), it, int(slot), ext, PHASE_ACCEPT).uniform()
    a, b = out["cuda-philox"], out["cuda-f32-philox"]
    both = (a.valid == 1) & (b.valid == 1)
    assert both.sum() >= 40 and np.array_equal(a.region[both], b.region[both])
    assert np.max(_wrap_diff(a.end, b.end, model.wrap_dims)[both] / np.maximum(np.abs(a.end[both]), 1.0)) < F32_RTOL
    assert not np.array_equal(a.control, kp.get_backend("cuda").propagate_batch(ctx, g["states"], slots, lam, it).control)


def test_philox_plans_solve_revalidate_and_do_not_depend_on_the_team(kp):
    """Whole plans on the Philox stream: deterministic for any team size, solutions re-validated by the host checker,
    success over 100 seeds of the full-size Trees configuration statistically equal to the reference's."""
    import json
    model = kp.get_model("di6")
    env = kp.gen_environment("forest", model, seed=0)
    cfg = small_cfg(kp, model, t_e=20000, seed=3)
    snaps = []
    for team in (0, 1, 8):
        with kp.KinoPax(cfg, env, model, backend="cuda-philox", team_ctas=team) as eng:
            res = eng.solve(capture_tree=True)
            snaps.append(res.tree_snapshot)
            assert res.solved and kp.ValidityChecker(env, model, 0.05).trajectory_valid(res.trajectory, start=env.start)
    for sn in snaps[1:]:
        assert sn["size"] == snaps[0]["size"]
        for k in ("states", "parent", "tag", "region", "dt", "control"):
            assert np.array_equal(sn[k], snaps[0][k]), k
    ref = kp.plan(cfg, env, model, backend="cuda", capture_tree=True).tree_snapshot
    assert ref["size"] != snaps[0]["size"] or not np.array_equal(ref["dt"], snaps[0]["dt"])      # other random numbers
    gold = json.load(open(os.path.join(GOLDEN, "outcomes_di6_forest.json")))
    ref_solved = sum(1 for r in gold["records"] if r["status"] == "solved")
    full = kp.PlannerConfig(t_e=model.default_t_e, lambda_max=32, t_prop=model.default_t_prop, epsilon=0.005, delta=1.0,
                            cells_per_dim=model.default_cells_per_dim, subcells_per_dim=4, t_max=60.0, seed=0)
    with kp.BatchPlanner(full, env, model, backend="cuda-f32-philox", team_ctas=1) as bp:
        r = bp.run(np.arange(100))
    assert abs(int(r.solved.sum()) - ref_solved) <= 4 and r.validated.sum() == r.solved.sum()
    with kp.KinoPax(full, env, model, backend="cuda-f32-philox") as eng:                         # batch == single query
        for q in (0, 17):
            eng.reset(seed=q)
            one = eng.solve()
            assert one.stats.iterations == r.records["iterations"][q] and one.stats.tree_size == r.records["tree_size"][q]


# ---------------------------------------------------------------------------------------------------------------
# Adaptive tree capacity (Remark 1) -- an extension the reference package does not have; the
# oracle carries the same rule (kpo_plan_set_capacity) so that the device can be held to it bit for bit.

def test_adaptive_capacity_matches_oracle_and_rescues_exhausted_runs(kp, orc):
    model = kp.get_model("di6")
    env = kp.gen_environment("forest", model, seed=0)
    small = small_cfg(kp, model, t_e=1500, seed=3)                    # the reference's own sweep: 6 of 6 seeds fail here
    assert kp.plan(small, env, model, backend="cuda").status is kp.PlanStatus.CAPACITY_EXHAUSTED
    big = small_cfg(kp, model, t_e=12000, seed=3)
    for backend in ("cuda", "cuda-f32"):
        # arena reserved for 12000 nodes, 1500 in effect, doubled whenever the run would end exhausted
        op = orc.plan_from_problem(kp.build_problem(big, env, model))
        op.set_capacity(1500, 2.0)
        with kp.KinoPax(small, env, model, backend=backend, t_e_max=12000, t_e_growth=2.0) as eng:
            for it in range(1, 200):
                st = eng.step()
                if backend == "cuda":
                    op.step()
                    a, b = eng.snapshot(), op.snapshot()
                    assert a["size"] == b["size"], it
                    for k in ("parent", "tag", "region", "states", "dt"):
                        assert np.array_equal(a[k], b[k]), (it, k)
                    assert int(st.capacity) == int(op.raw.t_e), it
                    assert eng.traces()[-1].branching == op.trace()["branching"], it
                if st.status != 4:
                    break
            assert st.status == 0 and int(st.capacity) in (3000, 6000, 12000) and int(st.tree_size) > 1500
            if backend == "cuda":
                assert op.status == "solved" and int(op.raw.growths) >= 1 and int(st.solution_slot) == int(op.raw.solution_slot)
    # t_e_max == t_e is the fixed-capacity planner; growth needs a factor above 1 and t_e_max >= t_e
    with kp.KinoPax(small, env, model, backend="cuda", t_e_max=1500) as eng:
        assert eng.solve().status is kp.PlanStatus.CAPACITY_EXHAUSTED
    for kw in ({"t_e_max": 1000}, {"t_e_max": 3000, "t_e_growth": 1.0}):
        with pytest.raises(kp.ConfigError):
            kp.KinoPax(small, env, model, backend="cuda", **kw)
    # the batch path: every seed of the sweep that failed at 1500 nodes is solved, each with the capacity it needed
    with kp.BatchPlanner(small, env, model, backend="cuda", n_teams=6, team_ctas=1, t_e_max=12000) as bp:
        res = bp.run(np.arange(3, 9))
        assert res.solved.all() and res.validated.all()
        assert set(res.records["capacity"].tolist()) <= {3000, 6000, 12000}
        for q, seed in ((0, 3), (4, 7)):                            # == the oracle planning the same seed
            op = orc.plan_from_problem(kp.build_problem(big.with_seed(seed), env, model))
            op.set_capacity(1500, 2.0)
            op.solve(t_max=60.0)
            assert int(op.raw.size) == res.records["tree_size"][q] and int(op.raw.iteration) == res.records["iterations"][q]
            assert int(op.raw.t_e) == res.records["capacity"][q]
