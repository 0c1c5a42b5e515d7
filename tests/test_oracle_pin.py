"""Pins the CPU oracle (oracle/kpx_oracle.c) to the UNMODIFIED reference.

* against golden vectors the reference itself produced (oracle/make_golden.py): always;
* against the live reference stepped side by side: when /root/reference is mounted.

Everything is bit-exact: the oracle is built with the reference's flags and runs on the
same libm, so even the trig models and p_accept (NumPy pairwise sum) must agree exactly.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, small_cfg


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode()); h.update(str(a.shape).encode()); h.update(a.tobytes())
    return h.hexdigest()


def test_rng_known_answers(orc):
    L = orc.lib()
    g = json.load(open(os.path.join(GOLDEN, "rng.json")))
    for m in g["mix64"]:
        assert L.kpo_mix64(int(m["z"])) == int(m["mix"])
    for c in g["stream_cases"]:
        key = L.kpo_stream_key(c["seed"] & (2**64 - 1), c["iteration"], c["slot"], c["ext"], c["phase"])
        assert key == int(c["key"])
        for i, (d, u) in enumerate(zip(c["draws"], c["units"])):
            assert L.kpo_draw(key, i) == int(d)
            assert L.kpo_unit(int(d)) == float.fromhex(u)


@pytest.mark.parametrize("model_name", ["di6", "dubins6", "quad12"])
def test_batch_matches_reference_golden(orc, model_name):
    """The reference's own test_batch_parity (tests/test_backends.py:37-54), oracle vs its recorded Batch."""
    g = np.load(os.path.join(GOLDEN, f"batch_{model_name}.npz"))
    mid = {"di6": 0, "dubins6": 1, "quad12": 2}[model_name]
    n = g["states"].shape[1]
    nu = g["control"].shape[1]
    lo = {0: [-2.0] * 3, 1: [-1, -1, -0.5], 2: [5, -0.05, -0.05, -0.05]}[mid]
    hi = {0: [2.0] * 3, 1: [1, 1, 0.5], 2: [15, 0.05, 0.05, 0.05]}[mid]
    ctx, keep = orc.make_ctx(mid, n, nu, lo, hi, float(g["t_prop"]), g["state_lo"], g["state_hi"], g["obs_min"],
                             g["obs_max"], float(g["check_res"]), g["grid_lo"], g["grid_width"], g["grid_cells"],
                             g["grid_strides"], int(g["subcells"]))
    out = orc.propagate_batch(ctx, g["states"], g["e_slots"], int(g["lam"]), int(g["seed"]), int(g["iteration"]))
    for f in ("valid", "region", "sub", "control", "dt", "accept_u", "end"):
        assert np.array_equal(out[f], g[f]), f
    # thread count must not matter (tests/test_backends.py:88)
    out4 = orc.propagate_batch(ctx, g["states"], g["e_slots"], int(g["lam"]), int(g["seed"]), int(g["iteration"]),
                               threads=4)
    for f in ("valid", "region", "sub", "end"):
        assert np.array_equal(out4[f], out[f])


def _oracle_for(kp, orc, model_name, scene, t_e, seed):
    model = kp.get_model(model_name)
    env = kp.gen_environment(scene, model, seed=0)
    prob = kp.build_problem(small_cfg(kp, model, t_e=t_e, seed=seed), env, model)
    return orc.plan_from_problem(prob), prob


def test_whole_plans_match_reference_digests(kp, orc):
    """Every iteration of six complete plans: trace counters and sha256 of tree / counters / estimates."""
    cases = json.load(open(os.path.join(GOLDEN, "plans.json")))
    for case in cases:
        op, _ = _oracle_for(kp, orc, case["model"], case["scene"], case["t_e"], case["seed"])
        for rec in case["iterations"]:
            op.step()
            tr = op.trace()
            for k in ("iteration", "branching", "ve_size", "vo_size", "attempted", "valid", "staged", "appended",
                      "tree_size"):
                assert tr[k] == rec[k], (case["model"], rec["iteration"], k)
            s, d = op.snapshot(), op.decomposition()
            assert _digest(s["states"], s["parent"], s["control"], s["dt"], s["tag"], s["region"]) == rec["tree"]
            assert _digest(d["n_valid"], d["n_invalid"], d["cov"], d["visited"], d["avail"]) == rec["counters"]
            assert _digest(d["free_vol"], d["score"], d["p_accept"]) == rec["estimates"]
        assert op.status == case["status"]
        if case["solution_slot"] is not None:
            assert int(op.raw.solution_slot) == case["solution_slot"]


def test_final_tree_fixture(kp, orc):
    g = np.load(os.path.join(GOLDEN, "tree_di6_forest_te6000_s1.npz"))
    op, _ = _oracle_for(kp, orc, "di6", "forest", 6000, 1)
    op.solve(t_max=60.0)
    s, d = op.snapshot(), op.decomposition()
    assert s["size"] == int(g["size"])
    for k in ("states", "parent", "control", "dt", "tag", "region"):
        assert np.array_equal(s[k], g[k]), k
    for k in ("p_accept", "n_valid", "n_invalid", "cov"):
        assert np.array_equal(d[k], g[k]), k


def test_checker_known_answers(kp, orc):
    """validity.py:108 restated in C: verdicts the reference checker gave on its own solutions."""
    for rec in json.load(open(os.path.join(GOLDEN, "checker.json"))):
        model = kp.get_model(rec["model"])
        env = kp.gen_environment(rec["scene"], model, seed=0)
        prob = kp.build_problem(small_cfg(kp, model, t_e=rec["t_e"], seed=rec["seed"]), env, model)
        ctx, keep = orc.ctx_from_problem(prob)
        for res, verdict in rec["valid"].items():
            ok, _ = orc.trajectory_valid(ctx, rec["seg_start"], rec["seg_control"], rec["seg_dt"], env.start,
                                         prob.goal4, float(res))
            assert ok == verdict
        # break the chain: a perturbed first control must be rejected (chain or goal)
        bad = np.array(rec["seg_control"])
        bad[0] = bad[0] * 0.5 + 0.1
        ok, code = orc.trajectory_valid(ctx, rec["seg_start"], bad, rec["seg_dt"], env.start, prob.goal4, 0.05)
        assert not ok and code in (2, 3, 4)
        # the product's host checker agrees with the reference's verdicts too
        segs = [kp.propagate_ode(model, x, u, dt) for x, u, dt in
                zip(rec["seg_start"], rec["seg_control"], rec["seg_dt"])]
        for res, verdict in rec["valid"].items():
            assert kp.ValidityChecker(env, model, float(res)).trajectory_valid(segs, start=env.start) == verdict


def _stacked_problem(kp, blocks, t_e, seed):
    model = kp.stacked_double_integrator(blocks)
    base = kp.gen_environment("forest", "di6", seed=0)
    start = np.tile(np.array([5.0, 5.0, 5.0, 0.0, 0.0, 0.0]), blocks)
    start[:3] = base.start[:3]
    env = kp.Environment(f"forest-{model.name}", base.workspace_lo, base.workspace_hi, base.obstacles_min,
                         base.obstacles_max, start, base.goal)
    return kp.build_problem(small_cfg(kp, model, t_e=t_e, seed=seed), env, model)


def test_stacked_integrators_match_reference_python_backend(kp, orc):
    """BASELINE.json config 4: oracle model id 3 (stacked 3-D double integrators, 12D and 24D) against what the
    reference's PYTHON backend produced for a custom DynamicsModel(kernel_id=None) -- SURVEY 8(d)'s oracle for
    this configuration (fixture: oracle/make_golden.py stacked).  Every iteration: the whole Batch, the tree, the
    counters and the estimates, bit for bit."""
    for case in json.load(open(os.path.join(GOLDEN, "plans_stacked.json"))):
        prob = _stacked_problem(kp, case["blocks"], case["t_e"], case["seed"])
        assert prob.cfg.cells_per_dim == case["cells"]
        op = orc.plan_from_problem(prob)
        for rec in case["iterations"]:
            op.step()
            tr = op.trace()
            for k in ("iteration", "branching", "ve_size", "vo_size", "attempted", "valid", "staged", "appended",
                      "tree_size"):
                assert tr[k] == rec[k], (case["blocks"], rec["iteration"], k)
            b = op.last_batch()
            assert _digest(b["valid"], b["region"], b["sub"], b["end"], b["control"], b["dt"], b["accept_u"]) == rec["batch"]
            s, d = op.snapshot(), op.decomposition()
            assert _digest(s["states"], s["parent"], s["control"], s["dt"], s["tag"], s["region"]) == rec["tree"]
            assert _digest(d["n_valid"], d["n_invalid"], d["cov"], d["visited"], d["avail"]) == rec["counters"]
            assert _digest(d["free_vol"], d["score"], d["p_accept"]) == rec["estimates"]


def test_step_given_equals_step(kp, orc):
    """The bookkeeping-only entry point (kpo_plan_step_given: passes 1b/2/3 on a supplied Batch) reproduces the full
    step when it is handed the full step's own Batch -- with and without the supplied goal flags -- and refuses a
    Batch of the wrong length."""
    for model_name, scene, t_e, seed in (("di6", "forest", 6000, 1), ("quad12", "narrow", 8000, 3)):
        a, prob = _oracle_for(kp, orc, model_name, scene, t_e, seed)
        b, _ = _oracle_for(kp, orc, model_name, scene, t_e, seed)
        c, _ = _oracle_for(kp, orc, model_name, scene, t_e, seed)
        goal = np.asarray(prob.goal4)
        with pytest.raises(ValueError):
            b.step_given(np.zeros(3, np.uint8), np.zeros(3, np.int64), np.zeros(3, np.int64), np.zeros((3, prob.model.n)))
        assert int(b.raw.iteration) == 0
        for it in range(60):
            st = a.step()
            ba = a.last_batch()
            hit = (np.sqrt(((ba["end"][:, :3] - goal[:3]) ** 2).sum(axis=1)) <= goal[3]).astype(np.uint8)
            assert b.step_given(ba["valid"], ba["region"], ba["sub"], ba["end"]) == st
            assert c.step_given(ba["valid"], ba["region"], ba["sub"], ba["end"], goal_hit=hit) == st
            for o in (b, c):
                sa, so = a.snapshot(), o.snapshot()
                assert sa["size"] == so["size"]
                for k in ("states", "parent", "control", "dt", "tag", "region"):
                    assert np.array_equal(sa[k], so[k]), (it, k)
                da, do = a.decomposition(), o.decomposition()
                for k in da:
                    assert np.array_equal(da[k], do[k]), (it, k)
                assert np.array_equal(a.last_batch()["staged_idx"], o.last_batch()["staged_idx"])
                assert a.trace() == o.trace()
            if st != 4:
                break
        assert a.status == b.status == c.status and a.status in ("solved", "capacity_exhausted")


def test_oracle_adaptive_capacity_rule(kp, orc):
    """kpo_plan_set_capacity (the paper's Remark 1, an extension): with growth 1 or the whole allocation in effect the
    plan is the reference's; with a small start it carries on past the point where the fixed-capacity plan ends
    exhausted, and its first iterations are the fixed-capacity plan's."""
    fixed, _ = _oracle_for(kp, orc, "di6", "forest", 1500, 3)
    same, _ = _oracle_for(kp, orc, "di6", "forest", 1500, 3)
    same.set_capacity(1500, 2.0)                                   # nothing to grow into
    grow, _ = _oracle_for(kp, orc, "di6", "forest", 12000, 3)
    grow.set_capacity(1500, 2.0)
    with pytest.raises(ValueError):
        grow.set_capacity(20000, 2.0)
    diverged = False
    for it in range(100):
        sf = fixed.step()
        assert same.step() == sf
        grow.step()
        if sf == 4:
            a, b = fixed.snapshot(), grow.snapshot()
            assert a["size"] == b["size"] and np.array_equal(a["tag"], b["tag"]) and np.array_equal(a["states"], b["states"])
        else:
            diverged = True
            break
    assert diverged and fixed.status == "capacity_exhausted" and same.status == "capacity_exhausted"
    assert grow.status == "running" and int(grow.raw.t_e) == 3000 and int(grow.raw.growths) == 1
    grow.solve(t_max=60.0)
    assert grow.status == "solved" and int(grow.raw.size) > 1500
    with pytest.raises(ValueError):
        grow.set_capacity(1500, 2.0)                               # only before the first iteration


def test_outcome_fixtures_are_consistent():
    """Full-size reference outcomes (100 seeds per config) that the GPU success-rate test compares against."""
    for name, min_solved in (("di6_forest", 100), ("dubins6_building", 100), ("quad12_narrow", 50),
                             ("quad12_forest", 100)):
        d = json.load(open(os.path.join(GOLDEN, f"outcomes_{name}.json")))
        assert d["seeds"] == 100 and len(d["records"]) == 100
        assert d["solved"] >= min_solved
        assert d["reval_res_fail"] == 0          # at the planning resolution every reference solution re-validates


# ---------------------------------------------------------------- live reference (build container only)

def _reference():
    import ref_loader
    if not ref_loader.reference_available():
        pytest.skip("reference tree not mounted")
    return ref_loader.load_reference()


@pytest.mark.reference
@pytest.mark.parametrize("model_name,scene,t_e,seed", [("di6", "forest", 4000, 7), ("dubins6", "narrow", 3000, 8),
                                                       ("quad12", "building", 5000, 9)])
def test_step_by_step_against_live_reference(kp, orc, model_name, scene, t_e, seed):
    K = _reference()
    from kinopax.planner import TAG_EXPAND, KinoPax
    op, _ = _oracle_for(kp, orc, model_name, scene, t_e, seed)
    rm = K.get_model(model_name)
    eng = KinoPax(K.PlannerConfig(t_e=t_e, t_prop=rm.default_t_prop, cells_per_dim=rm.default_cells_per_dim,
                                  seed=seed), K.gen_environment(scene, rm, seed=0), rm)
    for _ in range(40):
        eng.iteration += 1
        ve = len(eng.arena.slots_with_tag(TAG_EXPAND))
        lam = K.compute_branching_factor(t_e, eng.arena.size, ve, 32)
        staged = eng.propagate_pass(lam)
        eng.update_estimates_pass()
        slot, exhausted, _ = eng.update_node_sets_pass(staged)
        op.step()
        a, b = eng.arena.snapshot(), op.snapshot()
        assert a["size"] == b["size"]
        for k in ("states", "parent", "control", "dt", "tag", "region"):
            assert np.array_equal(a[k], b[k]), k
        d = op.decomposition()
        for k, v in (("n_valid", eng.decomp.n_valid), ("n_invalid", eng.decomp.n_invalid), ("cov", eng.decomp.cov),
                     ("visited", eng.decomp.visited), ("score", eng.decomp.score), ("p_accept", eng.decomp.p_accept)):
            assert np.array_equal(d[k], v), k
        if slot is not None or exhausted:
            break


@pytest.mark.reference
def test_stacked_integrators_against_live_reference_python_backend(kp, orc):
    """Live form of the config-4 pin: the reference's Python backend (custom DynamicsModel, kernel_id=None) and the
    oracle's model id 3 stepped side by side at 12D (full-state grid, cells 3) and 24D (cells 1)."""
    K = _reference()
    import make_golden
    from kinopax.planner import TAG_EXPAND, KinoPax
    for blocks, t_e, seed, n_iter in ((2, 500, 11, 5), (4, 400, 12, 4)):
        rm = make_golden.stacked_reference_model(K, blocks)
        eng = KinoPax(K.PlannerConfig(t_e=t_e, t_prop=rm.default_t_prop, cells_per_dim=rm.default_cells_per_dim, seed=seed),
                      make_golden.stacked_reference_env(K, rm), rm)
        assert eng.backend.name == "python"
        op = orc.plan_from_problem(_stacked_problem(kp, blocks, t_e, seed))
        for _ in range(n_iter):
            eng.iteration += 1
            ve = len(eng.arena.slots_with_tag(TAG_EXPAND))
            staged = eng.propagate_pass(K.compute_branching_factor(t_e, eng.arena.size, ve, 32))
            eng.update_estimates_pass()
            slot, exhausted, _ = eng.update_node_sets_pass(staged)
            op.step()
            a, b = eng.arena.snapshot(), op.snapshot()
            assert a["size"] == b["size"]
            for k in ("states", "parent", "control", "dt", "tag", "region"):
                assert np.array_equal(a[k], b[k]), k
            d = op.decomposition()
            for k, v in (("n_valid", eng.decomp.n_valid), ("n_invalid", eng.decomp.n_invalid), ("cov", eng.decomp.cov),
                         ("visited", eng.decomp.visited), ("score", eng.decomp.score), ("p_accept", eng.decomp.p_accept)):
                assert np.array_equal(d[k], v), k
            if slot is not None or exhausted:
                break


@pytest.mark.reference
def test_host_modules_against_live_reference(kp):
    K = _reference()
    rng = np.random.default_rng(3)
    for kind in ("forest", "narrow", "building"):
        for m in ("di6", "dubins6", "quad12"):
            a, b = kp.gen_environment(kind, m, 3), K.gen_environment(kind, m, 3)
            assert np.array_equal(a.obstacles_min, b.obstacles_min) and np.array_equal(a.obstacles_max, b.obstacles_max)
            assert np.array_equal(a.start, b.start) and a.name == b.name
    for m in ("di6", "dubins6", "quad12"):
        mm, rm = kp.get_model(m), K.get_model(m)
        for _ in range(10):
            x = rng.normal(size=mm.n) * 0.3
            u = rng.uniform(mm.control_lo, mm.control_hi)
            dt = float(rng.uniform(0.01, 1))
            assert np.array_equal(kp.propagate_ode(mm, x, u, dt).sampled_states, K.propagate_ode(rm, x, u, dt).sampled_states)
