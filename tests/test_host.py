"""Host-side logic and the C-ABI surface (no GPU needed)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, make_empty_env, small_cfg


def test_rng_matches_reference_golden(kp):
    from paper_2409_06807_b200 import rng
    g = json.load(open(os.path.join(GOLDEN, "rng.json")))
    for m in g["mix64"]:
        assert rng.mix64(int(m["z"])) == int(m["mix"])
        assert int(rng.mix64_np(np.array([int(m["z"])], dtype=np.uint64))[0]) == int(m["mix"])
    for c in g["stream_cases"]:
        key = rng.stream_key(c["seed"], c["iteration"], c["slot"], c["ext"], c["phase"])
        assert key == int(c["key"])
        kn = rng.stream_keys_np(c["seed"], c["iteration"], np.array([c["slot"]]), np.array([c["ext"]]), c["phase"])
        assert int(kn[0]) == key
        for i, (d, u) in enumerate(zip(c["draws"], c["units"])):
            assert rng.draw_u64(key, i) == int(d)
            assert rng.u64_to_unit(int(d)) == float.fromhex(u)
            assert rng.uniforms_np(kn, i)[0] == float.fromhex(u)
    s = rng.RngStream(seed=11)
    xs = np.array([s.duration(1.0) for _ in range(2000)])
    assert np.all((xs > 0.0) & (xs <= 1.0))                       # never exactly zero (tests/test_rng.py:64)
    assert rng.stream_key(-1, 0, 0, 0, 1) == rng.stream_key((1 << 64) - 1, 0, 0, 0, 1)


def test_scenes_match_reference_golden(kp):
    g = json.load(open(os.path.join(GOLDEN, "scenes.json")))
    for key, rec in g.items():
        kind, model, seed = key.split("/")
        env = kp.gen_environment(kind, model, seed=int(seed))
        assert env.name == rec["name"]
        assert env.obstacles_min.tolist() == rec["obs_min"] and env.obstacles_max.tolist() == rec["obs_max"]
        assert env.start.tolist() == rec["start"]
        assert env.goal.center.tolist() + [env.goal.radius] == rec["goal"]
    with pytest.raises(kp.GenerationError):
        kp.gen_environment("swamp", "di6")


def test_config_validation(kp):
    di6 = kp.get_model("di6")
    assert kp.validate_config(kp.PlannerConfig(t_e=100), di6).region_count == 4096
    for bad in (dict(t_e=0), dict(t_e=10, epsilon=0.0), dict(t_e=10, epsilon=1.0), dict(t_e=10, delta=0.0),
                dict(t_e=10, t_prop=0.0), dict(t_e=10, lambda_max=0), dict(t_e=10, cells_per_dim=0)):
        with pytest.raises(kp.ConfigError):
            kp.validate_config(kp.PlannerConfig(**bad), di6)
    with pytest.raises(kp.ConfigError, match="exceeding the cap"):
        kp.validate_config(kp.PlannerConfig(t_e=10, cells_per_dim=4), kp.get_model("quad12"))
    assert kp.suggest_cells_per_dim(12) == 3 and kp.suggest_cells_per_dim(6) == 11
    assert kp.compute_branching_factor(100, 1, 1, 32) == 32        # Eq. 6 known answers (tests/test_planner.py:17-28)
    assert kp.compute_branching_factor(100, 90, 20, 32) == 1
    assert kp.compute_branching_factor(1000, 100, 100, 32) == 9


def test_environment_json_roundtrip(kp, tmp_path):
    env = kp.gen_environment("building", "quad12", seed=0)
    p = tmp_path / "env.json"
    kp.save_environment(env, p)
    back = kp.load_environment(p)
    assert np.array_equal(back.obstacles_min, env.obstacles_min) and np.array_equal(back.start, env.start)
    with pytest.raises(kp.EnvironmentIOError):
        kp.load_environment(tmp_path / "missing.json")
    p.write_text("{not json")
    with pytest.raises(kp.EnvironmentFormatError):
        kp.load_environment(p)
    doc = kp.environment_to_dict(env)
    doc["start"][0] = 5.0    # inside the wall
    doc["start"][1] = 7.0
    with pytest.raises(kp.EnvironmentFormatError):
        kp.environment_from_dict(doc)


def test_grid_geometry_known_answers(kp):
    """Mapping rules of decomposition.py:76-106 (C-order strides, clamping, centre -> sub 7 at subcells=2)."""
    g = kp.GridGeometry(np.array([0, 0, 0, -5, -5, -5.0]), np.array([10, 10, 10, 5, 5, 5.0]), 4, 4)
    assert g.strides.tolist() == [1024, 256, 64, 16, 4, 1] and g.n_regions == 4096
    assert g.region_index(np.array([1, 1, 1, 0, 0, 0.0])) == 0 * 1024 + 0 + 0 + 2 * 16 + 2 * 4 + 2
    assert g.region_index(np.array([10, 10, 10, 5, 5, 5.0])) == 4095           # upper boundary clamps into last cell
    assert g.region_index(np.array([-3, 0, 0, -9, 0, 0.0])) == g.region_index(np.array([0, 0, 0, -5, 0, 0.0]))
    g2 = kp.GridGeometry(np.zeros(6), np.full(6, 8.0), 2, 2)
    r, s = g2.map_states(np.array([[3.0, 3.0, 3.0, 0, 0, 0]]))
    assert r[0] == 0 and s[0] == 7 and g2.subregion_index(np.array([3.0, 3.0, 3.0, 0, 0, 0]), 0) == 7


def test_validity_checker_rules(kp):
    env = kp.gen_environment("narrow", "di6", seed=0)
    chk = kp.ValidityChecker(env, kp.get_model("di6"), 0.05)
    assert not chk.state_valid(np.array([4.75, 5, 5, 0, 0, 0.0]))            # touching a face collides (closed box)
    assert chk.state_valid(np.array([4.7499, 5, 5, 0, 0, 0.0]))
    assert not chk.state_valid(np.array([1, 1, 1, 5.0001, 0, 0]))            # velocity box
    assert chk.state_valid(np.array([0, 0, 0, 5.0, 0, 0]))                   # boundary is valid
    from paper_2409_06807_b200.validity import densify_steps
    assert [densify_steps(d, 0.05) for d in (0.0, 0.05, 0.051, 0.1, 0.11, 0.2001)] == [1, 1, 2, 2, 4, 8]
    assert kp.in_goal(np.array([8.5, 5, 5 - 1.25, 0, 0, 0.0]), env.goal)
    ball = kp.GoalBall(np.array([0.0, 0, 0]), 1.0)
    assert ball.contains(np.array([1.0, 0, 0])) and not ball.contains(np.array([1.0000001, 0, 0]))


def test_backend_registry_contract(kp, monkeypatch):
    """backend.py:103-122: explicit name -> env override -> default; unknown names raise ConfigError."""
    if not kp.cuda_available():
        pytest.skip("libkpx.so not built")
    assert kp.get_backend("cuda").name == "cuda" and kp.get_backend("cuda-f32").name == "cuda-f32"
    assert kp.get_backend(None, kp.get_model("di6")).name == "cuda"
    monkeypatch.setenv("KINOPAX_BACKEND", "cuda-f32")
    assert kp.get_backend(None).name == "cuda-f32"
    with pytest.raises(kp.ConfigError):
        kp.get_backend("python")            # no CPU backend exists in this package
    with pytest.raises(kp.ConfigError):
        kp.get_backend("no-such-backend")


def test_problem_flattening(kp):
    m = kp.get_model("quad12")
    env = kp.gen_environment("narrow", m, seed=0)
    prob = kp.build_problem(small_cfg(kp, m, t_e=1000), env, m)
    assert prob.grid.n_regions == 3 ** 12 and prob.grid.subs_per_region == 64
    assert prob.state_lo[:3].tolist() == [0, 0, 0] and prob.state_hi[6] == 1.0
    with pytest.raises(kp.ConfigError):                              # start inside an obstacle
        bad = kp.Environment(env.name, env.workspace_lo, env.workspace_hi, env.obstacles_min, env.obstacles_max,
                             np.array([5.0, 5, 5] + [0] * 9, dtype=float), env.goal)
        kp.build_problem(small_cfg(kp, m, t_e=1000), bad, m)
    s = kp.stacked_double_integrator(4)
    assert s.n == 24 and s.control_dim == 12 and s.kernel_id == 3 and s.default_cells_per_dim == 1


def test_c_abi_exports_every_declared_symbol(kp):
    """libkpx.so must load and export exactly what include/kpx.h declares (no compute calls here)."""
    from paper_2409_06807_b200 import _lib
    if not os.path.isfile(_lib.LIB_PATH):
        pytest.skip("libkpx.so not built")
    header = open(os.path.join(ROOT, "include", "kpx.h")).read()
    declared = set(re.findall(r"^(?:int|void|const char \*)\s*(kpx_[a-z_0-9]+)\(", header, flags=re.M))
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in kpx.h but not exported"
    assert declared == set(_lib.EXPORTED_SYMBOLS), declared ^ set(_lib.EXPORTED_SYMBOLS)
    assert _lib.load().kpx_version() >= 100
    # struct layouts agree with the compiled header (checked inside load(); sizes are part of the ABI)
    L = _lib.load()
    assert [L.kpx_struct_size(i) for i in range(4)] == [ctypes.sizeof(c) for c in
                                                        (_lib.Problem, _lib.Stats, _lib.Trace, _lib.QueryResult)]
    assert _lib.QUERY_RESULT_DTYPE.itemsize == ctypes.sizeof(_lib.QueryResult)


def test_product_does_not_import_oracle():
    """The oracle is a checker: nothing under the package may import or load it."""
    pkg = os.path.join(ROOT, "paper_2409_06807_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".inl")):
                text = open(os.path.join(dirpath, f)).read()
                assert "kpx_oracle" not in text and "import oracle" not in text and "ref_loader" not in text, f


def test_native_trajectory_rebuild_and_check(kp):
    """kpx_trajectory / kpx_trajectory_valid are host-only float64 code in libkpx.so: they must equal
    propagate_ode (dynamics.py:242) bit for bit and reproduce the reference checker's recorded verdicts."""
    import ctypes as C
    from paper_2409_06807_b200 import _lib
    if not os.path.isfile(_lib.LIB_PATH):
        pytest.skip("libkpx.so not built")
    L = _lib.load()
    for rec in json.load(open(os.path.join(GOLDEN, "checker.json"))):
        model = kp.get_model(rec["model"])
        env = kp.gen_environment(rec["scene"], model, seed=0)
        prob = kp.build_problem(small_cfg(kp, model, t_e=rec["t_e"], seed=rec["seed"]), env, model)
        starts, ctrl, dts = (np.ascontiguousarray(rec[k], dtype=np.float64) for k in ("seg_start", "seg_control", "seg_dt"))
        n_seg = len(dts)
        rows = int((np.maximum(4, np.ceil(dts / 0.02)) + 1).sum())
        sampled, off = np.empty((rows, model.n)), np.zeros(n_seg + 1, np.int64)
        for from_root in (0, 1):
            _lib.check(L.kpx_trajectory(model.kernel_id, model.n, model.control_dim, n_seg, _lib.ptr(starts),
                                        _lib.ptr(ctrl), _lib.ptr(dts), from_root, _lib.ptr(sampled), rows,
                                        _lib.ptr(off)), "kpx_trajectory")
            x = starts[0]
            for i in range(n_seg):
                seg = kp.propagate_ode(model, x if from_root else starts[i], ctrl[i], float(dts[i]))
                assert np.array_equal(sampled[off[i]:off[i + 1]], seg.sampled_states), (rec["model"], i)
                x = seg.end_state
        ps, keep = _lib.problem_from(prob)
        for res, verdict in rec["valid"].items():
            ok, code = C.c_int32(0), C.c_int32(0)
            _lib.check(L.kpx_trajectory_valid(C.byref(ps), n_seg, _lib.ptr(sampled), _lib.ptr(off),
                                              _lib.ptr(prob.goal4), float(res), C.byref(ok), C.byref(code)), "valid")
            assert bool(ok.value) == verdict
        far = prob.goal4.copy()
        far[:3] = 0.5
        ok, code = C.c_int32(0), C.c_int32(0)
        L.kpx_trajectory_valid(C.byref(ps), n_seg, _lib.ptr(sampled), _lib.ptr(off), _lib.ptr(far), 0.05,
                               C.byref(ok), C.byref(code))
        assert ok.value == 0 and code.value == 4


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_cull_thresholds_are_exact(kp, precision):
    """The compare-only densification (kpx_device.cuh, Params::d2_thr) against validity.py:26-31: for squared
    lengths at and next to every threshold, `steps` from the compares equals the reference's sqrt + doubling loop
    evaluated in the same arithmetic."""
    from paper_2409_06807_b200 import _lib
    L = _lib.load()
    model = kp.get_model("di6")
    env = kp.gen_environment("forest", model, seed=0)
    ft = np.float64 if precision == "f64" else np.float32
    for res in (0.05, 0.013, 0.2):
        prob, keep = _lib.problem_from(kp.build_problem(kp.PlannerConfig(t_e=1000, seed=0), env, model, res))
        thr = np.zeros(4)
        _lib.check(L.kpx_cull_thresholds(ctypes.byref(prob), _lib.F64 if precision == "f64" else _lib.F32,
                                         _lib.ptr(thr)), "kpx_cull_thresholds")
        thr = thr.astype(ft)
        assert np.all(np.diff(thr) > 0)

        def steps_ref(d2):                      # densify_steps in the arithmetic of `ft`
            dist, t, m = np.sqrt(ft(d2)), ft(res), 1
            while t < dist:
                t, m = ft(t + t), m * 2
            return m

        def steps_cmp(d2):
            return 1 + (d2 > thr[0]) + 2 * (d2 > thr[1]) + 4 * (d2 > thr[2])

        rng = np.random.default_rng(0)
        probes = [ft(x) for x in rng.uniform(0, float(thr[3]), 2000)]
        for k in range(4):
            t = thr[k]
            probes += [t, np.nextafter(t, ft(0)), np.nextafter(t, ft(np.inf)), np.nextafter(np.nextafter(t, ft(np.inf)), ft(np.inf))]
        for d2 in probes:
            if d2 <= thr[3]:
                assert steps_cmp(d2) == steps_ref(d2), (res, float(d2))
            else:
                assert steps_ref(d2) > 8, (res, float(d2))


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_cull_tables_are_conservative(kp, precision):
    """Occupancy tables of the segment cull: a point inside a closed obstacle box always finds that obstacle's
    bit in its cell's mask; the dilated table is the OR of the 2x2x2 block starting at the cell."""
    from paper_2409_06807_b200 import _lib
    L = _lib.load()
    ft = np.float64 if precision == "f64" else np.float32
    G = 16
    for scene, name in (("forest", "di6"), ("building", "dubins6"), ("narrow", "quad12")):
        model = kp.get_model(name)
        env = kp.gen_environment(scene, model, seed=0)
        prob, keep = _lib.problem_from(kp.build_problem(kp.PlannerConfig(t_e=1000, seed=0,
                                                                         cells_per_dim=model.default_cells_per_dim),
                                                        env, model))
        masks, lo, inv = np.zeros(2 * G ** 3, np.uint32), np.zeros(3), np.zeros(3)
        _lib.check(L.kpx_cull_tables(ctypes.byref(prob), _lib.F64 if precision == "f64" else _lib.F32,
                                     _lib.ptr(masks), _lib.ptr(lo), _lib.ptr(inv)), "kpx_cull_tables")
        occ, occ2 = masks[:G ** 3].reshape(G, G, G), masks[G ** 3:].reshape(G, G, G)
        pad = np.zeros((G + 1, G + 1, G + 1), np.uint32)
        pad[:G, :G, :G] = occ
        dil = np.zeros_like(occ)
        for dx in (0, 1):
            for dy in (0, 1):
                for dz in (0, 1):
                    dil |= pad[dx:dx + G, dy:dy + G, dz:dz + G]
        assert np.array_equal(dil, occ2)
        omin, omax = env.obstacles_min.astype(ft), env.obstacles_max.astype(ft)
        rng = np.random.default_rng(1)
        pts = rng.uniform(env.workspace_lo, env.workspace_hi, size=(20000, 3)).astype(ft)
        # add points on obstacle faces / corners: the boxes are closed
        pts = np.vstack([pts, omin, omax, (omin + omax) / ft(2)])
        cell = ((pts - lo.astype(ft)) * inv.astype(ft)).astype(np.int64).clip(0, G - 1)      # the kernel's occ_cell
        m = occ[cell[:, 0], cell[:, 1], cell[:, 2]]
        inside = np.all((pts[:, None, :] >= omin[None]) & (pts[:, None, :] <= omax[None]), axis=2)   # (P, K)
        for k in range(len(omin)):
            assert np.all((m[inside[:, k]] >> np.uint32(k)) & 1), (scene, k)
        assert inside.any()


# Random123 known-answer vectors for Philox4x32-10 (kat_vectors of the Random123 distribution): counter, key, output
PHILOX_KAT = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
              ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
              ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
               (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]


def test_philox_known_answers_host(kp):
    """The production generator against the published vectors: the Python twin (rng.philox4x32_10) and the C++ one
    compiled into libkpx.so (host half of kpx_philox4x32; the device half is checked under -m gpu)."""
    from paper_2409_06807_b200 import _lib, rng
    lib = _lib.load()
    for ctr, key, want in PHILOX_KAT:
        assert rng.philox4x32_10(ctr, key) == want
        c, k, out = np.array(ctr, np.uint32), np.array(key, np.uint32), np.zeros(4, np.uint32)
        _lib.check(lib.kpx_philox4x32(_lib.ptr(c), _lib.ptr(k), _lib.ptr(out), None), "kpx_philox4x32")
        assert tuple(int(x) for x in out) == want
    # streams: distinct identities give distinct draws, uniforms lie in [0, 1), durations in (0, t_prop]
    s = rng.PhiloxStream(7, iteration=3, slot=11, extension=2, phase=rng.PHASE_SAMPLE)
    draws = [s.next_u64() for _ in range(6)]
    assert len(set(draws)) == 6
    other = rng.PhiloxStream(7, iteration=3, slot=11, extension=3, phase=rng.PHASE_SAMPLE)
    assert other.next_u64() not in draws
    u = [rng.PhiloxStream(1, slot=i).uniform() for i in range(2000)]
    assert 0.0 <= min(u) and max(u) < 1.0 and abs(np.mean(u) - 0.5) < 0.03
    assert all(0.0 < rng.PhiloxStream(2, slot=i).duration(0.5) <= 0.5 for i in range(200))
    assert kp.get_backend("cuda-f32-philox").rng == _lib.RNG_PHILOX and kp.get_backend("cuda").rng == _lib.RNG_SPLITMIX64
