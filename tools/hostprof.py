#!/usr/bin/env python3
"""Where the host time of KinoPax.solve goes (single query, whole GPU): C call vs trajectory rebuild vs rest."""
import sys, os, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_06807_b200 as kp
model = kp.get_model("di6"); env = kp.gen_environment("forest", model, seed=0)
cfg = kp.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=0, t_max=60.0)
eng = kp.KinoPax(cfg, env, model, backend="cuda-f32")
for w in range(3):
    eng.reset(seed=1000 + w); eng.solve()
t_reset, t_run, t_traj, t_total, dev = [], [], [], [], []
for seed in range(100):
    a = time.perf_counter(); eng.reset(seed=seed); b = time.perf_counter()
    st = eng._run(cfg.t_max); c = time.perf_counter()
    segs, ok = eng._trajectory(); d = time.perf_counter()
    t_reset.append(b - a); t_run.append(c - b); t_traj.append(d - c); dev.append(st.device_ms)
    a = time.perf_counter(); eng.reset(seed=seed); r = eng.solve(); t_total.append(time.perf_counter() - a)
us = lambda x: 1e6 * statistics.median(x)
print(f"median us: reset {us(t_reset):.1f}  _run {us(t_run):.1f} (device {1e3*statistics.median(dev):.1f})  _trajectory {us(t_traj):.1f}  reset+solve {us(t_total):.1f}")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for seed in range(50):
    eng.reset(seed=seed); eng.solve()
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
