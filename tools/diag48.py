#!/usr/bin/env python3
"""Per-iteration phase times of one stacked-integrator query on a single CTA (team_ctas=1) and on the whole GPU."""
import sys, os, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp
import bench
from paper_2409_06807_b200 import core, envgen, dynamics

name = sys.argv[1] if len(sys.argv) > 1 else "di48g6"
model = bench.get_workload_model(dynamics, name)
env = bench.make_env(envgen, core, model, "forest")
cfg = kp.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=0, t_max=60.0)
for team in (0, 1):
    eng = kp.KinoPax(cfg, env, model, backend="cuda-f32", team_ctas=team)
    eng.reset(seed=1); res = eng.solve()
    eng.reset(seed=0); res = eng.solve()
    d = res.device
    print(f"team={team}: {res.status.value} iters={res.stats.iterations} tree={res.stats.tree_size} device={d['device_ms']:.3f} ms items={d['items']} substeps={d['substeps']}")
    for tr in eng.traces():
        print(f"   it {tr.iteration:2d} lam {tr.branching:2d} items {tr.attempted:7d} valid {tr.valid:7d} app {tr.appended:6d} "
              f"[S0 {1e3*tr.phase_ms[0]:.0f} S1 {1e3*tr.phase_ms[1]:.0f} S2 {1e3*tr.phase_ms[2]:.0f} S3 {1e3*tr.phase_ms[3]:.0f} S4 {1e3*tr.phase_ms[4]:.0f} epi {1e3*tr.phase_ms[5]:.0f} us]")
    eng.close()
