#!/usr/bin/env python3
"""Small stacked-integrator batch for ncu: `prof48.py di48g6 148 20000`."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp
import bench
from paper_2409_06807_b200 import core, envgen, dynamics
name = sys.argv[1] if len(sys.argv) > 1 else "di48g6"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 148
t_e = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
model = bench.get_workload_model(dynamics, name)
env = bench.make_env(envgen, core, model, "forest")
cfg = kp.PlannerConfig(t_e=t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=0, t_max=60.0)
with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", team_ctas=1) as bp:
    for rep in range(2):
        r = bp.run(np.arange(nq), want_chains=False)
        print("batch", rep, "teams", bp.n_teams, "kernel_ms", r.kernel_ms, "solved", int(r.solved.sum()), "median iters", np.median(r.records["iterations"]))
