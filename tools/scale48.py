#!/usr/bin/env python3
"""Concurrency scaling of one-CTA teams: kernel time of a batch of T queries on T teams, T = 1, 2, 8, ..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp
import bench
from paper_2409_06807_b200 import core, envgen, dynamics
name = sys.argv[1] if len(sys.argv) > 1 else "di48g6"
model = bench.get_workload_model(dynamics, name)
env = bench.make_env(envgen, core, model, "forest")
cfg = kp.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=0, t_max=60.0)
for teams in [int(x) for x in (sys.argv[2:] or ["1", "2", "8", "32", "148"])]:
    with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", n_teams=teams, team_ctas=1) as bp:
        r = bp.run(np.arange(teams), want_chains=False)
        r = bp.run(np.arange(teams), want_chains=False)
        print(f"{name} teams {teams:4d}: kernel_ms {r.kernel_ms:9.1f}  per-query device_ms median {np.median(r.records['device_ms']):9.1f}  solved {int(r.solved.sum())}", flush=True)
