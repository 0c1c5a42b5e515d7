#!/usr/bin/env python3
"""Short workloads for ncu: `batch` = one persistent multi-query launch, `solo` = single-query launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp

mode = sys.argv[1] if len(sys.argv) > 1 else "batch"
model_name = sys.argv[2] if len(sys.argv) > 2 else "di6"
scene = sys.argv[3] if len(sys.argv) > 3 else "forest"
backend = sys.argv[4] if len(sys.argv) > 4 else "cuda-f32"
nq = int(sys.argv[5]) if len(sys.argv) > 5 else 296
model = kp.get_model(model_name)
env = kp.gen_environment(scene, model, seed=0)
cfg = kp.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim)
if mode == "batch":
    with kp.BatchPlanner(cfg, env, model, backend=backend, team_ctas=1) as bp:
        for rep in range(2):
            r = bp.run(np.arange(nq), want_chains=False)
            print("batch", rep, "kernel_ms", r.kernel_ms, "solved", int(r.solved.sum()))
else:
    with kp.KinoPax(cfg, env, model, backend=backend) as eng:
        for seed in range(3):
            eng.reset(seed=seed)
            res = eng.solve()
            print("solo", seed, res.status.value, res.device["device_ms"])
