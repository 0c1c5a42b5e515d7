#!/usr/bin/env python3
"""Hand-off of a batch's last queries (kpx_batch_set_handoff): how many were handed on, and the launch time with / without.
tools/handoff_probe.py [model scene queries]   (KPX_HANDOFF_WIDTHS=2,8,64 picks other stage widths)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp
name = sys.argv[1] if len(sys.argv) > 1 else "di6"
scene = sys.argv[2] if len(sys.argv) > 2 else "forest"
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 4736
model = kp.get_model(name)
env = kp.gen_environment(scene, model, seed=0)
cfg = kp.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, t_max=60.0)
for handoff in (False, True):
    with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", handoff=handoff) as bp:
        for rep in range(2):
            r = bp.run(np.arange(nq), want_chains=False)
        ms = r.records["device_ms"]
        print(f"{name}/{scene} {nq} queries on {bp.n_teams} teams, handoff={handoff} widths={os.environ.get('KPX_HANDOFF_WIDTHS', 'default')}: "
              f"kernel {r.kernel_ms:.1f} ms, handed on {bp.handoff_counts()}, solved {int(r.solved.sum())}, "
              f"query device ms median {np.median(ms):.2f} max {ms.max():.2f}")
