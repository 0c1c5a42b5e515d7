#!/usr/bin/env python3
"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): a one-CTA-team batch, a multi-CTA
team, the validation kernel and the kernel seam, all at a few thousand nodes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp
which = sys.argv[1] if len(sys.argv) > 1 else "di6"
scene = {"di6": "forest", "dubins6": "building", "quad12": "narrow"}[which]
model = kp.get_model(which)
env = kp.gen_environment(scene, model, seed=0)
cfg = kp.PlannerConfig(t_e=6000, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=0, t_max=60.0)
with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", n_teams=3, team_ctas=1) as bp:
    r = bp.run(np.arange(6))
    print("batch f32:", int(r.solved.sum()), "solved", int(r.validated.sum()), "validated")
with kp.BatchPlanner(cfg, env, model, backend="cuda", n_teams=2, team_ctas=2) as bp:
    r = bp.run(np.arange(3))
    print("batch f64, teams of 2 CTAs:", int(r.solved.sum()), "solved")
with kp.KinoPax(cfg, env, model, backend="cuda-f32", team_ctas=4) as eng:
    res = eng.solve()
    print("solo f32, 4 CTAs:", res.status.value, res.stats.iterations, res.stats.tree_size)
# round 2: per-query scenes, adaptive capacity, the Philox kernels, the packed chain download and the goal sampler
if which == "di6":
    with kp.BatchPlanner(cfg, env, model, backend="cuda-f32-philox", n_teams=3, team_ctas=1, t_e_max=12000) as bp:
        bp.set_scenes([env, kp.gen_environment(scene, model, seed=1)])
        r = bp.run(np.arange(6), scenes=np.arange(6) % 2)
        print("batch f32 philox, 2 scenes, adaptive capacity:", int(r.solved.sum()), "solved", int(r.validated.sum()), "validated")
    with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", n_teams=6, team_ctas=1) as bp:      # hand-off to teams of 8 / 64 CTAs
        r = bp.run(np.arange(20))
        print("batch f32 with hand-off:", int(r.solved.sum()), "solved", int(r.validated.sum()), "validated, handed on", bp.handoff_counts())
    g = kp.goals_for_queries(np.arange(40), env)
    print("goal sampler:", g.shape)
