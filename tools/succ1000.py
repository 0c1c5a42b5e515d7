import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2409_06807_b200 as kp
model = kp.get_model("quad12"); env = kp.gen_environment("narrow", model, seed=0)
cfg = kp.PlannerConfig(t_e=model.default_t_e, lambda_max=32, t_prop=model.default_t_prop, epsilon=0.005, delta=1.0, cells_per_dim=3, subcells_per_dim=4, t_max=60.0, seed=0)
for backend in ("cuda-f32", "cuda"):
    with kp.BatchPlanner(cfg, env, model, backend=backend, team_ctas=1) as bp:
        r = bp.run(np.arange(1000), want_chains=False)
    print(backend, "solved", int(r.solved.sum()), "of 1000; first 100:", int(r.solved[:100].sum()))
