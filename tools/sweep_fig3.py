#!/usr/bin/env python3
"""The paper's Fig. 3 (failures and runtime against the tree capacity t_e, 12D quadcopter, Trees,
50 queries per capacity) with the runner's sweep_te -- one batch launch per capacity, float32 and float64 kernels.

    python tools/sweep_fig3.py [out_dir] [trials]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_06807_b200 as kp

out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fig3"
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 50
model = kp.get_model("quad12")
env = kp.gen_environment("forest", model, seed=0)
cfg = kp.PlannerConfig(t_e=100_000, lambda_max=32, t_prop=model.default_t_prop, epsilon=0.005, delta=1.0,
                       cells_per_dim=model.default_cells_per_dim, subcells_per_dim=4, t_max=60.0, seed=0)
tes = [50_000, 100_000, 150_000, 200_000, 280_000, 400_000, 600_000, 1_000_000]
for backend in ("cuda-f32", "cuda"):
    rows = kp.sweep_te(cfg, env, model, tes, trials, backend=backend, out_dir=os.path.join(out_dir, backend), quiet=False)
    for r in rows:
        r["backend"] = backend
    with open(os.path.join(out_dir, f"sweep_te_quad12_forest_{backend}.jsonl"), "w") as fh:
        for r in rows:
            fh.write(json.dumps(r, sort_keys=True) + "\n")
