#!/usr/bin/env python3
"""quad12 / Narrow Passage (BASELINE.json configs[1]), seeds 0..99: the fixed capacity t_e = 400 000 (the reference solves
61 of these seeds, the rest end capacity_exhausted) against adaptive capacity starting at 400 000 (x2 up to 1.6 M) and
against fixed capacities at the grown sizes."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp

model = kp.get_model("quad12"); env = kp.gen_environment("narrow", model, seed=0)
def cfg(te): return kp.PlannerConfig(t_e=te, lambda_max=32, t_prop=model.default_t_prop, epsilon=0.005, delta=1.0,
                                     cells_per_dim=model.default_cells_per_dim, subcells_per_dim=4, t_max=60.0, seed=0)
seeds = np.arange(100)
out = []
for name, te, kw in (("fixed 400k", 400_000, {}), ("adaptive 400k -> 1.6M (x2)", 400_000, {"t_e_max": 1_600_000}),
                     ("fixed 800k", 800_000, {}), ("fixed 1.6M", 1_600_000, {})):
    for backend in ("cuda-f32", "cuda"):
        with kp.BatchPlanner(cfg(te), env, model, backend=backend, n_teams=100, team_ctas=1, **kw) as bp:
            t0 = time.perf_counter(); r = bp.run(seeds); dt = time.perf_counter() - t0
        caps = np.bincount(r.records["capacity"] // 100000)
        rec = {"case": name, "backend": backend, "solved": int(r.solved.sum()), "validated": int(r.validated.sum()),
               "median_device_ms_solved": float(np.median(r.records["device_ms"][r.solved])) if r.solved.any() else None,
               "capacity_histogram_x100k": {int(i): int(c) for i, c in enumerate(caps) if c}, "wall_s": dt}
        print(json.dumps(rec)); out.append(rec)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/adaptive_narrow.json", "w"), indent=1)
