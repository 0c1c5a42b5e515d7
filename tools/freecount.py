#!/usr/bin/env python3
"""Share of extensions the closed-form certificate finishes (FreeFlight), per workload: tools/freecount.py di6_forest ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp
import bench
from paper_2409_06807_b200 import core, dynamics, envgen
for wl in sys.argv[1:] or ["di6_forest"]:
    name, scene, _, _ = bench.WORKLOADS[wl]
    model = bench.get_workload_model(dynamics, name)
    env = bench.make_env(envgen, core, model, scene)
    cfg = bench._cfg(kp, model)
    with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", n_teams=64, team_ctas=1) as bp:
        r = bp.run(np.arange(64), want_chains=False).records
    with kp.KinoPax(cfg, env, model, backend="cuda-f32") as eng:
        eng.reset(seed=0); res = eng.solve()
    print("%s: batch free %.3f of %d items (valid share unknown here); solo seed 0 free %.3f, %d iterations, device %.3f ms" % (
        wl, r["free_items"].sum() / r["items"].sum(), r["items"].sum(), res.device["free_items"] / max(res.device["items"], 1),
        res.stats.iterations, res.device["device_ms"]))
