#!/usr/bin/env python3
"""Per-iteration timing breakdown of single-query plans (device trace), after warm-up."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp

def run(model_name, scene, backend, seeds=(0, 1, 2), t_e=None, team=0):
    model = kp.get_model(model_name)
    env = kp.gen_environment(scene, model, seed=0)
    cfg = kp.PlannerConfig(t_e=t_e or model.default_t_e, t_prop=model.default_t_prop,
                           cells_per_dim=model.default_cells_per_dim, seed=0, t_max=30.0)
    t0 = time.perf_counter()
    eng = kp.KinoPax(cfg, env, model, backend=backend, team_ctas=team)
    print(f"== {model_name}/{scene} {backend} team={team} create {1e3*(time.perf_counter()-t0):.1f} ms")
    for w in range(2):
        eng.reset(seed=1000 + w); eng.solve()
    for seed in seeds:
        eng.reset(seed=seed)
        res = eng.solve()
        d = res.device
        print(f" seed {seed}: {res.status.value} iters={res.stats.iterations} tree={res.stats.tree_size} "
              f"wall={res.stats.wall_time_ms:.3f} ms device={d['device_ms']:.3f} ms reset={d['reset_ms']:.3f} ms "
              f"items={d['items']} substeps={d['substeps']} points={d['points']}")
        if seed == seeds[0]:
            prev = 0.0
            for tr in eng.traces():
                print(f"   it {tr.iteration:2d} lam {tr.branching:2d} ve {tr.ve_size:6d} items {tr.attempted:7d} valid {tr.valid:7d} "
                      f"staged {tr.staged:6d} app {tr.appended:6d} tree {tr.tree_size:7d}  +{1e3*tr.elapsed_s-prev:.3f} ms  "
                      f"[S0 {1e3*tr.phase_ms[0]:.0f} S1 {1e3*tr.phase_ms[1]:.0f} S2 {1e3*tr.phase_ms[2]:.0f} "
                      f"S3 {1e3*tr.phase_ms[3]:.0f} S4 {1e3*tr.phase_ms[4]:.0f} epi {1e3*tr.phase_ms[5]:.0f} us]")
                prev = 1e3 * tr.elapsed_s
    eng.close()

if __name__ == "__main__":
    which = sys.argv[1:] or ["di6"]
    if "di6" in which:
        run("di6", "forest", "cuda-f32"); run("di6", "forest", "cuda")
    if "quad12" in which:
        run("quad12", "narrow", "cuda-f32", seeds=(0, 1)); run("quad12", "narrow", "cuda", seeds=(0,))
    if "dubins6" in which:
        run("dubins6", "building", "cuda-f32"); 
    if "team" in which:
        for team in (1, 4, 32):
            run("di6", "forest", "cuda-f32", seeds=(0,), team=team)
