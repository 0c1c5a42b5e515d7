#!/usr/bin/env python3
"""float32 vs float64 end states of the extensions of a large batch (the float64 kernel is pinned bit for bit
to the reference): max / p99.9 relative error over the items valid in both, verdict and cell agreement.

    [KPX_LIB_PATH=.../libkpx_<variant>.so] python tools/f32_err.py [scene] [lam] [model]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2409_06807_b200 as kp
from paper_2409_06807_b200.backend import PlanContext

scene = sys.argv[1] if len(sys.argv) > 1 else "narrow"
lam = int(sys.argv[2]) if len(sys.argv) > 2 else 8
model_name = sys.argv[3] if len(sys.argv) > 3 else "quad12"
model = kp.get_model(model_name)
env = kp.gen_environment(scene, model, seed=0)
cfg = kp.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=3)
prob = kp.build_problem(cfg, env, model)
with kp.KinoPax(cfg, env, model, backend="cuda") as eng:
    snap = eng.solve(capture_tree=True).tree_snapshot
size = int(snap["size"])
states = np.ascontiguousarray(snap["states"][:size], dtype=np.float64)
m = min(size, 125_000)
e_slots = np.sort(np.random.default_rng(0).choice(size, size=m, replace=False)).astype(np.int64)
g, ck = prob.grid, prob.checker
ctx = PlanContext(model=model, seed=11, t_prop=cfg.t_prop, state_lo=ck.state_lo, state_hi=ck.state_hi,
                  obs_min=env.obstacles_min, obs_max=env.obstacles_max, check_res=prob.check_resolution,
                  grid_lo=g.lo, grid_width=g.widths, grid_cells=g.cells, grid_strides=g.strides,
                  subcells=cfg.subcells_per_dim)
r = kp.get_backend("cuda").propagate_batch(ctx, states, e_slots, lam, 5)
b = kp.get_backend("cuda-f32").propagate_batch(ctx, states, e_slots, lam, 5)
keep = (b.valid == 1) & (r.valid == 1)
d = np.abs(b.end - r.end)
for w in model.wrap_dims:
    d[:, w] = np.minimum(d[:, w], np.abs(2 * np.pi - d[:, w]))
rel = (d / np.maximum(np.abs(r.end), 1.0))[keep]
per_item = rel.max(axis=1)
print(f"lib {os.environ.get('KPX_LIB_PATH', 'libkpx.so')}: {model_name}/{scene}, {m * lam} extensions of {m} tree nodes, "
      f"{int(keep.sum())} valid in both")
print(f"  relative end-state error (float32 vs float64): max {per_item.max():.3e}  p99.9 {np.quantile(per_item, 0.999):.3e}  "
      f"median {np.median(per_item):.3e}; worst component {int(np.unravel_index(rel.argmax(), rel.shape)[1])}")
print(f"  verdicts agree {np.mean(b.valid == r.valid):.6f} ({int(np.sum(b.valid != r.valid))} flips); "
      f"cells agree (valid in both) {np.mean(b.region[keep] == r.region[keep]):.6f}; "
      f"sub-cells {np.mean(b.sub[keep] == r.sub[keep]):.6f}")
