import sys, os, json, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2409_06807_b200 as kp
for name, model_name, scene in (("di6_forest","di6","forest"),("dubins6_building","dubins6","building"),("quad12_narrow","quad12","narrow"),("quad12_forest","quad12","forest")):
    gold = json.load(open(f"/root/repo/tests/golden/outcomes_{name}.json")); recs = sorted(gold["records"], key=lambda r: r["seed"])
    seeds = np.array([r["seed"] for r in recs]); model = kp.get_model(model_name); env = kp.gen_environment(scene, model, seed=0)
    cfg = kp.PlannerConfig(t_e=model.default_t_e, lambda_max=32, t_prop=model.default_t_prop, epsilon=0.005, delta=1.0, cells_per_dim=model.default_cells_per_dim, subcells_per_dim=4, t_max=60.0, seed=0)
    with kp.BatchPlanner(cfg, env, model, backend="cuda", team_ctas=1) as bp: res = bp.run(seeds)
    same = sum(res.status(i).value == r["status"] and int(res.records["iterations"][i]) == r["iterations"] and int(res.records["tree_size"][i]) == r["tree_size"] for i, r in enumerate(recs))
    with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", team_ctas=1) as bp: r32 = bp.run(seeds)
    print(name, "f64 identical to reference:", same, "/", len(recs), "| solved ref", sum(r["status"]=="solved" for r in recs), "f64", int(res.solved.sum()), "f32", int(r32.solved.sum()), "replanned", None if r32.replanned is None else len(r32.replanned))
