import sys, os, time
sys.path.insert(0, os.getcwd())
import paper_2409_06807_b200 as kp
from paper_2409_06807_b200 import runner
for name, scene in (("di6", "forest"), ("quad12", "narrow")):
    model = kp.get_model(name); env = kp.gen_environment(scene, model, seed=0)
    cfg = kp.PlannerConfig(t_e=model.default_t_e, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=0, t_max=60.0)
    for tc in (1, 0):
        t0 = time.perf_counter()
        table, recs = runner.run_trials(cfg, env, model, n_trials=100, backend="cuda-f32", team_ctas=tc)
        print(name, "team_ctas", tc, "solved", table.solved, "median ms solved %.2f mean all %.2f" % (table.median_ms_solved, table.mean_ms_all), "reval failures", table.revalidation_failures, "wall %.2f s" % (time.perf_counter() - t0))
