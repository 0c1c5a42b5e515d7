import sys, os, json, time
sys.path.insert(0, '/root/repo')
import bench, paper_2409_06807_b200 as kp
from paper_2409_06807_b200 import core, envgen, dynamics
model = kp.get_model("di6"); env = kp.gen_environment("forest", model, seed=0)
cfg = bench._cfg(kp, model)
print(json.dumps({k: v for k, v in bench.kernel_seam(kp, cfg, env, model, 0).items() if "items_per_s" in k or "parity" in k}, indent=1))
