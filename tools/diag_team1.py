import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import diag
diag.run("di6", "forest", "cuda-f32", seeds=(0,), team=1)
diag.run("quad12", "narrow", "cuda-f32", seeds=(0,), team=1)
diag.run("dubins6", "building", "cuda-f32", seeds=(0,), team=1)
