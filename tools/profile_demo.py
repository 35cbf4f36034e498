"""One warm demo step for ncu capture of the penalty / integrate kernels (developer tool)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
sc = W.demo_scene(n)
bodies = [api.surface_from_spec(b) for b in sc.bodies]
d = api.DemoBatch(bodies, np.ones(len(bodies)), is_static=sc.is_static(), poses=sc.poses(n), n_env=n)
d.step(1e-3, 3)
torch.cuda.synchronize()
print("ok")
