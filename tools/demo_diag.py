"""Developer probe: run the batched demo integrator and report the first
non-finite env / step (python tools/demo_diag.py [n_env] [steps])."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import PenaltyParams, SmoothingConfig

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 600
sc = W.demo_scene(n)
bodies = [api.surface_from_spec(b) for b in sc.bodies]
P0 = sc.poses(n)
b = api.DemoBatch(bodies, np.ones(len(bodies)), is_static=sc.is_static(), cfg=SmoothingConfig(),
                  params=PenaltyParams(), poses=P0, n_env=n)
for s in range(steps):
    prev = b.poses.clone(), b.velocities.clone()
    b.step(1e-3)
    ok = b.ok.cpu().numpy()
    if (ok == 0).any():
        bad = np.flatnonzero(ok == 0)
        e = int(bad[0])
        print(f"step {s}: {len(bad)} envs non-finite, first env {e}")
        print("prev poses", prev[0][e].cpu().numpy())
        print("prev vels", prev[1][e].cpu().numpy())
        print("init pose", P0[e])
        break
    if s % 100 == 0:
        v = b.velocities.cpu().numpy()
        print(s, "max |v|", np.abs(v).max(), "deepest min", b.deepest.min().item())
torch.cuda.synchronize()
print("done")
