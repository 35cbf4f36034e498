"""Developer probe: per-bucket time of config C (mixed primitives)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
for kind in W.MIXED_KINDS:
    ws = W.mixed_bucket(kind, n)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n)
    P1, P2 = torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda")
    out = {}
    for _ in range(3):
        api.generate_manifold_batch(s1, s2, P1, P2, SmoothingConfig(), out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); api.generate_manifold_batch(s1, s2, P1, P2, SmoothingConfig(), out=out); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    L = api.layout(s1, s2, SmoothingConfig())
    print(f"{kind:14s} {np.median(ts):.3f} ms  {n/np.median(ts)/1e3:.2f} M/s  kinds {s1.info.get('n_nodes')} layout {L}")
