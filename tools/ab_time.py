"""A/B timing of the box-box manifold step (developer tool): back-to-back
launches between two CUDA events, median of 5 windows. Library chosen by
CMGB_LIBRARY (default: the in-tree build). python tools/ab_time.py [workload]"""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.scene import SmoothingConfig
from paper_2602_20304_b200 import workloads as W

wl = sys.argv[1] if len(sys.argv) > 1 else "box-box"
n = 65536
if wl == "box-box":
    ws = W.box_box(n)
elif wl.startswith("eps"):
    ws = W.box_box_eps(float(wl[3:]), n)
else:
    ws = W.mixed_bucket(wl, n)
s1 = api.surface_from_spec(ws.bodies[0]); s2 = api.surface_from_spec(ws.bodies[1])
p1, p2 = ws.poses(n)
P1 = torch.as_tensor(p1, device="cuda"); P2 = torch.as_tensor(p2, device="cuda")
out = {}
cfg = SmoothingConfig()
step = lambda: api.generate_manifold_batch(s1, s2, P1, P2, cfg, out=out)
for _ in range(5): step()
torch.cuda.synchronize()
ws_ms = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): step()
    b.record(); b.synchronize()
    ws_ms.append(a.elapsed_time(b) / 20)
ms = float(np.median(ws_ms))
print(json.dumps({"lib": os.path.basename(os.environ.get("CMGB_LIBRARY", "libcmgb.so")), "workload": wl, "ms": ms,
                  "Mps": n / ms / 1e3, "spread": [min(ws_ms), max(ws_ms)]}))
