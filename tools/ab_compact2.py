"""Timing split of the fused compaction (developer tool): manifold step with
and without activity masks, and the masked compaction kernel alone."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.scene import SmoothingConfig
from paper_2602_20304_b200 import workloads as W

n = 65536
ws = W.box_box(n)
s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
p1, p2 = ws.poses(n)
P1 = torch.as_tensor(p1, device="cuda"); P2 = torch.as_tensor(p2, device="cuda")
cfg = SmoothingConfig()


def t(fn, k=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k): fn()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / k

o1, o2, comp = {}, {}, {}
plain = t(lambda: api.generate_manifold_batch(s1, s2, P1, P2, cfg, out=o1))
masked = t(lambda: api.generate_manifold_batch(s1, s2, P1, P2, cfg, out=o2, active_threshold=0.01))
gather = t(lambda: api.compact_contacts(o2["contacts"], mask=o2["active_mask"], count=o2["active_count"], out=comp))
scan = t(lambda: api.compact_contacts(o1["contacts"], 0.01, out=comp))
print(json.dumps({"manifold_ms": plain, "manifold_with_masks_ms": masked, "masked_compaction_ms": gather,
                  "standalone_compaction_ms": scan}))
