import os, sys, torch, json
sys.path.insert(0, os.getcwd())
from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig
ws = W.box_box(65536); s1, s2 = (api.surface_from_spec(b) for b in ws.bodies); p1, p2 = ws.poses(65536)
out = api.generate_manifold_batch(s1, s2, torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda"), SmoothingConfig())
comp = {}
for _ in range(5): api.compact_contacts(out["contacts"], 0.01, out=comp)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): api.compact_contacts(out["contacts"], 0.01, out=comp)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 50
print(json.dumps({"staged": os.environ.get("CMGB_COMPACT_STAGED", "0"), "ms": ms, "gbs": 65536*304*32/ms/1e6, "kept": int(comp["total"].item())}))
