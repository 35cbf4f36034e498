"""One warm launch of a kernel for ncu capture (python tools/profile_run.py manifold|compact|mixed:<bucket>|drop|drop-fwd|ee|vf [n])."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.scene import SmoothingConfig
from paper_2602_20304_b200 import workloads as W

kind = sys.argv[1] if len(sys.argv) > 1 else "manifold"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
if kind.startswith("mixed:"):
    ws = W.mixed_bucket(kind.split(":", 1)[1], n)
    s1 = api.surface_from_spec(ws.bodies[0]); s2 = api.surface_from_spec(ws.bodies[1])
    p1, p2 = ws.poses(n)
    P1 = torch.as_tensor(p1, device="cuda"); P2 = torch.as_tensor(p2, device="cuda")
    out = {}
    for _ in range(3):
        api.generate_manifold_batch(s1, s2, P1, P2, SmoothingConfig(), out=out)
elif kind in ("drop", "drop-fwd"):
    sc = W.drop_scene(n)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    P = torch.as_tensor(sc.poses(n), device="cuda")
    fn = api.generate_manifold_scene_jvp_batch if kind == "drop" else api.generate_manifold_scene_batch
    outs = None
    for _ in range(2):
        outs = fn(bodies, P, SmoothingConfig(), is_static=sc.is_static(), outs=outs)
elif kind in ("manifold", "compact", "compact-masked"):
    ws = W.box_box(n)
    s1 = api.surface_from_spec(ws.bodies[0]); s2 = api.surface_from_spec(ws.bodies[1])
    p1, p2 = ws.poses(n)
    P1 = torch.as_tensor(p1, device="cuda"); P2 = torch.as_tensor(p2, device="cuda")
    out = {}
    comp = {}
    thr = 0.01 if kind == "compact-masked" else None
    for _ in range(3):
        api.generate_manifold_batch(s1, s2, P1, P2, SmoothingConfig(), out=out, active_threshold=thr)
        if kind == "compact":
            api.compact_contacts(out["contacts"], 0.01, out=comp)
        elif kind == "compact-masked":
            api.compact_contacts(out["contacts"], mask=out["active_mask"], count=out["active_count"], out=comp)
else:
    pairs = torch.rand((n, 12), dtype=torch.float64, device="cuda")
    for _ in range(3):
        (api.run_ee_batch if kind == "ee" else api.run_vf_batch)(pairs, SmoothingConfig())
torch.cuda.synchronize()
print("ok")
