"""Developer timing probe (CUDA events) for the manifold and witness kernels."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.scene import SmoothingConfig
from paper_2602_20304_b200 import workloads as W

def time_fn(fn, reps=20, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
ws = W.box_box(n)
s1 = api.surface_from_spec(ws.bodies[0]); s2 = api.surface_from_spec(ws.bodies[1])
p1, p2 = ws.poses(n)
P1 = torch.as_tensor(p1, device="cuda"); P2 = torch.as_tensor(p2, device="cuda")
for var in ["ours", "ours_ns", "ours_ne", "ours_ne_s"]:
    cfg = SmoothingConfig().for_variant(var)
    out = {}
    fn = lambda: api.generate_manifold_batch(s1, s2, P1, P2, cfg, out=out)
    ms = time_fn(fn)
    print(f"manifold {var} n={n}: {ms:.3f} ms -> {n/ms*1e3/1e6:.2f} M manifolds/s")
pairs = torch.rand((1 << 22, 12), dtype=torch.float64, device="cuda")
for var in ["ours", "ours_ns"]:
    cfg = SmoothingConfig().for_variant(var)
    ms = time_fn(lambda: api.run_ee_batch(pairs, cfg))
    nb = pairs.shape[0] * (96 + 24)
    print(f"ee_witness {var} n={pairs.shape[0]}: {ms:.3f} ms -> {pairs.shape[0]/ms*1e3/1e9:.2f} G pairs/s, {nb/ms/1e6:.0f} GB/s")
    ms = time_fn(lambda: api.run_vf_batch(pairs, cfg))
    nb = pairs.shape[0] * (96 + 12)
    print(f"vf_witness {var}: {ms:.3f} ms -> {pairs.shape[0]/ms*1e3/1e9:.2f} G pairs/s, {nb/ms/1e6:.0f} GB/s")
for kind in W.MIXED_KINDS:
    ws = W.mixed_bucket(kind, n)
    a1 = api.surface_from_spec(ws.bodies[0]); a2 = api.surface_from_spec(ws.bodies[1])
    q1, q2 = ws.poses(n)
    Q1 = torch.as_tensor(q1, device="cuda"); Q2 = torch.as_tensor(q2, device="cuda")
    out = {}
    ms = time_fn(lambda: api.generate_manifold_batch(a1, a2, Q1, Q2, SmoothingConfig(), out=out))
    print(f"mixed {kind} n={n}: {ms:.3f} ms -> {n/ms*1e3/1e6:.2f} M manifolds/s")
for eps in (0.2, 0.5):
    ws = W.box_box_eps(eps, n)
    a1 = api.surface_from_spec(ws.bodies[0]); a2 = api.surface_from_spec(ws.bodies[1])
    q1, q2 = ws.poses(n)
    Q1 = torch.as_tensor(q1, device="cuda"); Q2 = torch.as_tensor(q2, device="cuda")
    out = {}
    ms = time_fn(lambda: api.generate_manifold_batch(a1, a2, Q1, Q2, SmoothingConfig(), out=out))
    print(f"box-box eps {eps} n={n}: {ms:.3f} ms -> {n/ms*1e3/1e6:.2f} M manifolds/s")
sc = W.drop_scene(32768)
bodies = [api.surface_from_spec(b) for b in sc.bodies]
P = torch.as_tensor(sc.poses(32768), device="cuda")
for fn_name in ("generate_manifold_scene_batch", "generate_manifold_scene_jvp_batch"):
    fn = getattr(api, fn_name)
    outs = [dict() for _ in range(10)]
    ms = time_fn(lambda: fn(bodies, P, SmoothingConfig(), is_static=sc.is_static(), outs=outs), reps=5)
    print(f"drop {fn_name}: {ms:.3f} ms -> {327680/ms*1e3/1e6:.2f} M pair-manifolds/s")
