"""Per-phase SM clocks of the JVP kernel, or of the manifold kernel with
`box-box` as the first argument (developer tool). Needs a library
built with `make -C paper_2602_20304_b200/csrc EXTRA_CUFLAGS=-DCMGB_PHASE_CLOCKS`
(after `make clean`); prints each phase's share of the CTA lifetime for one
config D forward + JVP step (python tools/phase_clocks.py [n_env])."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_20304_b200 import abi, api  # noqa: E402
from paper_2602_20304_b200 import workloads as W  # noqa: E402
from paper_2602_20304_b200.scene import SmoothingConfig  # noqa: E402

if len(sys.argv) > 1 and (sys.argv[1] == "box-box" or sys.argv[1].startswith("mixed:")):
    n = 65536
    ws = W.box_box(n) if sys.argv[1] == "box-box" else W.mixed_bucket(sys.argv[1].split(":", 1)[1], n)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n)
    P1, P2 = torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda")
    lib = abi.load()
    out = (C.c_ulonglong * 16)()
    api.generate_manifold_batch(s1, s2, P1, P2, SmoothingConfig())
    torch.cuda.synchronize()
    lib.cmgb_debug_manifold_phase_clocks(out)
    base = np.array(out[:], dtype=np.float64)
    api.generate_manifold_batch(s1, s2, P1, P2, SmoothingConfig())
    torch.cuda.synchronize()
    lib.cmgb_debug_manifold_phase_clocks(out)
    d = np.array(out[:], dtype=np.float64) - base
    names = {0: "A frames", 1: "B vertex scores", 2: "B edge scores", 3: "C rank sort", 4: "D slots",
             5: "E pairs (+ V-S)", 6: "F NN (+ V-S)", 7: "G activity + stores", 8: "H mean",
             9: "C2 top-K factors"}
    L = api.layout(s1, s2, SmoothingConfig())
    per_env = max(L["m1"] * L["m2"], L["n1"] + L["n2"], 1)
    epb = max(1, (288 if sys.argv[1] == "box-box" else 320) // per_env)
    ncta = -(-n // epb)
    tot = d[:10].sum()
    for k, nm in names.items():
        print(f"{nm:20s} {100 * d[k] / tot:6.2f} %  {d[k] / ncta:9.0f} clk per CTA")
    print(f"total {tot / ncta:.0f} clk per CTA ({ncta} CTAs)")
    sys.exit(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
sc = W.drop_scene(n)
bodies = [api.surface_from_spec(b) for b in sc.bodies]
P = torch.as_tensor(sc.poses(n), device="cuda")
lib = abi.load()
out = (C.c_ulonglong * 16)()
lib.cmgb_debug_jvp_phase_clocks(out)
base = np.array(out[:], dtype=np.float64)
api.generate_manifold_scene_jvp_batch(bodies, P, SmoothingConfig(), is_static=sc.is_static())
torch.cuda.synchronize()
lib.cmgb_debug_jvp_phase_clocks(out)
d = np.array(out[:], dtype=np.float64) - base
names = ["A frames", "B vertex scores", "B edge scores", "C rank sort", "D1 slot primals", "D2 slot tangents",
         "E1 Jacobians", "E1b pair primals", "E2 tangents", "F NN stats", "G activity"]
tot = d[:len(names)].sum()
ncta = sum(-(-n // upb) for upb in [int(sys.argv[2]) if len(sys.argv) > 2 else 2]) * 10
for k, nm in enumerate(names):
    print(f"{nm:20s} {100 * d[k] / tot:6.2f} %  {d[k] / ncta:9.0f} clk per CTA")
print(f"total {tot / ncta:.0f} clk per CTA (assuming {ncta} CTAs)")
