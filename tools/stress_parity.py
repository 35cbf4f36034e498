"""Developer stress check: GPU vs the C oracle on large jittered batches of the
manifold cases (python tools/stress_parity.py [n] [--jvp]); --jvp checks the
pose-Jacobian kernel's primal contacts (smooth cases) the same way."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from cases import manifold_cases
from helpers import parity_report, surfaces
from oracle import Oracle
from paper_2602_20304_b200 import api

args = [a for a in sys.argv[1:] if not a.startswith("--")]
jvp = "--jvp" in sys.argv
n = int(args[0]) if args else 16384
for name, ws, cfg, _ in manifold_cases():
    if jvp and cfg.hard_ops:
        continue
    (a1, a2), (o1, o2) = surfaces(ws)
    p1, p2 = ws.poses(n)
    ref = Oracle.manifold_batch(o1, o2, p1, p2, cfg, threads=os.cpu_count())
    fn = api.generate_manifold_jvp_batch if jvp else api.generate_manifold_batch
    r = fn(a1, a2, torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda"), cfg, want_src=True)
    torch.cuda.synchronize()
    rep, bad = parity_report(r["contacts"].cpu().numpy(), ref["contacts"])
    src_bad = int((r["src"].cpu().numpy() != ref["meta"][..., 2:]).any(axis=-1).sum())
    worst = max(v["max_ratio"] for k, v in rep.items() if k != "per_component")
    pc = rep["per_component"]
    print(f"{'jvp ' if jvp else ''}{name:26s} n={n} failing contacts {int(bad.sum()):5d} / {bad.size}  worst ratio {worst:.3g}"
          f"  per-component: failing {pc['fails']} worst ratio {pc['max_ratio']:.3g}  src mismatches {src_bad}")
