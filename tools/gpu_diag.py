"""Developer diagnostic: parity statistics of the CUDA path vs the C oracle
for every workload / variant (prints, never asserts). Run on a GPU box:
    python tools/gpu_diag.py [n_env]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import parity_report, surfaces  # noqa: E402
from oracle import Oracle  # noqa: E402
from paper_2602_20304_b200 import api  # noqa: E402
from paper_2602_20304_b200.scene import SmoothingConfig  # noqa: E402
from paper_2602_20304_b200 import workloads as W  # noqa: E402


def run_case(name, ws, cfg, n):
    (a1, a2), (o1, o2) = surfaces(ws)
    p1, p2 = ws.poses(n)
    t = time.time()
    ref = Oracle.manifold_batch(o1, o2, p1, p2, cfg, want_ee=True)
    t_orc = time.time() - t
    g = api.generate_manifold_batch(a1, a2, torch.as_tensor(p1, device="cuda"),
                                    torch.as_tensor(p2, device="cuda"), cfg, want_src=True,
                                    want_ee=True)
    torch.cuda.synchronize()
    got = g["contacts"].cpu().numpy()
    rep, bad = parity_report(got, ref["contacts"])
    src_ok = np.array_equal(g["src"].cpu().numpy(), ref["meta"][..., 2:])
    md = np.abs(g["mean_dist"].cpu().numpy() - ref["mean_dist"]).max()
    print(f"== {name} n={n} C={got.shape[1]} oracle {t_orc:.2f}s src_equal={src_ok} mean_dist_maxerr={md:.3g}")
    for f, r in rep.items():
        print(f"   {f:9s} fails {r['fails']:6d}/{r['n']} max_err {r['max_err']:.3g} max_ratio {r['max_ratio']:.3g}")
    if "ee" in g and ref["ee"] is not None and ref["ee"].shape[-1]:
        ee_g = g["ee"].cpu().numpy()
        names = ["dist", "con", "pen1", "pen2", "nn1", "nn2", "clash", "act1", "act2"]
        errs = np.abs(ee_g - ref["ee"])
        bound = 1e-6 + 1e-5 * np.abs(ref["ee"])
        for k, nm in enumerate(names):
            nb = int((errs[:, k] > bound[:, k]).sum())
            print(f"   ee.{nm:6s} fails {nb:6d} max_err {errs[:, k].max():.3g}")
    if bad.any():
        idx = np.argwhere(bad)[:6]
        for i in idx:
            e, c = (int(x) for x in i)
            print(f"   bad env {e} contact {c}: got {got[e, c]}\n                    ref {ref['contacts'][e, c]}")


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    base = SmoothingConfig()
    cases = [
        ("box-box ours", W.box_box(), base),
        ("box-box ours_ns", W.box_box(), base.for_variant("ours_ns")),
        ("box-box ours_ne", W.box_box(), base.for_variant("ours_ne")),
        ("box-box ours_ne_s", W.box_box(), base.for_variant("ours_ne_s")),
        ("box-on-plane ours", W.box_on_plane(), base),
        ("box-on-plane ours_ns", W.box_on_plane(), base.for_variant("ours_ns")),
    ]
    ws = W.box_box()
    ws.bodies[0].vertex_topk, ws.bodies[1].vertex_topk = 4, 3
    ws.bodies[0].edge_topk, ws.bodies[1].edge_topk = 5, 4
    cases.append(("box-box topk", ws, base))
    c2 = SmoothingConfig()
    c2.containment_safeguard = True
    cases.append(("box-box containment", W.box_box(), c2))
    for name, ws, cfg in cases:
        run_case(name, ws, cfg, n)

    # witness batches
    pairs = W.mt19937_64_uniform(0, 12 * 100000, 0.0, 1.0).reshape(-1, 12)
    for var in ["ours", "ours_ns"]:
        cfg = base.for_variant(var)
        ref, lab = Oracle.ee_witness(pairs, cfg)
        g = api.run_ee_batch(torch.as_tensor(pairs, device="cuda"), cfg, want_alpha=True, want_labels=True)
        got = g["out"].cpu().numpy()
        err = np.abs(got - ref[:, :6])
        bad = err > 1e-6 + 1e-5 * np.abs(ref[:, :6])
        lab_g = g["labels"].cpu().numpy()
        print(f"== ee_witness {var}: point fails {int(bad.sum())} max_err {err.max():.3g}; label mismatches {int((lab_g != lab).sum())}")
        refv, labv = Oracle.vf_witness(pairs, cfg)
        gv = api.run_vf_batch(torch.as_tensor(pairs, device="cuda"), cfg, want_labels=True)
        gotv = gv["out"].cpu().numpy()
        errv = np.abs(gotv - refv)
        badv = errv > 1e-6 + 1e-5 * np.abs(refv)
        print(f"== vf_witness {var}: fails {int(badv.sum())} max_err {errv.max():.3g}; label mismatches {int((gv['labels'].cpu().numpy() != labv).sum())}")


if __name__ == "__main__":
    main()
