#!/usr/bin/env python
"""Algorithmic work per unit for every bench workload (SURVEY.md §8(d) /
Appendix B recipe), written to profiles/work_per_unit.json, which bench.py
reads for its roofline.

W is counted by the REFERENCE itself: oracle/_ref/libcmgref.so's
cmgref_opcount_manifold instantiates generate_manifold<T>
(proj/include/cmg/manifold.hpp:336-377) with a counting scalar (one
add/sub/mul/div = 1 op, each transcendental = 1 op) -- or Dual<12, counting
scalar> for the reference's Jacobian formulation. Counts vary by a few ops with
the pose (branches on primals), so each figure is the mean over `--envs`
jittered envs of the workload's own pose stream.

Needs /root/reference (oracle/_ref is built from it); run in the dev
container, commit the JSON.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Ref  # noqa: E402
from paper_2602_20304_b200 import workloads as W  # noqa: E402
from paper_2602_20304_b200.scene import SmoothingConfig  # noqa: E402


def ref_surface(b):
    m = Ref.Mesh.box(b.mesh.box_half, b.mesh.subdivisions, b.mesh.quad_edges) if b.mesh.box_half is not None \
        else Ref.Mesh.parse_obj(b.mesh.obj_text)
    return Ref.Surface(m, b.sdf, b.vertex_topk, b.edge_topk)


def mean_count(s1, s2, p1, p2, cfg, jvp=False):
    rows = [Ref.opcount_manifold(s1, s2, p1[min(i, len(p1) - 1)], p2[min(i, len(p2) - 1)], cfg, jvp)
            for i in range(max(len(p1), len(p2)))]
    return {k: float(np.mean([r[k] for r in rows])) for k in rows[0]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=8)
    ap.add_argument("--jvp-envs", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "work_per_unit.json"))
    a = ap.parse_args()
    cfg = SmoothingConfig()
    out = {"recipe": "tools/count_work.py: the reference's generate_manifold<T> with a counting scalar "
                     "(oracle/ref_extra.cpp); W = arith + transcendentals, 1 op each; mean over jittered envs",
           "units": {}}

    def two_body(name, ws, note):
        s = [ref_surface(b) for b in ws.bodies]
        p1, p2 = ws.poses(a.envs)
        p1 = np.asarray(p1).reshape(-1, 6)
        p2 = np.asarray(p2).reshape(-1, 6)
        c = mean_count(s[0], s[1], p1, p2, cfg)
        out["units"][name] = {"W": c["W"], "arith": c["arith"], "transcendental": c["transcendental"],
                              "counts": c, "unit": "manifold", "note": note}
        print(name, c["W"], flush=True)
        return c

    two_body("box-box", W.box_box(a.envs), "config B: box-box, M=12, 304 contacts")
    for eps, note in ((0.2, "box-box with SQ eps 0.2 (integer 1/eps family)"),
                      (0.25, "box-box with SQ eps 0.25"), (0.5, "box-box with SQ eps 0.5")):
        if hasattr(W, "box_box_eps"):
            two_body(f"box-box-eps{eps:g}", W.box_box_eps(eps, a.envs), note)
    mixed = [two_body(f"mixed-{k}", W.mixed_bucket(k, a.envs), f"config C bucket {k}") for k in W.MIXED_KINDS]
    out["units"]["mixed"] = {"W": float(np.mean([c["W"] for c in mixed])), "unit": "manifold",
                             "note": "config C: mean over its 4 equal buckets"}

    # config D: every scene pair, forward and the reference's Dual12 formulation
    sc = W.drop_scene(a.envs)
    bodies = [ref_surface(b) for b in sc.bodies]
    pairs = [(i, j) for i in range(len(bodies)) for j in range(i + 1, len(bodies))
             if not (sc.bodies[i].is_static and sc.bodies[j].is_static)]
    P = sc.poses(a.envs)
    fw, jv = [], []
    for (i, j) in pairs:
        fw.append(mean_count(bodies[i], bodies[j], P[:, i], P[:, j], cfg)["W"])
        jv.append(mean_count(bodies[i], bodies[j], P[:a.jvp_envs, i], P[:a.jvp_envs, j], cfg, jvp=True)["W"])
        print("drop pair", i, j, fw[-1], jv[-1], flush=True)
    out["units"]["drop-fwd"] = {"W": float(np.mean(fw)), "unit": "pair manifold",
                                "per_pair": fw, "pairs": pairs, "note": "config D forward, mean over its 10 pairs"}
    out["units"]["drop"] = {"W": float(np.mean(jv)), "unit": "pair manifold (+ 12-tangent JVP)",
                            "per_pair": jv, "pairs": pairs,
                            "note": "config D: generate_manifold<Dual<12>> (the reference's Jacobian formulation)"}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
