"""Generate the committed golden fixtures from the COMPILED REFERENCE.

Runs only where /root/reference exists (this container): builds
oracle/_ref/libcmgref.so from the unmodified reference sources
(oracle/Makefile) and records its outputs on the shared cases of
tests/cases.py. The fixtures (*.npz next to this script) are what the CPU and
GPU tests compare against; nothing at test time reads /root/reference.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from oracle import Ref  # noqa: E402
from paper_2602_20304_b200.scene import SmoothingConfig  # noqa: E402
from paper_2602_20304_b200 import workloads as W  # noqa: E402
import cases  # noqa: E402


def ref_mesh(b):
    m = b.mesh
    return Ref.Mesh.box(m.box_half, m.subdivisions, m.quad_edges) if m.box_half is not None \
        else Ref.Mesh.parse_obj(m.obj_text)


def cfg_vec(c: SmoothingConfig):
    cc = c.to_c()
    return np.array([getattr(cc, f) for f, _ in cc._fields_], dtype=np.float64)


def main():
    oracle.build(ref=True)
    out = {}

    # --- witness batches: make_random_ee_pairs(2000, seed 0) ---------------
    pairs = Ref.random_pairs(2000, 0)
    out["witness"] = dict(pairs=pairs)
    for var in ("ours", "ours_ns"):
        c = SmoothingConfig().for_variant(var)
        out["witness"][f"ee_{var}"] = Ref.ee_witness_full(pairs, c)
        out["witness"][f"vf_{var}"] = Ref.vf_batch(pairs, c)[0]
        out["witness"][f"ee_checksum_{var}"] = np.array(Ref.ee_batch(pairs, c)[1])
    # --- raw box QPs -----------------------------------------------------------
    rng = np.random.default_rng(7)
    A = rng.normal(size=(500, 2, 2))
    Q = A @ np.transpose(A, (0, 2, 1)) + 1e-3 * np.eye(2)
    cvec = rng.normal(size=(500, 2))
    qp = np.stack([Q[:, 0, 0], Q[:, 0, 1], Q[:, 1, 1], cvec[:, 0], cvec[:, 1]], axis=1)
    out["box_qp"] = dict(qp=qp, ours=Ref.box_qp(qp, SmoothingConfig()),
                         ours_ns=Ref.box_qp(qp, SmoothingConfig().for_variant("ours_ns")))

    # --- SDF field queries -----------------------------------------------------
    rng = np.random.default_rng(11)
    pts = rng.uniform(-0.8, 0.8, size=(300, 3))
    sdf = {"points": pts}
    box = Ref.Mesh.box((0.5, 0.5, 0.5))
    for name, prog in cases.SDF_PROGRAMS.items():
        s = Ref.Surface(box, prog, 0, 0)
        for fl in (0, 1, 2):
            sdf[f"{name}_f{fl}"] = s.sdf_query(fl, pts)
        sdf[f"{name}_trace5"] = s.sphere_trace([0.1, -0.2, 0.3, 0.2, 0.1, -0.3], pts[:50], 5)
    out["sdf"] = sdf

    # --- soft top-K ------------------------------------------------------------
    xs = rng.normal(size=(20, 12))
    xs[3, 5] = xs[3, 7]  # an exact tie
    tk = {"xs": xs}
    for i, x in enumerate(xs):
        tk[f"w{i}"] = Ref.soft_topk(x, 4, 0.1)
    out["soft_topk"] = tk

    # --- meshes ------------------------------------------------------------------
    me = {}
    for i, (half, sub, quad) in enumerate(cases.BOX_MESHES):
        m = Ref.Mesh.box(half, sub, quad)
        me[f"box{i}_v"], me[f"box{i}_f"], me[f"box{i}_e"] = m.vertices, m.faces, m.edges
    for name, txt in cases.OBJ_TEXTS.items():
        m = Ref.Mesh.parse_obj(txt)
        me[f"obj_{name}_v"], me[f"obj_{name}_f"], me[f"obj_{name}_e"] = m.vertices, m.faces, m.edges
        me[f"obj_{name}_w"] = np.array(m.warnings, dtype=object).astype(str)
    for name, txt in cases.OBJ_ERRORS.items():
        try:
            Ref.Mesh.parse_obj(txt)
            me[f"err_{name}"] = np.array("no error")
        except ValueError as e:
            me[f"err_{name}"] = np.array(str(e))
    out["meshes"] = me

    # --- manifolds ----------------------------------------------------------------
    for name, ws, c, n in cases.manifold_cases():
        ms = [ref_mesh(b) for b in ws.bodies[:2]]
        rs = [Ref.Surface(m, b.sdf, b.vertex_topk, b.edge_topk) for m, b in zip(ms, ws.bodies[:2])]
        p1, p2 = ws.poses(n)
        r = Ref.manifold_batch(rs[0], rs[1], p1, p2, c, 1)
        one = Ref.manifold(rs[0], rs[1], p1[0], p2[0], c)
        out[f"manifold_{name}"] = dict(poses1=p1, poses2=p2, contacts=r["contacts"], meta=r["meta"],
                                       mean_dist=r["mean_dist"], layout=r["layout"], ee0=one["ee"],
                                       cfg=cfg_vec(c), warnings=np.array(rs[0].warnings + ["|"] + rs[1].warnings))

    # --- config D scene: all body pairs (DemoSim::step pair loop) ---------------------
    sc = W.drop_scene(4)
    P = sc.poses(4)
    ms = [ref_mesh(b) for b in sc.bodies]
    srs = [Ref.Surface(m, b.sdf, b.vertex_topk, b.edge_topk) for m, b in zip(ms, sc.bodies)]
    from paper_2602_20304_b200 import api
    pairs = api.scene_pairs(len(sc.bodies), sc.is_static())
    scene = {"poses": P, "pairs": pairs}
    for q, (i, j) in enumerate(pairs):
        r = Ref.manifold_batch(srs[i], srs[j], P[:, i], P[:, j], SmoothingConfig(), 1)
        scene[f"contacts{q}"] = r["contacts"]
        scene[f"meta{q}"] = r["meta"]
        scene[f"mean{q}"] = r["mean_dist"]
    out["scene_drop"] = scene

    # --- forward-mode pose Jacobian (Dual12) on box-on-plane, one env ---------------
    ws = W.box_on_plane()
    ms = [ref_mesh(b) for b in ws.bodies]
    rs = [Ref.Surface(m, b.sdf, b.vertex_topk, b.edge_topk) for m, b in zip(ms, ws.bodies)]
    j = Ref.manifold_jvp(rs[0], rs[1], ws.bodies[0].pose, ws.bodies[1].pose, SmoothingConfig())
    out["jvp_box_on_plane"] = dict(contacts=j["contacts"], tangents=j["tangents"],
                                   mean_dist=np.array(j["mean_dist"]), mean_dist_grad=j["mean_dist_grad"])
    # every smooth manifold case, first JVP_ENVS envs of its jittered batch
    jv = {}
    for name, ws, c, n in cases.manifold_cases():
        if c.hard_ops:
            continue
        ms = [ref_mesh(b) for b in ws.bodies[:2]]
        rs = [Ref.Surface(m, b.sdf, b.vertex_topk, b.edge_topk) for m, b in zip(ms, ws.bodies[:2])]
        p1, p2 = ws.poses(n)
        for e in range(cases.JVP_ENVS):
            j = Ref.manifold_jvp(rs[0], rs[1], p1[min(e, len(p1) - 1)], p2[min(e, len(p2) - 1)], c)
            if e < cases.JVP_FULL:
                jv[f"{name}_{e}_contacts"] = j["contacts"]
                jv[f"{name}_{e}_tangents"] = j["tangents"].astype(np.float32)  # the ABI emits FP32
            else:  # every JVP_STRIDE-th contact (keeps the fixture small)
                jv[f"{name}_{e}_contacts_sub"] = j["contacts"][::cases.JVP_STRIDE]
                jv[f"{name}_{e}_tangents_sub"] = j["tangents"][::cases.JVP_STRIDE].astype(np.float32)
            jv[f"{name}_{e}_mean"] = np.array([j["mean_dist"], *j["mean_dist_grad"]])
    # config D scene: pose Jacobians of every pair, env 0 (forward + 12-tangent JVP per pair)
    for q, (i, j) in enumerate(pairs):
        r = Ref.manifold_jvp(srs[i], srs[j], P[0, i], P[0, j], SmoothingConfig())
        jv[f"drop_pair{q}_0_contacts"] = r["contacts"]
        jv[f"drop_pair{q}_0_tangents"] = r["tangents"].astype(np.float32)
        jv[f"drop_pair{q}_0_mean"] = np.array([r["mean_dist"], *r["mean_dist_grad"]])
    out["jvp_cases"] = jv

    # --- DemoSim rollouts (src/demosim.cpp) on the demo scene, envs 0 and 1 --------------
    from paper_2602_20304_b200.scene import PenaltyParams
    dsc = W.demo_scene(2)
    DP = dsc.poses(2)
    drs = [Ref.Surface(ref_mesh(b), b.sdf, b.vertex_topk, b.edge_topk) for b in dsc.bodies]
    demo = {"init_poses": DP}
    for e in range(2):
        r = Ref.demo_run(drs, dsc.is_static(), np.ones(len(drs)), np.zeros((len(drs), 3)), DP[e],
                         np.zeros((len(drs), 6)), SmoothingConfig(), PenaltyParams(), cases.DEMO_DT, cases.DEMO_STEPS)
        for k, v in r.items():
            demo[f"{k}{e}"] = v
    # single box dropped on the ground, 16 jittered envs: poses after 100 / 200 steps
    dsc1 = W.demo_scene(16, n_boxes=1)
    DP1 = dsc1.poses(16)
    drs1 = [Ref.Surface(ref_mesh(b), b.sdf, b.vertex_topk, b.edge_topk) for b in dsc1.bodies]
    demo["box1_init_poses"] = DP1
    for e in range(16):
        r = Ref.demo_run(drs1, dsc1.is_static(), np.ones(2), np.zeros((2, 3)), DP1[e], np.zeros((2, 6)),
                         SmoothingConfig(), PenaltyParams(), cases.DEMO_DT, 200)
        demo[f"box1_{e}_s100"] = r["poses"][99]
        demo[f"box1_{e}_s200"] = r["poses"][199]
    out["demo"] = demo

    # --- Fig. 4 rotating-edge sweep + the reference tool's text outputs on the scene files ----
    tools = {f"sweep{v}": Ref.sweep(v, 1001) for v in range(3)}
    scenes_dir = os.path.join(os.path.dirname(HERE), "scenes")
    for name in ("box_on_plane", "capsule_vs_hollow"):
        sh = Ref.SceneHandle(open(os.path.join(scenes_dir, f"{name}.json")).read(), scenes_dir)
        b0, b1 = sh.bodies[0], sh.bodies[1]
        m = Ref.manifold(b0["surface"], b1["surface"], b0["pose"], b1["pose"], sh.smoothing)
        tools[f"{name}_contacts"] = m["contacts"]
        tools[f"{name}_meta"] = m["meta"]
    out["tools"] = tools

    for name, d in out.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


if __name__ == "__main__":
    main()
