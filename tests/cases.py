"""Shared test-case definitions (used by tests/golden/make_golden.py to produce
the committed fixtures from the compiled reference, and by the tests that
check the oracle and the CUDA path against them)."""
from __future__ import annotations

import math

import numpy as np

from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import (ConvexPolyhedron, OrientedPointcloud, SmoothingConfig,
                                         Subtraction, Superquadric, Union, box_planes)


def sphere_cloud(n=60, r=0.3, th=0.15, seed=3):
    """Oriented point cloud sampled on a sphere (OPC primitive, sdf.hpp:64-79)."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return OrientedPointcloud(points=v * r, normals=v.copy(), lengthscales=np.full(n, th))


def capsule(radius=0.1, half_len=0.2, tau=0.01):
    """Capsule = smooth union of an SQ cylinder and two SQ spheres."""
    cyl = Superquadric(0.1, 1.0, (radius, radius, half_len))
    s1 = Superquadric(1.0, 1.0, (radius, radius, radius), (0, 0, half_len, 0, 0, 0))
    s2 = Superquadric(1.0, 1.0, (radius, radius, radius), (0, 0, -half_len, 0, 0, 0))
    return Union([cyl, s1, s2], tau)


# SDF programs for field-level golden vectors (value / gradient / normal source).
SDF_PROGRAMS = {
    "sq_sphere": Superquadric(1.0, 1.0, (1.0, 1.0, 1.0)),
    "sq_box01": Superquadric(0.1, 0.1, (0.5, 0.5, 0.5)),
    "sq_round_posed": Superquadric(0.2, 0.2, (0.3, 0.2, 0.15), (0.05, -0.02, 0.1, 0.3, -0.2, 0.5)),
    "sq_cylinder": Superquadric(0.1, 1.0, (0.15, 0.15, 0.25)),
    "sq_general": Superquadric(0.7, 1.3, (0.4, 0.3, 0.2)),
    "cp_box": box_planes((0.4, 0.4, 0.1)),
    "cp_tet": ConvexPolyhedron(
        normals=np.array([[0, 0, -1.0], [0.942809, 0, 0.333333], [-0.471405, 0.816497, 0.333333],
                          [-0.471405, -0.816497, 0.333333]]) /
        np.linalg.norm(np.array([[0, 0, -1.0], [0.942809, 0, 0.333333], [-0.471405, 0.816497, 0.333333],
                                 [-0.471405, -0.816497, 0.333333]]), axis=1, keepdims=True),
        points=np.array([[0, 0, -0.1], [0.1, 0, 0], [0, 0.1, 0], [0, -0.1, 0.0]]), tau=0.005),
    "opc_sphere": sphere_cloud(),
    "union_capsule": capsule(),
    "subtraction": Subtraction(Superquadric(1.0, 1.0, (0.5, 0.5, 0.5)),
                               Superquadric(1.0, 1.0, (0.2, 0.2, 0.2), (0.1, 0, 0, 0, 0, 0)), 0.01),
    "nested": Union([Subtraction(box_planes((0.3, 0.3, 0.3)), Superquadric(1.0, 1.0, (0.15,) * 3), 0.02),
                     Superquadric(0.3, 0.3, (0.2, 0.1, 0.1), (0.35, 0, 0, 0, 0, 0))], 0.01),
}


JVP_ENVS = 16  # envs per case with recorded reference pose Jacobians (Dual12)
JVP_FULL = 2   # the first JVP_FULL envs keep every contact's tangents; later envs every JVP_STRIDE-th contact
JVP_STRIDE = 16
JVP_FD_ENVS = 4  # envs per case whose reference tangents are also checked by finite differences (CPU suite)
MANIFOLD_ENVS = 16
DEMO_DT = 1e-3  # DemoSim golden rollouts: step and length (demo scene, envs 0 and 1)
DEMO_STEPS = 300


def manifold_cases():
    """(name, workload, cfg, n_env) for manifold golden fixtures / parity tests."""
    base = SmoothingConfig()
    out = []
    for var in ("ours", "ours_ns", "ours_ne", "ours_ne_s"):
        out.append((f"box_box_{var}", W.box_box(), base.for_variant(var), MANIFOLD_ENVS))
    out.append(("box_on_plane_ours", W.box_on_plane(), base, MANIFOLD_ENVS))
    out.append(("box_on_plane_ours_ns", W.box_on_plane(), base.for_variant("ours_ns"), MANIFOLD_ENVS))
    ws = W.box_box()
    ws.bodies[0].vertex_topk, ws.bodies[1].vertex_topk = 4, 3
    ws.bodies[0].edge_topk, ws.bodies[1].edge_topk = 5, 4
    out.append(("box_box_topk", ws, base, MANIFOLD_ENVS))
    c = SmoothingConfig()
    c.containment_safeguard = True
    out.append(("box_box_containment", W.box_box(), c, MANIFOLD_ENVS))
    c = SmoothingConfig()
    c.sphere_trace = False
    out.append(("box_box_notrace", W.box_box(), c, MANIFOLD_ENVS))
    for name in ("mixed_rounded_box", "mixed_cylinder", "mixed_ellipsoid", "mixed_capsule"):
        out.append((name, W.mixed_bucket(name.split("_", 1)[1]), base, MANIFOLD_ENVS))
    out.append(("opc_vs_box", opc_vs_box(), base, MANIFOLD_ENVS))
    out.append(("subtraction_vs_box", subtraction_vs_box(), base, MANIFOLD_ENVS))
    out.append(("octahedron_vs_box", octahedron_vs_box(), base, MANIFOLD_ENVS))
    # the compile-time-exponent superquadric kinds beside eps 0.1 (common.h SdfKind)
    for eps, tag in ((0.2, "02"), (0.25, "025"), (0.5, "05"), (1.0, "1")):
        out.append((f"box_box_eps{tag}", W.box_box_eps(eps), base, MANIFOLD_ENVS))
    cyl = W.box_box()
    for b in cyl.bodies:
        b.sdf = Superquadric(0.1, 1.0, (0.5, 0.5, 0.5))
    out.append(("cyl_cyl", cyl, base, MANIFOLD_ENVS))
    return out


def opc_vs_box():
    """Oriented-pointcloud ball (mesh = tessellated sphere) against an SQ box."""
    ball = W.BodySpec("ball", W.MeshSpec(obj_text=W.sq_obj_text(1.0, 1.0, (0.3, 0.3, 0.3))),
                      sphere_cloud(), [0.0, 0.0, 0.0, 0.0, 0.0, 0.0], 8, 6)
    box = W.BodySpec("box", W.MeshSpec(box_half=(0.5, 0.5, 0.5)), W.BOX_SQ,
                     [0.1, -0.05, 0.78, 0.1, 0.2, 0.3], 0, 6)
    return W.Workload("opc-vs-box", [ball, box], 8)


def subtraction_vs_box():
    hollow = Subtraction(Superquadric(0.2, 0.2, (0.5, 0.5, 0.5)),
                         Superquadric(1.0, 1.0, (0.3, 0.3, 0.3), (0, 0, 0.35, 0, 0, 0)), 0.01)
    b1 = W.BodySpec("hollow", W.MeshSpec(box_half=(0.5, 0.5, 0.5)), hollow,
                    [0.0, 0.0, 0.5, 0.0, 0.0, 0.0], 0, 8)
    b2 = W.BodySpec("box", W.MeshSpec(box_half=(0.2, 0.2, 0.2)), Superquadric(0.1, 0.1, (0.2, 0.2, 0.2)),
                    [0.05, 0.0, 1.1, 0.0, 0.0, math.pi / 5], 6, 8)
    return W.Workload("subtraction-vs-box", [b1, b2], 8)


def octahedron_vs_box():
    """A general convex polyhedron (8 oblique planes: the kSingleCp path) with
    its own OBJ mesh against an SQ box."""
    r = 0.45
    verts = [(r, 0, 0), (-r, 0, 0), (0, r, 0), (0, -r, 0), (0, 0, r), (0, 0, -r)]
    faces = [(1, 3, 5), (3, 2, 5), (2, 4, 5), (4, 1, 5), (3, 1, 6), (2, 3, 6), (4, 2, 6), (1, 4, 6)]
    obj = "\n".join([f"v {x} {y} {z}" for x, y, z in verts] + [f"f {a} {b} {c}" for a, b, c in faces]) + "\n"
    s3 = 1.0 / math.sqrt(3.0)
    normals = [(sx * s3, sy * s3, sz * s3) for sx in (1, -1) for sy in (1, -1) for sz in (1, -1)]
    points = [(sx * r, 0.0, 0.0) for sx in (1, -1) for _ in (1, -1) for _ in (1, -1)]
    octa = W.BodySpec("octa", W.MeshSpec(obj_text=obj), ConvexPolyhedron(np.array(normals), np.array(points), 1e-3),
                      [0.02, -0.01, 0.0, 0.1, 0.05, 0.2], 0, 6)
    box = W.BodySpec("box", W.MeshSpec(box_half=(0.3, 0.3, 0.3)), Superquadric(0.1, 0.1, (0.3, 0.3, 0.3)),
                     [0.05, 0.02, 0.72, 0.0, 0.1, 0.3], 0, 6)
    return W.Workload("octahedron-vs-box", [octa, box], 8)


OBJ_TEXTS = {
    "tri_cube": """v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nv 0 0 1\nv 1 0 1\nv 1 1 1\nv 0 1 1
f 1 3 2\nf 1 4 3\nf 5 6 7\nf 5 7 8\nf 1 2 6\nf 1 6 5\nf 2 3 7\nf 2 7 6\nf 3 4 8\nf 3 8 7\nf 4 1 5\nf 4 5 8
""",
    "quad_cube": """# quad cube\nv -1 -1 -1\nv 1 -1 -1\nv 1 1 -1\nv -1 1 -1\nv -1 -1 1\nv 1 -1 1\nv 1 1 1\nv -1 1 1
f 1 4 3 2\nf 5 6 7 8\nf 1 2 6 5\nf 2 3 7 6\nf 3 4 8 7\nf 4 1 5 8
""",
    "slashes_negative": """v 0 0 0\nv 1 0 0\nv 0 1 0\nv 0 0 1\nvn 0 0 1\nf 1/1/1 2//1 3\nf -4 -3 -1\n""",
    "non_manifold": """v 0 0 0\nv 1 0 0\nv 0 1 0\nv 0 -1 0\nv 0 0 1\nf 1 2 3\nf 1 2 4\nf 1 2 5\n""",
    "sq_tessellated": W.sq_obj_text(0.2, 0.2, (0.3, 0.2, 0.15)),
}

OBJ_ERRORS = {
    "bad_vertex": "v 0 0\n",
    "pentagon": "v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nv 0 2 0\nf 1 2 3 4 5\n",
    "out_of_range": "v 0 0 0\nv 1 0 0\nf 1 2 3\n",
    "bad_index": "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 x 3\n",
    "empty": "# nothing\n",
}

BOX_MESHES = [((0.5, 0.5, 0.5), 1, True), ((2.0, 2.0, 0.1), 1, True), ((0.5, 0.5, 0.5), 4, True),
              ((0.4, 0.4, 0.1), 2, True), ((0.5, 0.3, 0.2), 3, False), ((1.0, 0.5, 0.25), 2, False)]
