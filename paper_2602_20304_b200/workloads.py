"""Synthetic workloads of BASELINE.json, pinned as in SURVEY.md §8(d).

A workload is a backend-neutral description: per body a mesh spec (box
generator or OBJ text), an SDF tree, top-K budgets and a base pose, plus the
pose-jitter rule of bench_manifold (src/batch.cpp:196-203): body 1 fixed,
body 2 += U(-0.05, 0.05)^6 from std::mt19937_64(seed), 6 draws per env in env
order (so the first N envs of a larger batch equal the N-env batch).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .scene import SdfNode, Superquadric, Union, box_planes


def so3_log(R: np.ndarray) -> np.ndarray:
    """so3_log (src/pose.cpp:10-33), generic branch (angles in (1e-8, pi-1e-6))."""
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    c = min(1.0, max(-1.0, 0.5 * (tr - 1.0)))
    th = math.acos(c)
    vee = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    if th < 1e-8:
        return vee * 0.5
    return vee * (0.5 * th / math.sin(th))


def so3_exp(w: Sequence[float]) -> np.ndarray:
    """so3_exp (include/cmg/pose.hpp:70-76) in double."""
    w = np.asarray(w, dtype=np.float64)
    th2 = float(w @ w)
    if th2 < 1e-8:
        a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0
        b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0
    else:
        th = math.sqrt(th2)
        a = math.sin(th) / th
        b = (1.0 - math.cos(th)) / th2
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    return np.eye(3) + W * a + (W @ W) * b


def rz_axis_angle(theta: float) -> List[float]:
    """Axis-angle of Rz(theta) through so3_exp/so3_log as the reference builds it."""
    return list(so3_log(so3_exp([0.0, 0.0, theta])))


@dataclass
class MeshSpec:
    box_half: Optional[Sequence[float]] = None
    subdivisions: int = 1
    quad_edges: bool = True
    obj_text: Optional[str] = None


@dataclass
class BodySpec:
    name: str
    mesh: MeshSpec
    sdf: SdfNode
    pose: Sequence[float]
    vertex_topk: int = 0
    edge_topk: int = 0
    is_static: bool = False


@dataclass
class Workload:
    name: str
    bodies: List[BodySpec]
    n_env: int
    jitter: float = 0.05
    seed: int = 0
    notes: str = ""
    pairs: Optional[List[tuple]] = None  # multi-body: list of (i, j) pairs

    def poses(self, n_env: Optional[int] = None):
        """(poses1 [1,6] shared, poses2 [n,6] jittered) as bench_manifold builds them."""
        n = self.n_env if n_env is None else n_env
        p1 = np.asarray(self.bodies[0].pose, dtype=np.float64)[None, :]
        p2 = jittered_poses(self.bodies[1].pose, n, self.jitter, self.seed)
        return p1, p2


def mt19937_64_uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    """std::mt19937_64(seed) + uniform_real_distribution<double>(lo, hi) (libstdc++).

    Pure numpy restatement used to synthesise poses identically to the
    reference's bench_manifold (src/batch.cpp:196-203)."""
    NN, MM = 312, 156
    mask = (1 << 64) - 1
    mt = [0] * NN
    mt[0] = seed & mask
    for i in range(1, NN):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & mask
    mt = np.array(mt, dtype=np.uint64)
    out = np.empty(n, dtype=np.float64)
    UM = np.uint64(0xFFFFFFFF80000000)
    LM = np.uint64(0x7FFFFFFF)
    A = np.uint64(0xB5026F5AA96619E9)
    k = 0
    while k < n:
        # twist (vectorised in the three dependency-free segments)
        for lo_i, hi_i in ((0, NN - MM), (NN - MM, NN - 1)):
            idx = np.arange(lo_i, hi_i)
            x = (mt[idx] & UM) | (mt[idx + 1] & LM)
            xa = x >> np.uint64(1)
            xa ^= np.where((x & np.uint64(1)) != 0, A, np.uint64(0))
            mt[idx] = mt[(idx + MM) % NN] ^ xa
        x = (mt[NN - 1] & UM) | (mt[0] & LM)
        xa = x >> np.uint64(1)
        if int(x) & 1:
            xa ^= A
        mt[NN - 1] = mt[MM - 1] ^ xa
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        take = min(NN, n - k)
        r = y[:take].astype(np.float64) / 18446744073709551616.0
        r = np.where(r >= 1.0, np.nextafter(1.0, 0.0), r)
        out[k:k + take] = r * (hi - lo) + lo
        k += take
    return out


def jittered_poses(base: Sequence[float], n_env: int, jitter: float = 0.05, seed: int = 0) -> np.ndarray:
    """bench_manifold's pose jitter (src/batch.cpp:196-203)."""
    j = mt19937_64_uniform(seed, 6 * n_env, -jitter, jitter).reshape(n_env, 6)
    return np.asarray(base, dtype=np.float64)[None, :] + j


# ---------------------------------------------------------------------------
# Config A / B: box-box (proj/tests/probe.cpp:23-47 geometry) and box-on-plane
# ---------------------------------------------------------------------------
BOX_SQ = Superquadric(0.1, 0.1, (0.5, 0.5, 0.5))


def box_box(n_env: int = 65536, edge_topk: int = 12) -> Workload:
    """Config B: quad cube half 0.5 + SQ eps 0.1 per body, vertex_topk 0,
    edge_topk 12 (304 contacts); body 1 at (0,0,0.5), body 2 at
    (0.02, 0.035, 1.46, Rz(pi/4)) + jitter."""
    mesh = MeshSpec(box_half=(0.5, 0.5, 0.5))
    b1 = BodySpec("box1", mesh, BOX_SQ, [0.0, 0.0, 0.5, 0.0, 0.0, 0.0], 0, edge_topk)
    b2 = BodySpec("box2", mesh, BOX_SQ, [0.02, 0.035, 1.46] + rz_axis_angle(math.pi / 4), 0,
                  edge_topk)
    return Workload("box-box", [b1, b2], n_env,
                    notes="box-box V-S + E-E, M=12 (144 E-E pairs, 304 contacts/env)")


def box_box_eps(eps: float, n_env: int = 65536, edge_topk: int = 12) -> Workload:
    """Config B's scene with superquadric boxiness eps1 = eps2 = eps instead of
    0.1 (the integer 1/eps family 0.2 / 0.25 / 0.5 runs on compile-time
    exponent kinds; any other eps on the runtime-exponent kind)."""
    w = box_box(n_env, edge_topk)
    sq = Superquadric(eps, eps, (0.5, 0.5, 0.5))
    for b in w.bodies:
        b.sdf = sq
    w.name = f"box-box-eps{eps:g}"
    w.notes = f"box-box, SQ eps {eps:g}, M=12 (304 contacts/env)"
    return w


def box_on_plane(n_env: int = 1) -> Workload:
    """Config A (box-on-plane): box (SQ eps .1) over a 2x2x0.1 ground (box_planes
    CP, tau 1e-3); full mode = 40 contacts (n 8/8, m 12/1)."""
    box = BodySpec("box", MeshSpec(box_half=(0.5, 0.5, 0.5)), BOX_SQ,
                   [0.0, 0.0, 0.49, 0.0, 0.0, 0.0], 0, 12)
    ground = BodySpec("ground", MeshSpec(box_half=(2.0, 2.0, 0.1)), box_planes((2.0, 2.0, 0.1)),
                      [0.0, 0.0, -0.1, 0.0, 0.0, 0.0], 0, 0, is_static=True)
    return Workload("box-on-plane", [box, ground], n_env)


def sq_obj_text(eps1: float, eps2: float, axes: Sequence[float], n_lat: int = 6, n_lon: int = 8,
                z_offset: float = 0.0) -> str:
    """Tessellated superquadric surface as OBJ text (quads + polar triangles),
    vertices on the parametric surface f = 1 (builder-generated
    meshes ingested by parse_obj)."""

    def spow(x, e):
        return math.copysign(abs(x) ** e, x)

    verts = [(0.0, 0.0, axes[2] + z_offset)]
    for i in range(1, n_lat):
        eta = math.pi / 2 - math.pi * i / n_lat
        for j in range(n_lon):
            om = -math.pi + 2 * math.pi * j / n_lon
            x = axes[0] * spow(math.cos(eta), eps1) * spow(math.cos(om), eps2)
            y = axes[1] * spow(math.cos(eta), eps1) * spow(math.sin(om), eps2)
            z = axes[2] * spow(math.sin(eta), eps1) + z_offset
            verts.append((x, y, z))
    verts.append((0.0, 0.0, -axes[2] + z_offset))
    south = len(verts)  # 1-based index of the south pole
    lines = [f"v {x:.17g} {y:.17g} {z:.17g}" for x, y, z in verts]

    def ring(i, j):  # 1-based OBJ index of ring i (1..n_lat-1), column j
        return 2 + (i - 1) * n_lon + (j % n_lon)

    for j in range(n_lon):
        lines.append(f"f 1 {ring(1, j)} {ring(1, j + 1)}")
    for i in range(1, n_lat - 1):
        for j in range(n_lon):
            lines.append(f"f {ring(i, j)} {ring(i + 1, j)} {ring(i + 1, j + 1)} {ring(i, j + 1)}")
    for j in range(n_lon):
        lines.append(f"f {south} {ring(n_lat - 1, j + 1)} {ring(n_lat - 1, j)}")
    return "\n".join(lines) + "\n"


def capsule_obj_text(radius: float, half_len: float, n_cap: int = 3, n_lon: int = 8) -> str:
    """Tessellated capsule (two hemispherical caps joined by a cylinder band)."""
    verts = [(0.0, 0.0, half_len + radius)]
    rings = []
    for cap_z, sgn in ((half_len, 1.0), (-half_len, -1.0)):
        etas = [math.pi / 2 * (1 - i / n_cap) for i in range(1, n_cap + 1)]
        if sgn < 0:
            etas = [-e for e in reversed(etas)]
        for eta in etas:
            ring = []
            for j in range(n_lon):
                om = -math.pi + 2 * math.pi * j / n_lon
                rho = radius * math.cos(eta)
                verts.append((rho * math.cos(om), rho * math.sin(om), cap_z + radius * math.sin(eta)))
                ring.append(len(verts))
            rings.append(ring)
    verts.append((0.0, 0.0, -half_len - radius))
    south = len(verts)
    lines = [f"v {x:.17g} {y:.17g} {z:.17g}" for x, y, z in verts]
    for j in range(n_lon):
        lines.append(f"f 1 {rings[0][j]} {rings[0][(j + 1) % n_lon]}")
    for a, b in zip(rings[:-1], rings[1:]):
        for j in range(n_lon):
            lines.append(f"f {a[j]} {b[j]} {b[(j + 1) % n_lon]} {a[(j + 1) % n_lon]}")
    for j in range(n_lon):
        lines.append(f"f {south} {rings[-1][(j + 1) % n_lon]} {rings[-1][j]}")
    return "\n".join(lines) + "\n"


def _mixed_primitive(kind: str):
    """(sdf, mesh spec, half height) of the config-C primitive families."""
    from .scene import Union as _Union

    if kind == "rounded_box":
        ax = (0.3, 0.2, 0.15)
        return Superquadric(0.2, 0.2, ax), MeshSpec(obj_text=sq_obj_text(0.2, 0.2, ax)), ax[2]
    if kind == "cylinder":
        ax = (0.15, 0.15, 0.25)
        return Superquadric(0.1, 1.0, ax), MeshSpec(obj_text=sq_obj_text(0.1, 1.0, ax)), ax[2]
    if kind == "ellipsoid":
        ax = (0.3, 0.2, 0.15)
        return Superquadric(1.0, 1.0, ax), MeshSpec(obj_text=sq_obj_text(1.0, 1.0, ax)), ax[2]
    if kind == "capsule":
        r, h = 0.1, 0.2
        sdf = _Union([Superquadric(0.1, 1.0, (r, r, h)),
                      Superquadric(1.0, 1.0, (r, r, r), (0, 0, h, 0, 0, 0)),
                      Superquadric(1.0, 1.0, (r, r, r), (0, 0, -h, 0, 0, 0))], 0.01)
        return sdf, MeshSpec(obj_text=capsule_obj_text(r, h)), h + r
    raise ValueError(f"unknown mixed primitive {kind!r}")


def mixed_bucket(kind: str, n_env: int = 65536) -> Workload:
    """One bucket of config C: a primitive-family body (body 2, jittered) resting
    on a convex mesh plate make_box_mesh({0.4,0.4,0.1}, 2) + box_planes
    (body 1, fixed); budgets vertex_topk 16/16, edge_topk 8/8 -> 160 contacts
    (builder-pinned parameters)."""
    sdf, mesh, hz = _mixed_primitive(kind)
    plate = BodySpec("plate", MeshSpec(box_half=(0.4, 0.4, 0.1), subdivisions=2),
                     box_planes((0.4, 0.4, 0.1)), [0.0, 0.0, 0.0, 0.0, 0.0, 0.0], 16, 8, is_static=True)
    prim = BodySpec(kind, mesh, sdf, [0.02, -0.03, 0.1 + hz - 0.01, 0.15, -0.1, 0.3], 16, 8)
    return Workload(f"mixed-{kind}", [plate, prim], n_env,
                    notes=f"{kind} vs convex mesh plate, soft top-K 16/16 vertices, 8/8 edges")


MIXED_KINDS = ("rounded_box", "cylinder", "ellipsoid", "capsule")


# ---------------------------------------------------------------------------
# Config D: multi-body drop scene (all geom pairs), SURVEY §8(d) D
# ---------------------------------------------------------------------------
@dataclass
class Scene:
    name: str
    bodies: List[BodySpec]
    n_env: int
    jitter: float = 0.05
    seed: int = 0

    def is_static(self) -> np.ndarray:
        return np.array([b.is_static for b in self.bodies], dtype=np.int32)

    def poses(self, n_env: Optional[int] = None) -> np.ndarray:
        """[n_env, n_bodies, 6]: base poses; every dynamic body jittered by
        U(-j, j)^6 from one std::mt19937_64(seed) stream in (env, body) order."""
        n = self.n_env if n_env is None else n_env
        base = np.array([b.pose for b in self.bodies], dtype=np.float64)
        dyn = np.flatnonzero(~self.is_static().astype(bool))
        j = mt19937_64_uniform(self.seed, 6 * n * len(dyn), -self.jitter, self.jitter).reshape(n, len(dyn), 6)
        out = np.repeat(base[None], n, axis=0)
        out[:, dyn] += j
        return out


def drop_scene(n_env: int = 32768, n_boxes: int = 4) -> Scene:
    """4 dynamic boxes (quad cube half 0.5, SQ eps 0.1, vertex_topk 0, edge_topk
    4) stacked with 1 cm overlaps and a yaw twist over a static ground
    (box_planes 2x2x0.1, edge_topk 4): 6 box-box + 4 box-ground pairs, 48
    contacts each (builder-pinned parameters of config D)."""
    ground = BodySpec("ground", MeshSpec(box_half=(2.0, 2.0, 0.1)), box_planes((2.0, 2.0, 0.1)),
                      [0.0, 0.0, -0.1, 0.0, 0.0, 0.0], 0, 4, is_static=True)
    boxes = [BodySpec(f"box{k}", MeshSpec(box_half=(0.5, 0.5, 0.5)), BOX_SQ,
                      [0.03 * k, -0.02 * k, 0.49 + 0.99 * k] + rz_axis_angle(0.2 * k + 0.05), 0, 4)
             for k in range(n_boxes)]
    return Scene("drop", [ground] + boxes, n_env)

def demo_scene(n_env: int = 4096, n_boxes: int = 3) -> Scene:
    """Demo-integrator scene (DemoSim, src/demosim.cpp): n_boxes dynamic boxes
    (as drop_scene) released with 5-7 cm gaps above a static box_planes
    ground, pose jitter U(-0.02, 0.02): they fall, collide and settle."""
    ground = BodySpec("ground", MeshSpec(box_half=(2.0, 2.0, 0.1)), box_planes((2.0, 2.0, 0.1)),
                      [0.0, 0.0, -0.1, 0.0, 0.0, 0.0], 0, 4, is_static=True)
    boxes = [BodySpec(f"box{k}", MeshSpec(box_half=(0.5, 0.5, 0.5)), BOX_SQ,
                      [0.03 * k, -0.02 * k, 0.55 + 1.07 * k] + rz_axis_angle(0.2 * k + 0.05), 0, 4)
             for k in range(n_boxes)]
    return Scene("demo", [ground] + boxes, n_env, jitter=0.02)


WORKLOADS = {
    "box-box": box_box,
    "box-on-plane": box_on_plane,
}
