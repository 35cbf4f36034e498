"""Scene documents and text outputs of the reference's tools, on this package's
API: parse_scene / load_scene (src/scene.cpp:130-185: the JSON scene schema,
its defaults and its error messages), write_manifold_csv / manifold_to_json
(src/manifold_io.cpp:24-52: CSV schema v1 and the JSON mirror), write_bench_csv
(src/batch.cpp:122-129, "cmg-bench-csv v1") and write_sweep_csv
(src/sweep.cpp:58-72). The bodies of a parsed scene are live Surfaces
(geometry uploaded to the GPU on first use)."""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import abi, api
from .scene import (ConvexPolyhedron, OrientedPointcloud, SmoothingConfig, Subtraction, Superquadric,
                    Union)


class SceneError(ValueError):
    """cmg::SceneError (include/cmg/scene.hpp:29-31)."""


@dataclass
class SceneBody:
    """cmg::SceneBody (include/cmg/scene.hpp:15-22)."""

    name: str
    surface: api.Surface
    sdf: object
    pose: np.ndarray
    mass: float = 1.0
    inertia_diag: np.ndarray = field(default_factory=lambda: np.zeros(3))
    is_static: bool = False
    vertex_topk: int = 0
    edge_topk: int = 0


@dataclass
class SceneDoc:
    bodies: List[SceneBody]
    smoothing: SmoothingConfig


def _vec3(j, what):
    if not isinstance(j, list) or len(j) != 3:
        raise SceneError(f"{what}: expected [x, y, z]")
    return [float(x) for x in j]


def _pose(j, what):
    if not isinstance(j, list) or len(j) != 6:
        raise SceneError(f"{what}: expected a 6-vector [tx, ty, tz, rx, ry, rz]")
    return [float(x) for x in j]


def _at(j, key):
    if not isinstance(j, dict) or key not in j:
        raise SceneError(f"scene schema error: missing key '{key}'")
    return j[key]


def _sdf_primitive(j, defaults: SmoothingConfig):
    t = _at(j, "type")
    if t == "superquadric":
        pose = _pose(j["pose"], "superquadric pose") if "pose" in j else [0.0] * 6
        return Superquadric(float(_at(j, "eps1")), float(_at(j, "eps2")), _vec3(_at(j, "axes"), "superquadric axes"),
                            pose)
    if t == "convex_polyhedron":
        planes = _at(j, "planes")
        return ConvexPolyhedron([_vec3(_at(p, "normal"), "plane normal") for p in planes],
                                [_vec3(_at(p, "point"), "plane point") for p in planes], float(j.get("tau", 1e-3)))
    if t == "box_planes":
        h = _vec3(_at(j, "half_extents"), "box_planes half_extents")
        normals, points = [], []
        for a in range(3):
            for sgn in (1.0, -1.0):
                n = [0.0, 0.0, 0.0]
                n[a] = sgn
                p = [0.0, 0.0, 0.0]
                p[a] = sgn * h[a]
                normals.append(n)
                points.append(p)
        return ConvexPolyhedron(normals, points, float(j.get("tau", 1e-3)))
    if t == "oriented_pointcloud":
        return OrientedPointcloud([_vec3(p, "pointcloud point") for p in _at(j, "points")],
                                  [_vec3(n, "pointcloud normal") for n in _at(j, "normals")],
                                  [float(x) for x in _at(j, "lengthscales")])
    if t == "union":
        return Union([_sdf_node(c, defaults) for c in _at(j, "children")], float(j.get("tau", defaults.tau_union)))
    if t == "subtraction":
        return Subtraction(_sdf_node(_at(j, "positive"), defaults), _sdf_node(_at(j, "negative"), defaults),
                           float(j.get("tau", defaults.tau_union)))
    raise SceneError(f"unknown sdf node type: {t}")


def _sdf_node(j, defaults):
    if isinstance(j, list):  # array shorthand: implicit union, single child collapses
        children = [_sdf_node(c, defaults) for c in j]
        return children[0] if len(children) == 1 else Union(children, defaults.tau_union)
    return _sdf_primitive(j, defaults)


def _mesh(j, base_dir):
    if "obj" in j:
        p = j["obj"]
        if not os.path.isabs(p):
            p = os.path.join(base_dir, p)
        try:
            text = open(p).read()
        except OSError as e:  # load_obj (src/mesh.cpp:117-121)
            raise SceneError(f"cannot open mesh file: {p}") from e
        return api.Mesh.parse_obj(text)
    if "box" in j:
        b = j["box"]
        return api.Mesh.box(_vec3(_at(b, "half_extents"), "box half_extents"), int(b.get("subdivisions", 1)),
                            bool(b.get("quad_edges", True)))
    raise SceneError("mesh: expected an 'obj' path or a 'box' generator")


_MODES = {"full": abi.MODE_FULL, "no-ee": abi.MODE_NO_EE, "one-sided": abi.MODE_ONE_SIDED}
_SMOOTH_KEYS = ("lambda", "tau_clip", "tau_min", "tau_comp", "tau_sign", "tau_pen", "tau_nn", "tau_clash",
                "tau_cont", "tau_topk_verts", "tau_topk_edges", "tau_normal", "tau_union", "hard_ops",
                "sphere_trace", "sphere_trace_iters", "containment_safeguard")


def _smoothing(j) -> SmoothingConfig:
    c = SmoothingConfig()
    if j is None:
        return c
    for k in _SMOOTH_KEYS:
        if k in j:
            setattr(c, "lambda_" if k == "lambda" else k, j[k])
    if "mode" in j:
        if j["mode"] not in _MODES:
            raise SceneError("mode must be one of: full, no-ee, one-sided")
        c.mode = _MODES[j["mode"]]
    api.validate_config(c)
    return c


def parse_scene(json_text: str, base_dir: str = ".") -> SceneDoc:
    """parse_scene (src/scene.cpp:130-172)."""
    try:
        doc = json.loads(json_text)
    except json.JSONDecodeError as e:
        raise SceneError(f"scene JSON parse error: {e}") from e
    smoothing = _smoothing(doc.get("smoothing") if isinstance(doc, dict) else None)
    bodies_j = doc.get("bodies") if isinstance(doc, dict) else None
    if not isinstance(bodies_j, list) or not bodies_j:
        raise SceneError("scene: needs a non-empty 'bodies' array")
    bodies = []
    for jb in bodies_j:
        name = jb.get("name", f"body{len(bodies)}")
        mesh = _mesh(_at(jb, "mesh"), base_dir)
        sdf = _sdf_node(_at(jb, "sdf"), smoothing)
        vk, ek = int(jb.get("vertex_topk", 0)), int(jb.get("edge_topk", 0))
        surface = api.Surface(mesh, sdf, vk, ek)
        pose = np.array(_pose(_at(jb, "pose"), "body pose"))
        mass = float(jb.get("mass", 1.0))
        if not mass > 0.0:
            raise SceneError("body mass must be positive")
        inertia = np.array(_vec3(jb["inertia"], "inertia")) if "inertia" in jb else np.zeros(3)
        bodies.append(SceneBody(name, surface, sdf, pose, mass, inertia, bool(jb.get("static", False)), vk, ek))
    return SceneDoc(bodies, smoothing)


def load_scene(path: str) -> SceneDoc:
    """load_scene (src/scene.cpp:174-181)."""
    try:
        text = open(path).read()
    except OSError as e:
        raise SceneError(f"cannot open scene file: {path}") from e
    return parse_scene(text, os.path.dirname(path))


# ---- text outputs ------------------------------------------------------------------
_KIND = {0: "VS", 1: "EE"}
_MODE_NAME = {abi.MODE_FULL: "full", abi.MODE_NO_EE: "no-ee", abi.MODE_ONE_SIDED: "one-sided"}


def _g17(x) -> str:
    """std::setprecision(17) << double: printf %.17g."""
    return format(float(x), ".17g")


def write_manifold_csv(f, contacts: np.ndarray, meta: np.ndarray) -> None:
    """write_manifold_csv (src/manifold_io.cpp:24-33), CSV schema v1. contacts
    [C, 8] (px, py, pz, dist, nx, ny, nz, activity), meta [C, 4] (kind, side,
    src_a, src_b)."""
    f.write("index,kind,side,src_a,src_b,px,py,pz,dist,nx,ny,nz,activity\n")
    for i, (c, m) in enumerate(zip(np.asarray(contacts, np.float64), np.asarray(meta))):
        f.write(f"{i},{_KIND[int(m[0])]},{int(m[1])},{int(m[2])},{int(m[3])}," + ",".join(_g17(x) for x in c) + "\n")


def manifold_to_json(contacts: np.ndarray, meta: np.ndarray, layout: dict) -> str:
    """manifold_to_json (src/manifold_io.cpp:35-52): nlohmann::json dump(2) --
    object keys sorted (std::map), shortest round-trip doubles."""
    rows = []
    for c, m in zip(np.asarray(contacts, np.float64), np.asarray(meta)):
        c = [float(x) for x in c]
        rows.append({"kind": _KIND[int(m[0])], "side": int(m[1]), "src_a": int(m[2]), "src_b": int(m[3]),
                     "point": c[0:3], "dist": c[3], "normal": c[4:7], "activity": c[7]})
    doc = {"layout": {"n1": int(layout["n1"]), "n2": int(layout["n2"]), "m1": int(layout["m1"]),
                      "m2": int(layout["m2"]), "mode": _MODE_NAME[int(layout["mode"])]},
           "contacts": rows}
    return json.dumps(doc, indent=2, sort_keys=True)


BENCH_CSV_VERSION = "cmg-bench-csv v1"


def write_bench_csv(f, records) -> None:
    """write_bench_csv (src/batch.cpp:122-129). records: dicts with kind,
    variant, batch, repetitions, median_s, std_s, throughput_qps."""
    f.write(f"# {BENCH_CSV_VERSION}\n")
    f.write("kind,variant,batch,repetitions,median_s,std_s,throughput_qps\n")
    for r in records:
        f.write(f"{r['kind']},{r['variant']},{int(r['batch'])},{int(r['repetitions'])},{_g6(r['median_s'])},"
                f"{_g6(r['std_s'])},{_g6(r['throughput_qps'])}\n")


def _g6(x) -> str:
    """default ostream << double: printf %g."""
    return format(float(x), "g")


def write_sweep_csv(f, ns: np.ndarray, l2: np.ndarray, smooth: np.ndarray) -> None:
    """write_sweep_csv (src/sweep.cpp:58-72); each input [n, 7] = theta, p1, dp1."""
    f.write("theta,ns_px,ns_py,ns_dpx,ns_dpy,l2_px,l2_py,l2_dpx,l2_dpy,smooth_px,smooth_py,"
            "smooth_dpx,smooth_dpy\n")
    for a, b, c in zip(ns, l2, smooth):
        vals = [a[0], a[1], a[2], a[4], a[5], b[1], b[2], b[4], b[5], c[1], c[2], c[4], c[5]]
        f.write(",".join(_g17(x) for x in vals) + "\n")
