"""Host-side descriptors mirroring the reference's C++ types.

* ``SmoothingConfig``  — cmg::SmoothingConfig (include/cmg/config.hpp:17-74) and
  ``config_for_variant`` (src/batch.cpp:131-150).
* SDF primitives / composition — SuperquadricParams, ConvexPolyhedronParams,
  OrientedPointcloudParams, SmoothSdf::smooth_union / ::subtraction
  (include/cmg/sdf.hpp:35-202), flattened to the postfix ``cmgb_sdf_node``
  program of include/cmgb.h. ``box_planes`` is the scene-loader convenience of
  src/scene.cpp:49-62.

These are plain descriptors (no device work); surfaces are created by the
native library (see ``surface.py``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields
from typing import List, Sequence

import numpy as np

from . import abi


@dataclass
class SmoothingConfig:
    lambda_: float = 0.01
    tau_clip: float = 0.1
    tau_min: float = 0.1
    tau_comp: float = 0.1
    tau_sign: float = 0.1
    tau_pen: float = 0.01
    tau_nn: float = 0.01
    tau_clash: float = 0.1
    tau_cont: float = 0.01
    tau_topk_verts: float = 0.01
    tau_topk_edges: float = 0.01
    tau_normal: float = 1e-9
    tau_union: float = 0.01
    hard_ops: bool = False
    sphere_trace: bool = True
    sphere_trace_iters: int = 5
    containment_safeguard: bool = False
    mode: int = abi.MODE_FULL

    kEdgeNormalEps = 1e-12  # config.hpp:46

    @staticmethod
    def no_smoothing() -> "SmoothingConfig":
        """config.hpp:48-53."""
        return SmoothingConfig(lambda_=1e-6, hard_ops=True)

    def for_variant(self, variant: str) -> "SmoothingConfig":
        """config_for_variant (src/batch.cpp:131-150)."""
        c = SmoothingConfig(**{f.name: getattr(self, f.name) for f in fields(self)})
        if variant == "ours":
            c.hard_ops, c.mode = False, abi.MODE_FULL
        elif variant == "ours_ns":
            c.hard_ops, c.lambda_, c.mode = True, 1e-6, abi.MODE_FULL
        elif variant == "ours_ne":
            c.hard_ops, c.mode = False, abi.MODE_NO_EE
        elif variant == "ours_ne_s":
            c.hard_ops, c.mode = False, abi.MODE_ONE_SIDED
        else:
            raise ValueError(
                f"unknown variant: {variant} (expected ours|ours_ns|ours_ne|ours_ne_s)"
            )
        return c

    def to_c(self) -> abi.CmgbConfig:
        c = abi.CmgbConfig()
        for f in fields(self):
            v = getattr(self, f.name)
            setattr(c, f.name, int(v) if f.name in _INT_FIELDS else float(v))
        c.reserved = 0
        return c


_INT_FIELDS = {"hard_ops", "sphere_trace", "sphere_trace_iters", "containment_safeguard", "mode"}


# ---------------------------------------------------------------------------
# SDF program
# ---------------------------------------------------------------------------
@dataclass
class PenaltyParams:
    """cmg::PenaltyParams (include/cmg/demosim.hpp:24-31)."""

    stiffness: float = 1e4
    damping: float = 100.0
    friction: float = 0.5
    friction_viscous: float = 100.0
    tau_force: float = 1e-4
    gravity: tuple = (0.0, 0.0, -9.81)

    def to_c(self) -> abi.CmgbDemoParams:
        c = abi.CmgbDemoParams()
        for f in ("stiffness", "damping", "friction", "friction_viscous", "tau_force"):
            setattr(c, f, float(getattr(self, f)))
        for k in range(3):
            c.gravity[k] = float(self.gravity[k])
        return c


class SdfNode:
    """Base: ``postfix()`` returns this subtree's nodes in postfix order."""

    def postfix(self) -> List["SdfNode"]:
        return [self]

    def leaf_count(self) -> int:
        return 1


@dataclass
class Superquadric(SdfNode):
    eps1: float = 1.0
    eps2: float = 1.0
    axes: Sequence[float] = (1.0, 1.0, 1.0)
    pose: Sequence[float] = (0.0, 0.0, 0.0, 0.0, 0.0, 0.0)


@dataclass
class ConvexPolyhedron(SdfNode):
    normals: np.ndarray = None
    points: np.ndarray = None
    tau: float = 1e-3


def box_planes(half_extents: Sequence[float], tau: float = 1e-3) -> ConvexPolyhedron:
    """The six half-space planes of an axis-aligned box (src/scene.cpp:49-62)."""
    normals, points = [], []
    for a in range(3):
        for s in (1.0, -1.0):
            n = [0.0, 0.0, 0.0]
            n[a] = s
            p = [0.0, 0.0, 0.0]
            p[a] = s * half_extents[a]
            normals.append(n)
            points.append(p)
    return ConvexPolyhedron(np.array(normals, dtype=np.float64), np.array(points, dtype=np.float64), tau)


@dataclass
class OrientedPointcloud(SdfNode):
    points: np.ndarray = None
    normals: np.ndarray = None
    lengthscales: np.ndarray = None


@dataclass
class Union(SdfNode):
    children: List[SdfNode] = field(default_factory=list)
    tau: float = 0.01

    def postfix(self):
        out = []
        for c in self.children:
            out += c.postfix()
        return out + [self]

    def leaf_count(self):
        return sum(c.leaf_count() for c in self.children)


@dataclass
class Subtraction(SdfNode):
    positive: SdfNode = None
    negative: SdfNode = None
    tau: float = 0.01

    def postfix(self):
        return self.positive.postfix() + self.negative.postfix() + [self]

    def leaf_count(self):
        return self.positive.leaf_count() + self.negative.leaf_count()


class SdfProgram:
    """ctypes array of cmgb_sdf_node for a tree; keeps numpy buffers alive."""

    def __init__(self, root: SdfNode):
        self.root = root
        nodes = root.postfix()
        self.n = len(nodes)
        self.array = (abi.CmgbSdfNode * self.n)()
        self._keep = []
        for i, nd in enumerate(nodes):
            c = self.array[i]
            if isinstance(nd, Superquadric):
                c.op = abi.SDF_SUPERQUADRIC
                c.count = 0
                c.eps1, c.eps2 = float(nd.eps1), float(nd.eps2)
                for k in range(3):
                    c.axes[k] = float(nd.axes[k])
                for k in range(6):
                    c.pose[k] = float(nd.pose[k])
            elif isinstance(nd, ConvexPolyhedron):
                c.op = abi.SDF_CONVEX_POLYHEDRON
                n = np.ascontiguousarray(nd.normals, dtype=np.float64).reshape(-1, 3)
                p = np.ascontiguousarray(nd.points, dtype=np.float64).reshape(-1, 3)
                c.count = n.shape[0]
                c.tau = float(nd.tau)
                c.normals = n.ctypes.data_as(C.POINTER(C.c_double))
                c.points = p.ctypes.data_as(C.POINTER(C.c_double))
                self._keep += [n, p]
            elif isinstance(nd, OrientedPointcloud):
                c.op = abi.SDF_ORIENTED_POINTCLOUD
                n = np.ascontiguousarray(nd.normals, dtype=np.float64).reshape(-1, 3)
                p = np.ascontiguousarray(nd.points, dtype=np.float64).reshape(-1, 3)
                t = np.ascontiguousarray(nd.lengthscales, dtype=np.float64).reshape(-1)
                c.count = n.shape[0]
                c.normals = n.ctypes.data_as(C.POINTER(C.c_double))
                c.points = p.ctypes.data_as(C.POINTER(C.c_double))
                c.lengthscales = t.ctypes.data_as(C.POINTER(C.c_double))
                self._keep += [n, p, t]
            elif isinstance(nd, Union):
                c.op = abi.SDF_UNION
                c.count = len(nd.children)
                c.tau = float(nd.tau)
            elif isinstance(nd, Subtraction):
                c.op = abi.SDF_SUBTRACTION
                c.count = 2
                c.tau = float(nd.tau)
            else:
                raise TypeError(f"unknown SDF node {nd!r}")
