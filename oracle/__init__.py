"""TEST INFRASTRUCTURE — Python bindings of the CPU checkers.

* ``Oracle`` wraps ``oracle/liboracle.so``: the plain-C restatement of the
  reference algorithm (cmg_oracle.c), pinned against the reference's golden
  vectors by tests/test_oracle_golden.py.
* ``Ref`` wraps ``oracle/_ref/libcmgref.so``: the unmodified reference sources
  compiled by oracle/Makefile (only present where it was built; it travels to
  the GPU box as a built artefact).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2602_20304_b200 import abi
from paper_2602_20304_b200.scene import SdfProgram, SmoothingConfig

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcmgref.so")

_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_P = C.c_void_p


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(_I32) if a is not None else None


def build(ref: bool = True) -> None:
    """Compile the checkers (the reference only where /root/reference exists)."""
    targets = ["oracle"]
    if ref and os.path.isdir(os.environ.get("CMG_REF", "/root/reference/proj")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _cfg(cfg):
    if cfg is None:
        cfg = SmoothingConfig()
    return cfg.to_c() if isinstance(cfg, SmoothingConfig) else cfg


# ---------------------------------------------------------------------------
class Oracle:
    """Plain-C restatement (double precision)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                build(ref=False)
            L = C.CDLL(ORACLE_SO)
            L.orc_surface_create.restype = _P
            L.orc_surface_create.argtypes = [_D, C.c_int32, _I32, C.c_int32,
                                             C.POINTER(abi.CmgbSdfNode), C.c_int32, C.c_int32, C.c_int32]
            L.orc_surface_destroy.argtypes = [_P]
            L.orc_surface_budgets.argtypes = [_P, _I32]
            L.orc_sdf_query.argtypes = [_P, C.c_int32, _D, C.c_int64, _D]
            L.orc_sphere_trace.argtypes = [_P, _D, _D, C.c_int64, C.c_int32, C.c_double, _D]
            L.orc_manifold.argtypes = [_P, _P, _D, _D, C.POINTER(abi.CmgbConfig), _D, _I32, _D, _I32]
            L.orc_manifold_batch.argtypes = [_P, _P, _D, C.c_int32, _D, C.c_int32, C.c_int64,
                                             C.POINTER(abi.CmgbConfig), C.c_int32, _D, _I32, _D, _D]
            L.orc_ee_witness.argtypes = [_D, C.c_int64, C.POINTER(abi.CmgbConfig), _D, _I32]
            L.orc_vf_witness.argtypes = [_D, C.c_int64, C.POINTER(abi.CmgbConfig), _D, _I32]
            L.orc_box_qp.argtypes = [_D, C.c_int64, C.POINTER(abi.CmgbConfig), _D]
            L.orc_se3_exp.argtypes = [_D, _D, _D]
            L.orc_soft_topk.argtypes = [_D, C.c_int32, C.c_int32, C.c_double, _D]
            L.orc_mt19937_64_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, _D]
            cls._lib = L
        return cls._lib

    class Surface:
        def __init__(self, vertices, edges, sdf_root, vertex_topk=0, edge_topk=0):
            L = Oracle.lib()
            self.vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
            self.edges = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
            self.prog = SdfProgram(sdf_root)
            self.h = L.orc_surface_create(_dp(self.vertices), len(self.vertices), _ip(self.edges),
                                          len(self.edges), self.prog.array, self.prog.n,
                                          vertex_topk, edge_topk)
            if not self.h:
                raise ValueError("oracle: bad surface program")

        def __del__(self):
            if getattr(self, "h", None):
                Oracle.lib().orc_surface_destroy(self.h)
                self.h = None

        def budgets(self):
            out = np.zeros(3, np.int32)
            Oracle.lib().orc_surface_budgets(self.h, _ip(out))
            return out

        def sdf_query(self, flavor, pts):
            pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
            out = np.zeros((len(pts), 4))
            Oracle.lib().orc_sdf_query(self.h, flavor, _dp(pts), len(pts), _dp(out))
            return out

        def sphere_trace(self, pose, pts, iters, tau=1e-9):
            pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
            pose = np.ascontiguousarray(pose, dtype=np.float64)
            out = np.zeros_like(pts)
            Oracle.lib().orc_sphere_trace(self.h, _dp(pose), _dp(pts), len(pts), iters, tau, _dp(out))
            return out

    @staticmethod
    def manifold(s1, s2, pose1, pose2, cfg=None):
        L = Oracle.lib()
        c = _cfg(cfg)
        p1 = np.ascontiguousarray(pose1, dtype=np.float64)
        p2 = np.ascontiguousarray(pose2, dtype=np.float64)
        layout = np.zeros(5, np.int32)
        L.orc_manifold(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c), None, None, None, _ip(layout))
        n = int(layout[4])
        m = int(layout[2] * layout[3])
        contacts = np.zeros((n, 8))
        meta = np.zeros((n, 4), np.int32)
        ee = np.zeros((9, max(m, 1)))
        L.orc_manifold(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c), _dp(contacts), _ip(meta), _dp(ee),
                       _ip(layout))
        return dict(contacts=contacts, meta=meta, ee=ee[:, :m], layout=layout)

    @staticmethod
    def manifold_batch(s1, s2, poses1, poses2, cfg=None, threads=None, want_meta=True,
                       want_ee=False):
        L = Oracle.lib()
        c = _cfg(cfg)
        poses1 = np.ascontiguousarray(poses1, dtype=np.float64).reshape(-1, 6)
        poses2 = np.ascontiguousarray(poses2, dtype=np.float64).reshape(-1, 6)
        n_env = max(len(poses1), len(poses2))
        st1 = 1 if len(poses1) == n_env else 0
        st2 = 1 if len(poses2) == n_env else 0
        layout = np.zeros(5, np.int32)
        L.orc_manifold(s1.h, s2.h, _dp(poses1), _dp(poses2), C.byref(c), None, None, None, _ip(layout))
        per = int(layout[4])
        m = int(layout[2] * layout[3])
        contacts = np.zeros((n_env, per, 8))
        meta = np.zeros((n_env, per, 4), np.int32) if want_meta else None
        ee = np.zeros((n_env, 9, m)) if want_ee else None
        mean = np.zeros(n_env)
        L.orc_manifold_batch(s1.h, s2.h, _dp(poses1), st1, _dp(poses2), st2, n_env, C.byref(c),
                             threads or os.cpu_count() or 1, _dp(contacts), _ip(meta), _dp(ee),
                             _dp(mean))
        return dict(contacts=contacts, meta=meta, ee=ee, mean_dist=mean, layout=layout)

    @staticmethod
    def ee_witness(pairs, cfg=None):
        pairs = np.ascontiguousarray(pairs, dtype=np.float64).reshape(-1, 12)
        out = np.zeros((len(pairs), 9))
        labels = np.zeros(len(pairs), np.int32)
        c = _cfg(cfg)
        Oracle.lib().orc_ee_witness(_dp(pairs), len(pairs), C.byref(c), _dp(out), _ip(labels))
        return out, labels

    @staticmethod
    def vf_witness(pairs, cfg=None):
        pairs = np.ascontiguousarray(pairs, dtype=np.float64).reshape(-1, 12)
        out = np.zeros((len(pairs), 3))
        labels = np.zeros(len(pairs), np.int32)
        c = _cfg(cfg)
        Oracle.lib().orc_vf_witness(_dp(pairs), len(pairs), C.byref(c), _dp(out), _ip(labels))
        return out, labels

    @staticmethod
    def box_qp(qp, cfg=None):
        qp = np.ascontiguousarray(qp, dtype=np.float64).reshape(-1, 5)
        out = np.zeros((len(qp), 3))
        c = _cfg(cfg)
        Oracle.lib().orc_box_qp(_dp(qp), len(qp), C.byref(c), _dp(out))
        return out

    @staticmethod
    def se3_exp(pose):
        pose = np.ascontiguousarray(pose, dtype=np.float64)
        R = np.zeros(9)
        t = np.zeros(3)
        Oracle.lib().orc_se3_exp(_dp(pose), _dp(R), _dp(t))
        return R.reshape(3, 3), t

    @staticmethod
    def soft_topk(xs, k, tau):
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        w = np.zeros((k, len(xs)))
        if Oracle.lib().orc_soft_topk(_dp(xs), len(xs), k, tau, _dp(w)) != 0:
            raise ValueError("soft_topk: require 1 <= K <= D")
        return w

    @staticmethod
    def uniform(seed, n, lo=0.0, hi=1.0):
        """std::mt19937_64(seed) + uniform_real_distribution<double>(lo, hi)."""
        out = np.zeros(n)
        Oracle.lib().orc_mt19937_64_uniform(seed, n, lo, hi, _dp(out))
        return out


# ---------------------------------------------------------------------------
class Ref:
    """The compiled reference (oracle/_ref/libcmgref.so)."""

    _lib = None

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference)")
            L = C.CDLL(REF_SO)
            L.cmgref_last_error.restype = C.c_char_p
            L.cmgref_mesh_box.restype = _P
            L.cmgref_mesh_box.argtypes = [_D, C.c_int, C.c_int]
            L.cmgref_mesh_parse_obj.restype = _P
            L.cmgref_mesh_parse_obj.argtypes = [C.c_char_p, _I32]
            L.cmgref_mesh_arrays.restype = _P
            L.cmgref_mesh_arrays.argtypes = [_D, C.c_int, _I32, C.c_int, _I32, C.c_int]
            L.cmgref_mesh_sizes.argtypes = [_P, _I32, _I32, _I32, _I32]
            L.cmgref_mesh_read.argtypes = [_P, _D, _I32, _I32]
            L.cmgref_mesh_warning.restype = C.c_char_p
            L.cmgref_mesh_warning.argtypes = [_P, C.c_int]
            L.cmgref_mesh_destroy.argtypes = [_P]
            L.cmgref_surface_create.restype = _P
            L.cmgref_surface_create.argtypes = [_P, C.POINTER(abi.CmgbSdfNode), C.c_int, C.c_int,
                                                C.c_int, C.c_double]
            L.cmgref_surface_destroy.argtypes = [_P]
            L.cmgref_surface_info.argtypes = [_P, _I32]
            L.cmgref_surface_warning.restype = C.c_char_p
            L.cmgref_surface_warning.argtypes = [_P, C.c_int]
            L.cmgref_sdf_query.argtypes = [_P, C.c_int, _D, C.c_int64, _D]
            L.cmgref_sphere_trace.argtypes = [_P, _D, _D, C.c_int64, C.c_int, C.c_double, _D]
            L.cmgref_manifold.argtypes = [_P, _P, _D, _D, C.POINTER(abi.CmgbConfig), _D, _I32, _D, _I32]
            L.cmgref_manifold_batch.argtypes = [_P, _P, _D, C.c_int, _D, C.c_int, C.c_int64,
                                                C.POINTER(abi.CmgbConfig), C.c_int, _D, _I32, _D]
            L.cmgref_manifold_jvp.argtypes = [_P, _P, _D, _D, C.POINTER(abi.CmgbConfig), _D, _D, _D]
            L.cmgref_random_pairs.argtypes = [C.c_int64, C.c_uint64, _D]
            L.cmgref_sweep.argtypes = [C.c_int, C.c_int, _D]
            L.cmgref_sweep_csv.argtypes = [C.c_int, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
            L.cmgref_scene_parse.restype = _P
            L.cmgref_scene_parse.argtypes = [C.c_char_p, C.c_char_p]
            L.cmgref_scene_destroy.argtypes = [_P]
            L.cmgref_scene_n_bodies.argtypes = [_P]
            L.cmgref_scene_body.restype = _P
            L.cmgref_scene_body.argtypes = [_P, C.c_int, _D, _D, _D, _I32, _I32, C.c_char_p, C.c_int]
            L.cmgref_scene_smoothing.argtypes = [_P, C.POINTER(abi.CmgbConfig)]
            L.cmgref_manifold_text.argtypes = [_P, _P, _D, _D, C.POINTER(abi.CmgbConfig), C.c_int, C.c_char_p,
                                               C.c_int64, C.POINTER(C.c_int64)]
            L.cmgref_demo_run.restype = C.c_int
            L.cmgref_demo_run.argtypes = [C.POINTER(_P), C.c_int, _I32, _D, _D, _D, _D, C.POINTER(abi.CmgbConfig),
                                          C.POINTER(abi.CmgbDemoParams), C.c_double, C.c_int, _D, _D, _D, _D]
            L.cmgref_ee_batch.restype = C.c_double
            L.cmgref_ee_batch.argtypes = [_D, C.c_int64, C.POINTER(abi.CmgbConfig), C.c_int, _D]
            L.cmgref_vf_batch.restype = C.c_double
            L.cmgref_vf_batch.argtypes = [_D, C.c_int64, C.POINTER(abi.CmgbConfig), C.c_int, _D]
            L.cmgref_ee_witness_full.argtypes = [_D, C.c_int64, C.POINTER(abi.CmgbConfig), _D]
            L.cmgref_box_qp.argtypes = [_D, C.c_int64, C.POINTER(abi.CmgbConfig), _D]
            L.cmgref_bench_manifold.argtypes = [_P, _P, _D, _D, C.POINTER(abi.CmgbConfig), C.c_int64,
                                                C.c_char_p, C.c_uint64, C.c_int, C.c_int, _D, _D]
            L.cmgref_bench_witness.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_uint64, C.c_int,
                                               C.c_int, _D, _D]
            L.cmgref_se3_exp.argtypes = [_D, _D, _D]
            L.cmgref_so3_log.argtypes = [_D, _D]
            L.cmgref_so3_exp.argtypes = [_D, _D]
            L.cmgref_soft_topk.argtypes = [_D, C.c_int, C.c_int, C.c_double, _D]
            L.cmgref_config_validate.argtypes = [C.POINTER(abi.CmgbConfig)]
            L.cmgref_opcount_manifold.argtypes = [_P, _P, _D, _D, C.POINTER(abi.CmgbConfig), C.c_int,
                                                  C.POINTER(C.c_int64)]
            L.cmgref_scene_bench.argtypes = [C.POINTER(_P), C.c_int, _I32, C.c_int, _D, C.c_int64,
                                             C.POINTER(abi.CmgbConfig), C.c_int, C.c_int, C.c_int, C.c_int,
                                             _D, _D, _D]
            cls._lib = L
        return cls._lib

    @staticmethod
    def err():
        return Ref.lib().cmgref_last_error().decode()

    class Mesh:
        def __init__(self, h):
            self.h = h
            L = Ref.lib()
            nv, nf, ne, nw = (C.c_int32() for _ in range(4))
            L.cmgref_mesh_sizes(h, C.byref(nv), C.byref(nf), C.byref(ne), C.byref(nw))
            self.vertices = np.zeros((nv.value, 3))
            self.faces = np.zeros((nf.value, 3), np.int32)
            self.edges = np.zeros((ne.value, 2), np.int32)
            L.cmgref_mesh_read(h, _dp(self.vertices), _ip(self.faces), _ip(self.edges))
            self.warnings = [L.cmgref_mesh_warning(h, i).decode() for i in range(nw.value)]

        @staticmethod
        def box(half, subdivisions=1, quad_edges=True):
            h = np.ascontiguousarray(half, dtype=np.float64)
            m = Ref.lib().cmgref_mesh_box(_dp(h), subdivisions, int(quad_edges))
            if not m:
                raise ValueError(Ref.err())
            return Ref.Mesh(m)

        @staticmethod
        def parse_obj(text):
            line = C.c_int32(0)
            m = Ref.lib().cmgref_mesh_parse_obj(text.encode(), C.byref(line))
            if not m:
                raise ValueError(f"{Ref.err()}|{line.value}")
            return Ref.Mesh(m)

        @staticmethod
        def arrays(v, f, e):
            v = np.ascontiguousarray(v, dtype=np.float64)
            f = np.ascontiguousarray(f, dtype=np.int32)
            e = np.ascontiguousarray(e, dtype=np.int32)
            return Ref.Mesh(Ref.lib().cmgref_mesh_arrays(_dp(v), len(v), _ip(f), len(f), _ip(e), len(e)))

        def __del__(self):
            if getattr(self, "h", None):
                Ref.lib().cmgref_mesh_destroy(self.h)
                self.h = None

    class Surface:
        def __init__(self, mesh, sdf_root, vertex_topk=0, edge_topk=0, tol=1e-2):
            self.mesh = mesh
            self.prog = SdfProgram(sdf_root)
            self.h = Ref.lib().cmgref_surface_create(mesh.h, self.prog.array, self.prog.n,
                                                     vertex_topk, edge_topk, tol)
            if not self.h:
                raise ValueError(Ref.err())
            info = np.zeros(6, np.int32)
            Ref.lib().cmgref_surface_info(self.h, _ip(info))
            self.info = info
            self.warnings = [Ref.lib().cmgref_surface_warning(self.h, i).decode()
                             for i in range(int(info[5]))]

        def __del__(self):
            if getattr(self, "h", None) and getattr(self, "_owned", True):
                Ref.lib().cmgref_surface_destroy(self.h)
                self.h = None

        def sdf_query(self, flavor, pts):
            pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
            out = np.zeros((len(pts), 4))
            Ref.lib().cmgref_sdf_query(self.h, flavor, _dp(pts), len(pts), _dp(out))
            return out

        def sphere_trace(self, pose, pts, iters, tau=1e-9):
            pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
            pose = np.ascontiguousarray(pose, dtype=np.float64)
            out = np.zeros_like(pts)
            Ref.lib().cmgref_sphere_trace(self.h, _dp(pose), _dp(pts), len(pts), iters, tau, _dp(out))
            return out

    @staticmethod
    def manifold(s1, s2, pose1, pose2, cfg=None):
        L = Ref.lib()
        c = _cfg(cfg)
        p1 = np.ascontiguousarray(pose1, dtype=np.float64)
        p2 = np.ascontiguousarray(pose2, dtype=np.float64)
        layout = np.zeros(5, np.int32)
        if L.cmgref_manifold(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c), None, None, None, _ip(layout)):
            raise ValueError(Ref.err())
        n = int(layout[4])
        m = int(layout[2] * layout[3])
        contacts = np.zeros((n, 8))
        meta = np.zeros((n, 4), np.int32)
        ee = np.zeros((9, max(m, 1)))
        L.cmgref_manifold(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c), _dp(contacts), _ip(meta), _dp(ee),
                          _ip(layout))
        return dict(contacts=contacts, meta=meta, ee=ee[:, :m], layout=layout)

    @staticmethod
    def manifold_batch(s1, s2, poses1, poses2, cfg=None, workers=None):
        L = Ref.lib()
        c = _cfg(cfg)
        poses1 = np.ascontiguousarray(poses1, dtype=np.float64).reshape(-1, 6)
        poses2 = np.ascontiguousarray(poses2, dtype=np.float64).reshape(-1, 6)
        n_env = max(len(poses1), len(poses2))
        st1 = 1 if len(poses1) == n_env else 0
        st2 = 1 if len(poses2) == n_env else 0
        one = Ref.manifold(s1, s2, poses1[0], poses2[0], cfg)
        per = int(one["layout"][4])
        contacts = np.zeros((n_env, per, 8))
        meta = np.zeros((n_env, per, 4), np.int32)
        mean = np.zeros(n_env)
        if L.cmgref_manifold_batch(s1.h, s2.h, _dp(poses1), st1, _dp(poses2), st2, n_env, C.byref(c),
                                   workers or os.cpu_count() or 1, _dp(contacts), _ip(meta), _dp(mean)):
            raise ValueError(Ref.err())
        return dict(contacts=contacts, meta=meta, mean_dist=mean, layout=one["layout"])

    @staticmethod
    def manifold_jvp(s1, s2, pose1, pose2, cfg=None):
        L = Ref.lib()
        c = _cfg(cfg)
        n = int(Ref.manifold(s1, s2, pose1, pose2, cfg)["layout"][4])
        p1 = np.ascontiguousarray(pose1, dtype=np.float64)
        p2 = np.ascontiguousarray(pose2, dtype=np.float64)
        contacts = np.zeros((n, 8))
        tangents = np.zeros((n, 8, 12))
        md = np.zeros(13)
        if L.cmgref_manifold_jvp(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c), _dp(contacts),
                                 _dp(tangents), _dp(md)):
            raise ValueError(Ref.err())
        return dict(contacts=contacts, tangents=tangents, mean_dist=md[0], mean_dist_grad=md[1:])

    @staticmethod
    def demo_run(surfaces, is_static, mass, inertia, poses, vels, cfg=None, params=None, dt=1e-3, steps=1):
        """DemoSim (src/demosim.cpp) from a state: per-step poses / velocities
        [steps, n, 6], deepest_penetration [steps], kinetic_energy [steps]."""
        from paper_2602_20304_b200.scene import PenaltyParams

        L = Ref.lib()
        n = len(surfaces)
        hs = (_P * n)(*[s.h for s in surfaces])
        st = np.ascontiguousarray(is_static, dtype=np.int32)
        m = np.ascontiguousarray(mass, dtype=np.float64)
        I = np.ascontiguousarray(inertia, dtype=np.float64).reshape(n, 3)
        P = np.ascontiguousarray(poses, dtype=np.float64).reshape(n, 6)
        V = np.ascontiguousarray(vels, dtype=np.float64).reshape(n, 6)
        po = np.zeros((steps, n, 6))
        vo = np.zeros((steps, n, 6))
        de = np.zeros(steps)
        ke = np.zeros(steps)
        c = _cfg(cfg)
        pp = (params or PenaltyParams()).to_c()
        done = L.cmgref_demo_run(hs, n, _ip(st), _dp(m), _dp(I), _dp(P), _dp(V), C.byref(c), C.byref(pp), dt, steps,
                                 _dp(po), _dp(vo), _dp(de), _dp(ke))
        if done < 0:
            raise ValueError(Ref.err())
        return dict(poses=po[:done], velocities=vo[:done], deepest=de[:done], kinetic_energy=ke[:done])

    @staticmethod
    def sweep(variant, n):
        """rotating_edge_sweep (src/sweep.cpp:44-56): [n, 7] theta, p1, dp1/dtheta."""
        out = np.zeros((n, 7))
        if Ref.lib().cmgref_sweep(variant, n, _dp(out)):
            raise ValueError(Ref.err())
        return out

    @staticmethod
    def _text(call):
        n = C.c_int64()
        call(None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        if call(buf, n.value + 1, C.byref(n)):
            raise ValueError(Ref.err())
        return buf.value.decode()

    @staticmethod
    def sweep_csv(n):
        L = Ref.lib()
        return Ref._text(lambda b, cap, ln: L.cmgref_sweep_csv(n, b, cap, ln))

    @staticmethod
    def manifold_text(s1, s2, pose1, pose2, cfg=None, as_json=False):
        """write_manifold_csv / manifold_to_json (src/manifold_io.cpp) of one manifold."""
        L = Ref.lib()
        c = _cfg(cfg)
        p1 = np.ascontiguousarray(pose1, dtype=np.float64)
        p2 = np.ascontiguousarray(pose2, dtype=np.float64)
        return Ref._text(lambda b, cap, ln: L.cmgref_manifold_text(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c),
                                                                   int(as_json), b, cap, ln))

    class SceneHandle:
        """A parse_scene result (src/scene.cpp:130-172); body surfaces are owned
        by the scene (SurfaceModel handles usable wherever Ref.Surface is)."""

        def __init__(self, json_text, base_dir="."):
            L = Ref.lib()
            self.h = L.cmgref_scene_parse(json_text.encode(), base_dir.encode())
            if not self.h:
                raise ValueError(Ref.err())
            self.bodies = []
            for i in range(L.cmgref_scene_n_bodies(self.h)):
                pose, mass, inertia = np.zeros(6), np.zeros(1), np.zeros(3)
                st, topk = np.zeros(1, np.int32), np.zeros(2, np.int32)
                name = C.create_string_buffer(256)
                sh = L.cmgref_scene_body(self.h, i, _dp(pose), _dp(mass), _dp(inertia), _ip(st), _ip(topk), name, 256)
                surf = Ref.Surface.__new__(Ref.Surface)
                surf.h, surf._owned = sh, False
                self.bodies.append(dict(name=name.value.decode(), pose=pose, mass=float(mass[0]), inertia=inertia,
                                        is_static=bool(st[0]), vertex_topk=int(topk[0]), edge_topk=int(topk[1]),
                                        surface=surf))
            c = abi.CmgbConfig()
            L.cmgref_scene_smoothing(self.h, C.byref(c))
            self.smoothing = c

        def __del__(self):
            if getattr(self, "h", None):
                Ref.lib().cmgref_scene_destroy(self.h)
                self.h = None

    @staticmethod
    def random_pairs(n, seed=0):
        out = np.zeros((n, 12))
        Ref.lib().cmgref_random_pairs(n, seed, _dp(out))
        return out

    @staticmethod
    def ee_witness_full(pairs, cfg=None):
        pairs = np.ascontiguousarray(pairs, dtype=np.float64).reshape(-1, 12)
        out = np.zeros((len(pairs), 9))
        c = _cfg(cfg)
        Ref.lib().cmgref_ee_witness_full(_dp(pairs), len(pairs), C.byref(c), _dp(out))
        return out

    @staticmethod
    def vf_batch(pairs, cfg=None, workers=1):
        pairs = np.ascontiguousarray(pairs, dtype=np.float64).reshape(-1, 12)
        out = np.zeros((len(pairs), 3))
        c = _cfg(cfg)
        cs = Ref.lib().cmgref_vf_batch(_dp(pairs), len(pairs), C.byref(c), workers, _dp(out))
        return out, cs

    @staticmethod
    def ee_batch(pairs, cfg=None, workers=1):
        pairs = np.ascontiguousarray(pairs, dtype=np.float64).reshape(-1, 12)
        out = np.zeros((len(pairs), 6))
        c = _cfg(cfg)
        cs = Ref.lib().cmgref_ee_batch(_dp(pairs), len(pairs), C.byref(c), workers, _dp(out))
        return out, cs

    @staticmethod
    def box_qp(qp, cfg=None):
        qp = np.ascontiguousarray(qp, dtype=np.float64).reshape(-1, 5)
        out = np.zeros((len(qp), 3))
        c = _cfg(cfg)
        Ref.lib().cmgref_box_qp(_dp(qp), len(qp), C.byref(c), _dp(out))
        return out

    @staticmethod
    def bench_manifold(s1, s2, pose1, pose2, batch, variant="ours", cfg=None, seed=0, reps=3,
                       workers=None):
        c = _cfg(cfg)
        p1 = np.ascontiguousarray(pose1, dtype=np.float64)
        p2 = np.ascontiguousarray(pose2, dtype=np.float64)
        med, sd = C.c_double(), C.c_double()
        if Ref.lib().cmgref_bench_manifold(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c), batch,
                                           variant.encode(), seed, reps, workers or os.cpu_count(),
                                           C.byref(med), C.byref(sd)):
            raise ValueError(Ref.err())
        return med.value, sd.value

    OPCOUNT_KINDS = ("arith", "pow", "sqrt", "exp", "log", "tanh", "other")

    @staticmethod
    def opcount_manifold(s1, s2, pose1, pose2, cfg=None, jvp=False) -> dict:
        """SURVEY Appendix B's op counter: the reference's generate_manifold<T>
        with a counting scalar (jvp: Dual<12, counting scalar>). W = arith +
        every transcendental, 1 op each."""
        c = _cfg(cfg)
        p1 = np.ascontiguousarray(pose1, dtype=np.float64).reshape(6)
        p2 = np.ascontiguousarray(pose2, dtype=np.float64).reshape(6)
        out = (C.c_int64 * 7)()
        Ref.lib().cmgref_opcount_manifold(s1.h, s2.h, _dp(p1), _dp(p2), C.byref(c), int(bool(jvp)), out)
        d = {k: int(out[i]) for i, k in enumerate(Ref.OPCOUNT_KINDS)}
        d["transcendental"] = sum(d[k] for k in Ref.OPCOUNT_KINDS[1:])
        d["W"] = d["arith"] + d["transcendental"]
        return d

    @staticmethod
    def scene_bench(surfaces, pairs, poses, cfg=None, jvp=False, reps=3, warmups=1, workers=None):
        """Config D's CPU reference: every pair of every env through
        generate_manifold<double> / <Dual12>, std::thread chunks, time_run
        median / std (s). poses [n_env, n_bodies, 6]."""
        c = _cfg(cfg)
        P = np.ascontiguousarray(poses, dtype=np.float64)
        pr = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        hs = (_P * len(surfaces))(*[s.h for s in surfaces])
        med, sd, cs = C.c_double(), C.c_double(), C.c_double()
        if Ref.lib().cmgref_scene_bench(hs, len(surfaces), _ip(pr), len(pr), _dp(P), P.shape[0], C.byref(c),
                                        int(bool(jvp)), reps, warmups, workers or os.cpu_count(),
                                        C.byref(med), C.byref(sd), C.byref(cs)):
            raise ValueError(Ref.err())
        return med.value, sd.value, cs.value

    @staticmethod
    def bench_witness(kind, batch, variant="ours", seed=0, reps=3, workers=None):
        med, sd = C.c_double(), C.c_double()
        if Ref.lib().cmgref_bench_witness(kind.encode(), batch, variant.encode(), seed, reps,
                                          workers or os.cpu_count(), C.byref(med), C.byref(sd)):
            raise ValueError(Ref.err())
        return med.value, sd.value

    @staticmethod
    def se3_exp(pose):
        pose = np.ascontiguousarray(pose, dtype=np.float64)
        R = np.zeros(9)
        t = np.zeros(3)
        Ref.lib().cmgref_se3_exp(_dp(pose), _dp(R), _dp(t))
        return R.reshape(3, 3), t

    @staticmethod
    def so3_log(R):
        R = np.ascontiguousarray(R, dtype=np.float64).reshape(9)
        w = np.zeros(3)
        Ref.lib().cmgref_so3_log(_dp(R), _dp(w))
        return w

    @staticmethod
    def so3_exp(w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        R = np.zeros(9)
        Ref.lib().cmgref_so3_exp(_dp(w), _dp(R))
        return R.reshape(3, 3)

    @staticmethod
    def soft_topk(xs, k, tau):
        xs = np.ascontiguousarray(xs, dtype=np.float64)
        w = np.zeros((k, len(xs)))
        if Ref.lib().cmgref_soft_topk(_dp(xs), len(xs), k, tau, _dp(w)):
            raise ValueError(Ref.err())
        return w
