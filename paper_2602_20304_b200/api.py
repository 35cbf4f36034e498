"""Python mirror of the reference C++ collision API over the C ABI (libcmgb.so).

Reference interface -> this module:
  make_box_mesh / parse_obj (src/mesh.cpp)          -> Mesh.box / Mesh.parse_obj
  build_surface (src/surface.cpp:9-44)               -> Surface(...)
  generate_manifold<double> (manifold.hpp:336-377)   -> generate_manifold (one env)
  bench_manifold's per-env loop (batch.cpp:207-215)  -> generate_manifold_batch (device tensors)
  run_ee_batch / run_vf_batch (batch.cpp:53-98)      -> run_ee_batch / run_vf_batch
Errors mirror the reference's exceptions: ValueError for std::invalid_argument,
MeshParseError for cmg::MeshParseError.

Device memory and streams come from PyTorch; every compute call goes through
the native library (no CPU path exists).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import abi
from .scene import SdfNode, SdfProgram, SmoothingConfig


class MeshParseError(ValueError):
    def __init__(self, message: str, line: int):
        super().__init__(message)
        self.line_number = line


def _raise(status: int):
    lib = abi.load()
    msg = (lib.cmgb_last_error() or b"").decode()
    if status == 1:
        raise ValueError(msg)
    raise abi.CmgbError(status, msg)


def _ok(status: int):
    if status != abi.CMGB_OK:
        _raise(status)


def _cfg(cfg) -> abi.CmgbConfig:
    if cfg is None:
        cfg = SmoothingConfig()
    return cfg.to_c() if isinstance(cfg, SmoothingConfig) else cfg


class Mesh:
    """cmg::CollisionMesh (include/cmg/mesh.hpp:25-34)."""

    def __init__(self, handle):
        self._h = handle
        lib = abi.load()
        nv, nf, ne, nw = (C.c_int32() for _ in range(4))
        _ok(lib.cmgb_mesh_sizes(handle, C.byref(nv), C.byref(nf), C.byref(ne), C.byref(nw)))
        self.vertices = np.zeros((nv.value, 3))
        self.faces = np.zeros((nf.value, 3), np.int32)
        self.edges = np.zeros((ne.value, 2), np.int32)
        _ok(lib.cmgb_mesh_read(handle, self.vertices.ctypes.data, self.faces.ctypes.data,
                               self.edges.ctypes.data))
        self.warnings = [lib.cmgb_mesh_warning(handle, i).decode() for i in range(nw.value)]

    @staticmethod
    def box(half_extents, subdivisions: int = 1, quad_edges: bool = True) -> "Mesh":
        lib = abi.load()
        h = (C.c_double * 3)(*[float(x) for x in half_extents])
        out = C.c_void_p()
        _ok(lib.cmgb_mesh_box(h, int(subdivisions), int(bool(quad_edges)), C.byref(out)))
        return Mesh(out)

    @staticmethod
    def parse_obj(text: str) -> "Mesh":
        lib = abi.load()
        b = text.encode()
        out = C.c_void_p()
        line = C.c_int32(0)
        st = lib.cmgb_mesh_parse_obj(b, len(b), C.byref(out), C.byref(line))
        if st == 2:
            raise MeshParseError(lib.cmgb_last_error().decode(), line.value)
        _ok(st)
        return Mesh(out)

    @staticmethod
    def from_arrays(vertices, faces, edges) -> "Mesh":
        lib = abi.load()
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        f = np.ascontiguousarray(faces, dtype=np.int32).reshape(-1, 3)
        e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
        out = C.c_void_p()
        _ok(lib.cmgb_mesh_from_arrays(v.ctypes.data, len(v), f.ctypes.data, len(f), e.ctypes.data,
                                      len(e), C.byref(out)))
        return Mesh(out)

    def __del__(self):
        if getattr(self, "_h", None) and abi is not None and abi.load is not None:  # not at interpreter exit
            abi.load().cmgb_mesh_destroy(self._h)
            self._h = None


class Surface:
    """cmg::SurfaceModel via build_surface (src/surface.cpp:9-44)."""

    def __init__(self, mesh: Mesh, sdf: SdfNode, vertex_topk: int = 0, edge_topk: int = 0,
                 tolerance_fraction: float = 1e-2):
        lib = abi.load()
        self.mesh = mesh
        self.sdf = sdf
        self._prog = SdfProgram(sdf)
        out = C.c_void_p()
        _ok(lib.cmgb_surface_create(mesh._h, self._prog.array, self._prog.n, int(vertex_topk),
                                    int(edge_topk), float(tolerance_fraction), C.byref(out)))
        self._h = out
        info = abi.CmgbSurfaceInfo()
        _ok(lib.cmgb_surface_get_info(out, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in abi.CmgbSurfaceInfo._fields_}
        self.build_warnings = [lib.cmgb_surface_warning(out, i).decode()
                               for i in range(info.n_warnings)]

    def effective_vertex_topk(self) -> int:
        return self.info["effective_vertex_topk"]

    def effective_edge_topk(self) -> int:
        return self.info["effective_edge_topk"]

    def __del__(self):
        if getattr(self, "_h", None) and abi is not None and abi.load is not None:  # not at interpreter exit
            abi.load().cmgb_surface_destroy(self._h)
            self._h = None


def validate_config(cfg) -> None:
    """SmoothingConfig::validate (config.hpp:57-73): raises ValueError with the
    reference's message."""
    c = _cfg(cfg)
    if abi.load().cmgb_config_validate(C.byref(c)) != abi.CMGB_OK:
        raise ValueError(abi.load().cmgb_last_error().decode())


def layout(s1: Surface, s2: Surface, cfg=None) -> dict:
    """ContactManifold sizes (manifold.hpp:62-72)."""
    L = abi.CmgbLayout()
    _ok(abi.load().cmgb_layout_query(s1._h, s2._h, C.byref(_cfg(cfg)), C.byref(L)))
    return {f: getattr(L, f) for f, _ in abi.CmgbLayout._fields_}


def layout_metadata(s1: Surface, s2: Surface, cfg=None) -> np.ndarray:
    """Per-contact (kind, side, src_a, src_b); src = -1 where top-K decides it."""
    n = layout(s1, s2, cfg)["n_contacts"]
    meta = np.zeros((4, n), np.int32)
    _ok(abi.load().cmgb_layout_metadata(s1._h, s2._h, C.byref(_cfg(cfg)), meta[0].ctypes.data,
                                        meta[1].ctypes.data, meta[2].ctypes.data,
                                        meta[3].ctypes.data))
    return meta.T.copy()


def _pose_rows(r1: int, r2: int):
    """(n, stride1, stride2) for pose arrays of r1 / r2 rows: each must have n
    rows (one pose per env) or exactly 1 row (shared by every env)."""
    n = max(r1, r2)
    for r in (r1, r2):
        if r != n and r != 1:
            raise ValueError(f"pose arrays must have n_env rows or 1 row (got {r1} and {r2})")
    if n == 1:
        return 1, 1, 1
    return n, int(r1 == n), int(r2 == n)


def _cuda_tensor(t, dtypes, what: str):
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype not in dtypes:
        names = " or ".join(str(d).replace("torch.", "") for d in dtypes)
        raise ValueError(f"{what} must be a CUDA {names} tensor")
    return t


def _reuse(res: dict, key: str, shape, dtype, device):
    """res[key] if it is a tensor of exactly this shape / dtype / device, else a
    fresh one (a buffer left from a larger batch or another surface pair must
    never be written past its end)."""
    import torch

    t = res.get(key)
    if not (isinstance(t, torch.Tensor) and tuple(t.shape) == tuple(shape) and t.dtype == dtype
            and t.device == device and t.is_contiguous()):
        t = torch.empty(shape, dtype=dtype, device=device)
        res[key] = t
    return t


def _stream_ptr(stream) -> Optional[int]:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def generate_manifold_batch(s1: Surface, s2: Surface, poses1, poses2, cfg=None, *,
                            want_src: bool = False, want_ee: bool = False,
                            want_mean: bool = True, active_threshold: Optional[float] = None,
                            out: Optional[dict] = None, stream=None) -> dict:
    """Batched generate_manifold over envs: poses* are CUDA float64 tensors
    [n, 6] (or [1, 6] / [6] for a pose shared by every env). Returns CUDA
    tensors: contacts [n, C, 8] (px,py,pz,dist,nx,ny,nz,activity), and
    optionally src [n, C, 2], ee [n, 9, m1*m2], mean_dist [n]; with
    active_threshold, the kernels also emit the compaction extra's inputs:
    active_mask [n, ceil(C / 32)] (int32 words, bit c = activity > threshold)
    and active_count [n] (see compact_contacts(..., mask=, count=))."""
    import torch

    c = _cfg(cfg)
    p1 = _cuda_tensor(poses1, (torch.float64,), "poses1").reshape(-1, 6).contiguous()
    p2 = _cuda_tensor(poses2, (torch.float64,), "poses2").reshape(-1, 6).contiguous()
    n, st1, st2 = _pose_rows(p1.shape[0], p2.shape[0])
    L = layout(s1, s2, c)
    Cn = L["n_contacts"]
    P = L["m1"] * L["m2"]
    dev = p2.device
    res = out if out is not None else {}
    contacts = _reuse(res, "contacts", (n, Cn, 8), torch.float32, dev)
    src = _reuse(res, "src", (n, Cn, 2), torch.int32, dev) if want_src else None
    ee = _reuse(res, "ee", (n, 9, P), torch.float32, dev) if (want_ee and P > 0) else None
    mean = _reuse(res, "mean_dist", (n,), torch.float32, dev) if want_mean else None
    amask = acount = None
    if active_threshold is not None:
        amask = _reuse(res, "active_mask", (n, (Cn + 31) // 32), torch.int32, dev)
        acount = _reuse(res, "active_count", (n,), torch.int32, dev)
    ws = abi.load().cmgb_manifold_workspace_bytes(n, st1, st2)
    wsb = res.get("workspace")
    if not (isinstance(wsb, torch.Tensor) and wsb.device == dev and wsb.dtype == torch.uint8 and wsb.numel() >= ws):
        res["workspace"] = torch.empty((max(ws, 8),), dtype=torch.uint8, device=dev)
    o = abi.CmgbManifoldOut()
    o.contacts = contacts.data_ptr()
    o.src = src.data_ptr() if src is not None else None
    o.ee = ee.data_ptr() if ee is not None else None
    o.mean_dist = mean.data_ptr() if mean is not None else None
    o.workspace = res["workspace"].data_ptr()
    o.workspace_bytes = res["workspace"].numel()
    if amask is not None:
        o.active_mask = amask.data_ptr()
        o.active_count = acount.data_ptr()
        o.active_threshold = float(active_threshold)
    with torch.cuda.device(dev):
        _ok(abi.load().cmgb_manifold_batch(s1._h, s2._h, p1.data_ptr(), st1, p2.data_ptr(), st2, n,
                                           C.byref(c), C.byref(o), _stream_ptr(stream)))
    return res


def compact_contacts(contacts, activity_threshold: Optional[float] = None, *, src=None,
                     capacity: Optional[int] = None, mask=None, count=None,
                     out: Optional[dict] = None, stream=None) -> dict:
    """Active-contact compaction (an extra output; the fixed layout stays as
    it is): the contacts of a batch with activity > activity_threshold, in
    fixed-layout order, env after env. contacts: CUDA float32 [n, C, 8] from
    generate_manifold_batch (src: its optional [n, C, 2] provenance). Returns
    CUDA tensors: contacts [capacity, 8] (rows >= total unused), slot
    [capacity] (index in the env's fixed layout), src [capacity, 2] (when src is
    given), env_offset [n + 1] (int64; env_offset[n] = total), env_count [n],
    total [1] (int64). With mask / count (generate_manifold_batch's
    active_mask / active_count) the fixed layout is not scanned again: only the
    kept contacts are read (cmgb_compact_masked); activity_threshold is then
    the one the batch used and is not needed."""
    import torch

    c = _cuda_tensor(contacts, (torch.float32,), "contacts")
    if c.dim() != 3 or c.shape[2] != 8 or not c.is_contiguous():
        raise ValueError("contacts must be a contiguous [n_env, n_contacts, 8] tensor")
    n, Cn = int(c.shape[0]), int(c.shape[1])
    if src is not None:
        _cuda_tensor(src, (torch.int32,), "src")
        if tuple(src.shape) != (n, Cn, 2) or not src.is_contiguous():
            raise ValueError("src must be a contiguous [n_env, n_contacts, 2] int32 tensor")
    cap = n * Cn if capacity is None else int(capacity)
    dev = c.device
    res = out if out is not None else {}
    oc = _reuse(res, "contacts", (cap, 8), torch.float32, dev)
    slot = _reuse(res, "slot", (cap,), torch.int32, dev)
    osrc = _reuse(res, "src", (cap, 2), torch.int32, dev) if src is not None else None
    offs = _reuse(res, "env_offset", (n + 1,), torch.int64, dev)
    cnt = _reuse(res, "env_count", (n,), torch.int32, dev)
    tot = _reuse(res, "total", (1,), torch.int64, dev)
    lib = abi.load()
    masked = mask is not None
    if masked:
        _cuda_tensor(mask, (torch.int32,), "mask")
        _cuda_tensor(count, (torch.int32,), "count")
        if tuple(mask.shape) != (n, (Cn + 31) // 32) or tuple(count.shape) != (n,):
            raise ValueError("mask must be [n_env, ceil(n_contacts / 32)] and count [n_env]")
    elif activity_threshold is None:
        raise ValueError("compact_contacts needs activity_threshold or mask / count")
    ws = lib.cmgb_compact_masked_workspace_bytes(n) if masked else lib.cmgb_compact_workspace_bytes(n, Cn)
    wsb = res.get("workspace")
    if not (isinstance(wsb, torch.Tensor) and wsb.device == dev and wsb.numel() >= ws):
        res["workspace"] = torch.empty((max(ws, 16),), dtype=torch.uint8, device=dev)
    o = abi.CmgbCompactOut()
    o.contacts = oc.data_ptr()
    o.slot = slot.data_ptr()
    o.src = osrc.data_ptr() if osrc is not None else None
    o.env_offset = offs.data_ptr()
    o.env_count = cnt.data_ptr()
    o.total = tot.data_ptr()
    o.capacity = cap
    o.workspace = res["workspace"].data_ptr()
    o.workspace_bytes = res["workspace"].numel()
    with torch.cuda.device(dev):
        if masked:
            _ok(lib.cmgb_compact_masked(c.data_ptr(), src.data_ptr() if src is not None else None, n, Cn,
                                        mask.data_ptr(), count.data_ptr(), C.byref(o), _stream_ptr(stream)))
        else:
            _ok(lib.cmgb_compact_contacts(c.data_ptr(), src.data_ptr() if src is not None else None, n, Cn,
                                          float(activity_threshold), C.byref(o), _stream_ptr(stream)))
    return res


def generate_manifold_jvp_batch(s1: Surface, s2: Surface, poses1, poses2, cfg=None, *,
                                want_src: bool = False, want_f64_mean: bool = False, stream=None) -> dict:
    """Pose Jacobians of the batched manifold: generate_manifold<Dual12> seeded
    by seed_pose_tangents (dual.hpp:249-263) for every env. poses* as in
    generate_manifold_batch. Returns CUDA tensors: contacts [n, C, 8] (primal),
    tangents [n, C, 8, 12] (d field / d (pose1[0..5], pose2[0..5])), mean_dist [n],
    mean_dist_grad [n, 12], optionally src [n, C, 2]. Smooth mode only."""
    import torch

    c = _cfg(cfg)
    p1 = _cuda_tensor(poses1, (torch.float64,), "poses1").reshape(-1, 6).contiguous()
    p2 = _cuda_tensor(poses2, (torch.float64,), "poses2").reshape(-1, 6).contiguous()
    n, st1, st2 = _pose_rows(p1.shape[0], p2.shape[0])
    Cn = layout(s1, s2, c)["n_contacts"]
    dev = p2.device
    res = {
        "contacts": torch.empty((n, Cn, 8), dtype=torch.float32, device=dev),
        "tangents": torch.empty((n, Cn, 8, 12), dtype=torch.float32, device=dev),
        "mean_dist": torch.empty((n,), dtype=torch.float32, device=dev),
        "mean_dist_grad": torch.empty((n, 12), dtype=torch.float32, device=dev),
    }
    if want_src:
        res["src"] = torch.empty((n, Cn, 2), dtype=torch.int32, device=dev)
    if want_f64_mean:  # FP64 mean + tangents (as accumulated on the device; for gradchecks)
        res["mean_dist_f64"] = torch.empty((n,), dtype=torch.float64, device=dev)
        res["mean_dist_grad_f64"] = torch.empty((n, 12), dtype=torch.float64, device=dev)
    o = abi.CmgbManifoldJvpOut()
    o.contacts = res["contacts"].data_ptr()
    o.tangents = res["tangents"].data_ptr()
    o.src = res["src"].data_ptr() if want_src else None
    o.mean_dist = res["mean_dist"].data_ptr()
    o.mean_dist_grad = res["mean_dist_grad"].data_ptr()
    o.mean_dist_f64 = res["mean_dist_f64"].data_ptr() if want_f64_mean else None
    o.mean_dist_grad_f64 = res["mean_dist_grad_f64"].data_ptr() if want_f64_mean else None
    with torch.cuda.device(dev):
        _ok(abi.load().cmgb_manifold_jvp_batch(s1._h, s2._h, p1.data_ptr(), st1, p2.data_ptr(), st2, n,
                                               C.byref(c), C.byref(o), _stream_ptr(stream)))
    return res


def sdf_query(surface: Surface, points, flavor: int = 1, stream=None):
    """SmoothSdf queries (sdf.hpp:177-195) on the GPU: points CUDA float64
    [n, 3] in the body frame -> [n, 4] value + gradient (flavor 1), normal
    source (2) or value only (0)."""
    import torch

    pts = _cuda_tensor(points, (torch.float64,), "points").reshape(-1, 3).contiguous()
    out = torch.empty((pts.shape[0], 4), dtype=torch.float64, device=pts.device)
    with torch.cuda.device(pts.device):
        _ok(abi.load().cmgb_sdf_query(surface._h, int(flavor), pts.data_ptr(), pts.shape[0], out.data_ptr(),
                                      _stream_ptr(stream)))
    return out


def sphere_trace(surface: Surface, pose, points, iters: int = 5, tau: float = 1e-9, stream=None):
    """sphere_trace_project (sdf.hpp:318-326) of world points [n, 3] (CUDA
    float64) against the surface posed by pose [6]."""
    import torch

    pts = _cuda_tensor(points, (torch.float64,), "points").reshape(-1, 3).contiguous()
    pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(6)
    out = torch.empty(pts.shape, dtype=torch.float64, device=pts.device)
    with torch.cuda.device(pts.device):
        _ok(abi.load().cmgb_sphere_trace(surface._h, pose.ctypes.data, pts.data_ptr(), pts.shape[0], int(iters),
                                         float(tau), out.data_ptr(), _stream_ptr(stream)))
    return out


def mean_contact_distance(contacts, tangents=None):
    """mean_contact_distance (manifold.hpp:379-384) over contacts [..., C, 8]
    (torch or numpy); with tangents [..., C, 8, 12] also its 12 pose tangents.
    (The batch calls return it per env directly; this is the reduction for
    caller-side use.)"""
    d = contacts[..., 3]
    m = d.mean(-1)
    if tangents is None:
        return m
    return m, tangents[..., 3, :].mean(-2)


def activity_weighted_distance(contacts, tangents=None):
    """activity_weighted_distance (manifold.hpp:386-391): sum of activity x
    dist over contacts [..., C, 8]; with tangents [..., C, 8, 12] also its pose
    tangents (product rule: act' dist + act dist')."""
    d, a = contacts[..., 3], contacts[..., 7]
    v = (a * d).sum(-1)
    if tangents is None:
        return v
    g = (tangents[..., 7, :] * d[..., None] + a[..., None] * tangents[..., 3, :]).sum(-2)
    return v, g


def scene_pairs(n_bodies: int, is_static=None) -> np.ndarray:
    """Body pairs (i < j, skipping static-static) in DemoSim::step's order
    (src/demosim.cpp:88-104)."""
    lib = abi.load()
    st = None if is_static is None else np.ascontiguousarray(is_static, dtype=np.int32)
    n = C.c_int32()
    _ok(lib.cmgb_scene_pairs(st.ctypes.data if st is not None else None, n_bodies, None, C.byref(n)))
    out = np.zeros((n.value, 2), np.int32)
    _ok(lib.cmgb_scene_pairs(st.ctypes.data if st is not None else None, n_bodies, out.ctypes.data,
                             C.byref(n)))
    return out


def generate_manifold_scene_batch(bodies, poses, cfg=None, *, is_static=None, pairs=None,
                                  want_src: bool = False, want_ee: bool = False,
                                  outs: Optional[list] = None, stream=None) -> list:
    """All-pairs manifolds of a multi-body scene for every env: poses is a CUDA
    float64 tensor [n_env, n_bodies, 6]; returns one result dict per pair (as
    generate_manifold_batch) plus its (i, j)."""
    import torch

    c = _cfg(cfg)
    P = poses.contiguous()
    if P.dtype != torch.float64 or not P.is_cuda or P.dim() != 3 or P.shape[2] != 6:
        raise ValueError("poses must be a CUDA float64 tensor [n_env, n_bodies, 6]")
    n_env, nb = P.shape[0], P.shape[1]
    if len(bodies) != nb:
        raise ValueError("one surface per body")
    pr = scene_pairs(nb, is_static) if pairs is None else np.ascontiguousarray(pairs, dtype=np.int32)
    res = outs if outs is not None else [dict() for _ in range(len(pr))]
    arr = (abi.CmgbManifoldOut * max(len(pr), 1))()
    lib = abi.load()
    for q, (i, j) in enumerate(pr):
        L = layout(bodies[i], bodies[j], c)
        r = res[q]
        r["pair"] = (int(i), int(j))
        Pq = L["m1"] * L["m2"]
        contacts = _reuse(r, "contacts", (n_env, L["n_contacts"], 8), torch.float32, P.device)
        src = _reuse(r, "src", (n_env, L["n_contacts"], 2), torch.int32, P.device) if want_src else None
        ee = _reuse(r, "ee", (n_env, 9, Pq), torch.float32, P.device) if (want_ee and Pq > 0) else None
        mean = _reuse(r, "mean_dist", (n_env,), torch.float32, P.device)
        ws = lib.cmgb_manifold_workspace_bytes(n_env, 1, 1)
        wsb = r.get("workspace")
        if not (isinstance(wsb, torch.Tensor) and wsb.device == P.device and wsb.numel() >= ws):
            r["workspace"] = torch.empty((max(ws, 8),), dtype=torch.uint8, device=P.device)
        o = arr[q]
        o.contacts = contacts.data_ptr()
        o.src = src.data_ptr() if src is not None else None
        o.ee = ee.data_ptr() if ee is not None else None
        o.mean_dist = mean.data_ptr()
        o.workspace = r["workspace"].data_ptr()
        o.workspace_bytes = r["workspace"].numel()
    handles = (C.c_void_p * nb)(*[b._h.value if isinstance(b._h, C.c_void_p) else b._h for b in bodies])
    with torch.cuda.device(P.device):
        _ok(lib.cmgb_manifold_scene_batch(handles, nb, pr.ctypes.data, len(pr), P.data_ptr(), n_env,
                                          C.byref(c), arr, _stream_ptr(stream)))
    return res


def generate_manifold_scene_batch_host(bodies, poses, cfg=None, *, is_static=None, pairs=None,
                                       mean_out: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
    """End-to-end C-ABI scene path (cmgb_manifold_scene_batch_host): HOST
    float64 poses [n_env, n_bodies, 6] in, each pair's per-env mean contact
    distance [n_pairs, n_env] float32 out (copies inside, synchronous). Pairs
    in scene_pairs order unless given."""
    c = _cfg(cfg)
    P = np.ascontiguousarray(poses, dtype=np.float64)
    if P.ndim != 3 or P.shape[2] != 6:
        raise ValueError("poses must be [n_env, n_bodies, 6]")
    n_env, nb = P.shape[0], P.shape[1]
    if len(bodies) != nb:
        raise ValueError("one surface per body")
    pr = scene_pairs(nb, is_static) if pairs is None else np.ascontiguousarray(pairs, dtype=np.int32)
    mean = mean_out if mean_out is not None else np.empty((len(pr), n_env), np.float32)
    if mean.dtype != np.float32 or mean.size < len(pr) * n_env or not mean.flags.c_contiguous:
        raise ValueError("mean_out must be a contiguous float32 array of n_pairs x n_env elements")
    handles = (C.c_void_p * nb)(*[b._h.value if isinstance(b._h, C.c_void_p) else b._h for b in bodies])
    _ok(abi.load().cmgb_manifold_scene_batch_host(handles, nb, pr.ctypes.data, len(pr), P.ctypes.data, n_env,
                                                   C.byref(c), mean.ctypes.data, _stream_ptr(stream)))
    return mean


def generate_manifold_scene_jvp_batch(bodies, poses, cfg=None, *, is_static=None, pairs=None,
                                      want_src: bool = False, outs: Optional[list] = None,
                                      stream=None) -> list:
    """Config D's forward + 12-tangent JVP per pair: for every scene pair (i, j)
    and env, the primal contacts and their Jacobian w.r.t. (pose_i, pose_j)
    (as generate_manifold_jvp_batch). poses: CUDA float64 [n_env, n_bodies, 6]."""
    import torch

    c = _cfg(cfg)
    P = poses.contiguous()
    if P.dtype != torch.float64 or not P.is_cuda or P.dim() != 3 or P.shape[2] != 6:
        raise ValueError("poses must be a CUDA float64 tensor [n_env, n_bodies, 6]")
    n_env, nb = P.shape[0], P.shape[1]
    if len(bodies) != nb:
        raise ValueError("one surface per body")
    pr = scene_pairs(nb, is_static) if pairs is None else np.ascontiguousarray(pairs, dtype=np.int32)
    res = outs if outs is not None else [dict() for _ in range(len(pr))]
    arr = (abi.CmgbManifoldJvpOut * max(len(pr), 1))()
    dev = P.device
    for q, (i, j) in enumerate(pr):
        Cn = layout(bodies[i], bodies[j], c)["n_contacts"]
        r = res[q]
        r["pair"] = (int(i), int(j))
        for k, shape, dt in (("contacts", (n_env, Cn, 8), torch.float32),
                             ("tangents", (n_env, Cn, 8, 12), torch.float32),
                             ("mean_dist", (n_env,), torch.float32),
                             ("mean_dist_grad", (n_env, 12), torch.float32)):
            _reuse(r, k, shape, dt, dev)
        src = _reuse(r, "src", (n_env, Cn, 2), torch.int32, dev) if want_src else None
        o = arr[q]
        o.contacts = r["contacts"].data_ptr()
        o.tangents = r["tangents"].data_ptr()
        o.src = src.data_ptr() if src is not None else None
        o.mean_dist = r["mean_dist"].data_ptr()
        o.mean_dist_grad = r["mean_dist_grad"].data_ptr()
    handles = (C.c_void_p * nb)(*[b._h.value if isinstance(b._h, C.c_void_p) else b._h for b in bodies])
    with torch.cuda.device(dev):
        _ok(abi.load().cmgb_manifold_scene_jvp_batch(handles, nb, pr.ctypes.data, len(pr), P.data_ptr(), n_env,
                                                     C.byref(c), arr, _stream_ptr(stream)))
    return res


def generate_manifold_batch_host(s1: Surface, s2: Surface, poses1: np.ndarray, poses2: np.ndarray,
                                 cfg=None, mean_out: Optional[np.ndarray] = None,
                                 contacts_out: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
    """End-to-end C-ABI path: HOST poses in, HOST mean distances out (copies inside)."""
    c = _cfg(cfg)
    p1 = np.ascontiguousarray(poses1, dtype=np.float64).reshape(-1, 6)
    p2 = np.ascontiguousarray(poses2, dtype=np.float64).reshape(-1, 6)
    n, st1, st2 = _pose_rows(len(p1), len(p2))
    mean = mean_out if mean_out is not None else np.empty(n, np.float32)
    if mean.dtype != np.float32 or mean.size < n or not mean.flags.c_contiguous:
        raise ValueError("mean_out must be a contiguous float32 array of n_env elements")
    if contacts_out is not None:
        Cn = layout(s1, s2, c)["n_contacts"]
        if contacts_out.dtype != np.float32 or contacts_out.size < n * Cn * 8 or not contacts_out.flags.c_contiguous:
            raise ValueError("contacts_out must be a contiguous float32 array of n_env x n_contacts x 8")
    _ok(abi.load().cmgb_manifold_batch_host(
        s1._h, s2._h, p1.ctypes.data, st1, p2.ctypes.data, st2, n, C.byref(c), mean.ctypes.data,
        contacts_out.ctypes.data if contacts_out is not None else None, _stream_ptr(stream)))
    return mean


def generate_manifold(s1: Surface, s2: Surface, pose1, pose2, cfg=None) -> dict:
    """One env, reference-shaped result (numpy): contacts [C, 8], meta [C, 4]
    (kind, side, src_a, src_b), ee [9, m1*m2], layout."""
    import torch

    p1 = torch.as_tensor(np.asarray(pose1, dtype=np.float64).reshape(1, 6), device="cuda")
    p2 = torch.as_tensor(np.asarray(pose2, dtype=np.float64).reshape(1, 6), device="cuda")
    r = generate_manifold_batch(s1, s2, p1, p2, cfg, want_src=True, want_ee=True)
    torch.cuda.synchronize()
    meta = layout_metadata(s1, s2, cfg)
    meta[:, 2:] = r["src"][0].cpu().numpy()
    out = {"contacts": r["contacts"][0].cpu().numpy(), "meta": meta, "layout": layout(s1, s2, cfg),
           "mean_dist": float(r["mean_dist"][0].item())}
    out["ee"] = r["ee"][0].cpu().numpy() if "ee" in r else np.zeros((9, 0), np.float32)
    return out


def run_ee_batch(pairs, cfg=None, *, want_alpha: bool = False, want_labels: bool = False,
                 stream=None) -> dict:
    """run_ee_batch (batch.cpp:53-76) on a CUDA [n, 12] float64/float32 tensor."""
    import torch

    c = _cfg(cfg)
    pr = _cuda_tensor(pairs, (torch.float64, torch.float32), "pairs").reshape(-1, 12).contiguous()
    n = pr.shape[0]
    res = {"out": torch.empty((n, 6), dtype=torch.float32, device=pr.device)}
    if want_alpha:
        res["alpha_gamma"] = torch.empty((n, 3), dtype=torch.float32, device=pr.device)
    if want_labels:
        res["labels"] = torch.empty((n,), dtype=torch.int32, device=pr.device)
    with torch.cuda.device(pr.device):
        _ok(abi.load().cmgb_ee_witness_batch(
            pr.data_ptr(), int(pr.dtype == torch.float64), n, C.byref(c), res["out"].data_ptr(),
            res["alpha_gamma"].data_ptr() if want_alpha else None,
            res["labels"].data_ptr() if want_labels else None, _stream_ptr(stream)))
    return res


def run_ee_batch_f64(pairs, cfg=None, *, want_alpha: bool = False, want_labels: bool = False,
                     stream=None) -> dict:
    """Reference-precision E-E witnesses (FP64 indicators, FP64 outputs) on a
    CUDA [n, 12] float64 tensor: what ee_witness<double> returns."""
    import torch

    c = _cfg(cfg)
    pr = _cuda_tensor(pairs, (torch.float64,), "pairs").reshape(-1, 12).contiguous()
    n = pr.shape[0]
    res = {"out": torch.empty((n, 6), dtype=torch.float64, device=pr.device)}
    if want_alpha:
        res["alpha_gamma"] = torch.empty((n, 3), dtype=torch.float64, device=pr.device)
    if want_labels:
        res["labels"] = torch.empty((n,), dtype=torch.int32, device=pr.device)
    with torch.cuda.device(pr.device):
        _ok(abi.load().cmgb_ee_witness_batch_f64(
            pr.data_ptr(), n, C.byref(c), res["out"].data_ptr(),
            res["alpha_gamma"].data_ptr() if want_alpha else None,
            res["labels"].data_ptr() if want_labels else None, _stream_ptr(stream)))
    return res


SWEEP_VARIANTS = {"no_smoothing": 0, "l2": 1, "smooth": 2}


def rotating_edge_sweep(variant, n_samples: int = 10000) -> np.ndarray:
    """rotating_edge_sweep (src/sweep.cpp:44-56, the paper's Fig. 4) on the GPU:
    [n, 7] = theta, p1 (3), dp1/dtheta (3). variant: 0 / "no_smoothing", 1 /
    "l2", 2 / "smooth"."""
    v = SWEEP_VARIANTS.get(variant, variant)
    out = np.zeros((n_samples, 7))
    _ok(abi.load().cmgb_rotating_edge_sweep(int(v), int(n_samples), out.ctypes.data))
    return out


def run_vf_batch(pairs, cfg=None, *, want_labels: bool = False, stream=None) -> dict:
    """run_vf_batch (batch.cpp:78-98) on a CUDA [n, 12] tensor."""
    import torch

    c = _cfg(cfg)
    pr = _cuda_tensor(pairs, (torch.float64, torch.float32), "pairs").reshape(-1, 12).contiguous()
    n = pr.shape[0]
    res = {"out": torch.empty((n, 3), dtype=torch.float32, device=pr.device)}
    if want_labels:
        res["labels"] = torch.empty((n,), dtype=torch.int32, device=pr.device)
    with torch.cuda.device(pr.device):
        _ok(abi.load().cmgb_vf_witness_batch(
            pr.data_ptr(), int(pr.dtype == torch.float64), n, C.byref(c), res["out"].data_ptr(),
            res["labels"].data_ptr() if want_labels else None, _stream_ptr(stream)))
    return res


def _witness_host(sym: str, width: int, pairs, cfg, out, labels, stream) -> np.ndarray:
    c = _cfg(cfg)
    pr = np.ascontiguousarray(pairs, dtype=np.float64).reshape(-1, 12)
    n = pr.shape[0]
    if out is None:
        out = np.empty((n, width), np.float64)
    if out.dtype != np.float64 or out.size < n * width or not out.flags.c_contiguous:
        raise ValueError(f"out must be a contiguous float64 array of n x {width} elements")
    if labels is not None and (labels.dtype != np.int32 or labels.size < n or not labels.flags.c_contiguous):
        raise ValueError("labels must be a contiguous int32 array of n elements")
    _ok(getattr(abi.load(), sym)(pr.ctypes.data, n, C.byref(c), out.ctypes.data,
                                 labels.ctypes.data if labels is not None else None, _stream_ptr(stream)))
    return out


def run_ee_batch_host(pairs, cfg=None, *, out: Optional[np.ndarray] = None, labels: Optional[np.ndarray] = None,
                      stream=None) -> np.ndarray:
    """run_ee_batch with HOST buffers (batch.cpp:53-76: the reference's problem
    set in, doubles out): [n, 12] float64 pairs -> [n, 6] float64 witness
    points of the FP64 solver; copies inside, pipelined over pair chunks on two
    streams (with pinned buffers, e.g. torch's pin_memory().numpy(), the
    downloads overlap the uploads). Synchronous."""
    return _witness_host("cmgb_ee_witness_batch_host", 6, pairs, cfg, out, labels, stream)


def run_vf_batch_host(pairs, cfg=None, *, out: Optional[np.ndarray] = None, labels: Optional[np.ndarray] = None,
                      stream=None) -> np.ndarray:
    """run_vf_batch with HOST buffers (batch.cpp:78-98): [n, 12] float64 pairs
    -> [n, 3] witness points (the FP32-output solver, widened to float64 on
    the device). Synchronous."""
    return _witness_host("cmgb_vf_witness_batch_host", 3, pairs, cfg, out, labels, stream)


def surface_from_spec(body) -> Surface:
    """Build a Surface from a workloads.BodySpec."""
    m = body.mesh
    mesh = Mesh.box(m.box_half, m.subdivisions, m.quad_edges) if m.box_half is not None \
        else Mesh.parse_obj(m.obj_text)
    return Surface(mesh, body.sdf, body.vertex_topk, body.edge_topk)


class DemoBatch:
    """DemoSim (src/demosim.cpp:68-186) over a batch of n_env copies of a
    scene, stepped on the GPU (cmgb_demo_step_batch): all-pairs manifolds ->
    penalty_forces -> semi-implicit Euler on SE(3), every env in one call per
    step. State lives in CUDA float64 tensors: poses / velocities
    [n_env, n_bodies, 6] (velocity = world [linear; angular])."""

    def __init__(self, bodies, masses=None, *, inertia=None, is_static=None, cfg=None, params=None,
                 poses=None, velocities=None, n_env: int = 1, device="cuda"):
        import torch

        from .scene import PenaltyParams

        nb = len(bodies)
        self.bodies = list(bodies)
        self.cfg = _cfg(cfg)
        self.params = (params or PenaltyParams()).to_c()
        masses = np.ones(nb) if masses is None else np.asarray(masses, dtype=np.float64)
        inertia = np.zeros((nb, 3)) if inertia is None else np.asarray(inertia, dtype=np.float64).reshape(nb, 3)
        is_static = np.zeros(nb, bool) if is_static is None else np.asarray(is_static, bool)
        self.is_static = is_static
        self.masses = masses
        self._bodies = (abi.CmgbDemoBody * nb)()
        for i, b in enumerate(bodies):
            d = self._bodies[i]
            d.surface = b._h.value if isinstance(b._h, C.c_void_p) else b._h
            d.mass = float(masses[i])
            for k in range(3):
                d.inertia_diag[k] = float(inertia[i, k])
            d.is_static = int(is_static[i])
        P = np.zeros((n_env, nb, 6)) if poses is None else np.array(np.broadcast_to(
            np.asarray(poses, dtype=np.float64), (n_env, nb, 6)))
        V = np.zeros((n_env, nb, 6)) if velocities is None else np.array(np.broadcast_to(
            np.asarray(velocities, dtype=np.float64), (n_env, nb, 6)))
        self.poses = torch.as_tensor(np.ascontiguousarray(P), device=device)
        self.velocities = torch.as_tensor(np.ascontiguousarray(V), device=device)
        self.deepest = torch.zeros(n_env, dtype=torch.float64, device=device)
        self.ok = torch.ones(n_env, dtype=torch.int32, device=device)
        ws = abi.load().cmgb_demo_workspace_bytes(self._bodies, nb, C.byref(self.cfg), n_env)
        self._ws = torch.empty(max(ws, 256), dtype=torch.uint8, device=device)
        self.n_env = n_env
        self.time = 0.0

    def step(self, dt: float, n: int = 1, stream=None) -> None:
        """n DemoSim::step(dt) calls for every env (stream-ordered)."""
        import torch

        lib = abi.load()
        with torch.cuda.device(self.poses.device):
            for _ in range(n):
                _ok(lib.cmgb_demo_step_batch(self._bodies, len(self.bodies), C.byref(self.cfg),
                                             C.byref(self.params), float(dt), self.n_env,
                                             self.poses.data_ptr(), self.velocities.data_ptr(),
                                             self.deepest.data_ptr(), self.ok.data_ptr(), self._ws.data_ptr(),
                                             self._ws.numel(), _stream_ptr(stream)))
                self.time += dt

    def inertia_diag(self) -> np.ndarray:
        """Per-body inertia as DemoSim uses it: given, or the mesh-AABB box
        inertia (demosim.cpp:17-23, 68-79)."""
        out = np.zeros((len(self.bodies), 3))
        for i, b in enumerate(self.bodies):
            given = np.array([self._bodies[i].inertia_diag[k] for k in range(3)])
            out[i] = given if (given > 0).all() else _box_inertia(self.masses[i], b.mesh.vertices)
        return out

    def linear_momentum(self):
        """DemoSim::linear_momentum (demosim.cpp:157-166) per env: [n_env, 3]
        (CUDA tensor; static bodies excluded)."""
        import torch

        m = torch.as_tensor(np.where(self.is_static, 0.0, self.masses), device=self.velocities.device)
        return (self.velocities[:, :, :3] * m[None, :, None]).sum(dim=1)

    def states(self):
        """DemoSim::states (demosim.hpp:57-58): (poses, velocities), each
        [n_env, n_bodies, 6] on the device (velocity = world [linear; angular])."""
        return self.poses, self.velocities

    def deepest_penetration(self):
        """DemoSim::deepest_penetration (demosim.hpp:63-64) of the last step, per env."""
        return self.deepest

    def kinetic_energy(self) -> np.ndarray:
        """DemoSim::kinetic_energy (demosim.cpp:140-155) per env (host)."""
        return kinetic_energy_np(self.poses.cpu().numpy(), self.velocities.cpu().numpy(), self.masses,
                                 self.inertia_diag(), self.is_static)


def kinetic_energy_np(poses, vels, masses, inertia, is_static) -> np.ndarray:
    """DemoSim::kinetic_energy (demosim.cpp:140-155) for [n_env, n_bodies, 6] states."""
    poses = np.asarray(poses, np.float64).reshape(-1, len(masses), 6)
    vels = np.asarray(vels, np.float64).reshape(-1, len(masses), 6)
    e = np.zeros(len(poses))
    for i in range(len(masses)):
        if is_static[i]:
            continue
        v = vels[:, i]
        e += 0.5 * masses[i] * (v[:, :3] ** 2).sum(axis=1)
        for n in range(len(poses)):
            wb = _so3_exp_np(poses[n, i, 3:]).T @ v[n, 3:]
            e[n] += 0.5 * float((inertia[i] * wb * wb).sum())
    return e


def _box_inertia(mass, vertices):
    s = vertices.max(axis=0) - vertices.min(axis=0)
    return mass / 12.0 * np.array([s[1] ** 2 + s[2] ** 2, s[0] ** 2 + s[2] ** 2, s[0] ** 2 + s[1] ** 2])


def _so3_exp_np(w):
    th2 = float(w @ w)
    if th2 < 1e-8:
        a, b = 1 - th2 / 6 + th2 * th2 / 120, 0.5 - th2 / 24 + th2 * th2 / 720
    else:
        th = np.sqrt(th2)
        a, b = np.sin(th) / th, (1 - np.cos(th)) / th2
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    return np.eye(3) + W * a + (W @ W) * b
