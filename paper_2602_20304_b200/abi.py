"""ctypes mirror of include/cmgb.h and the loader for the native library.

The product path is the in-tree shared library ``libcmgb.so`` (host C++ +
sm_100a CUDA kernels). There is no CPU fallback: if the library is missing,
``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CMGB_LIBRARY: developer override (e.g. an instrumented -DCMGB_PHASE_CLOCKS build)
LIB_PATH = os.environ.get("CMGB_LIBRARY") or os.path.join(_HERE, "libcmgb.so")

CMGB_OK = 0
STATUS_NAMES = {
    0: "CMGB_OK",
    1: "CMGB_ERR_INVALID_ARGUMENT",
    2: "CMGB_ERR_PARSE",
    3: "CMGB_ERR_CUDA",
    4: "CMGB_ERR_NO_DEVICE",
    5: "CMGB_ERR_UNSUPPORTED",
}

MODE_FULL, MODE_NO_EE, MODE_ONE_SIDED = 0, 1, 2
SDF_SUPERQUADRIC, SDF_CONVEX_POLYHEDRON, SDF_ORIENTED_POINTCLOUD, SDF_UNION, SDF_SUBTRACTION = range(5)


class CmgbConfig(C.Structure):
    """cmgb_config == cmg::SmoothingConfig (config.hpp:17-46)."""

    _fields_ = [
        ("lambda_", C.c_double),
        ("tau_clip", C.c_double),
        ("tau_min", C.c_double),
        ("tau_comp", C.c_double),
        ("tau_sign", C.c_double),
        ("tau_pen", C.c_double),
        ("tau_nn", C.c_double),
        ("tau_clash", C.c_double),
        ("tau_cont", C.c_double),
        ("tau_topk_verts", C.c_double),
        ("tau_topk_edges", C.c_double),
        ("tau_normal", C.c_double),
        ("tau_union", C.c_double),
        ("hard_ops", C.c_int32),
        ("sphere_trace", C.c_int32),
        ("sphere_trace_iters", C.c_int32),
        ("containment_safeguard", C.c_int32),
        ("mode", C.c_int32),
        ("reserved", C.c_int32),
    ]


class CmgbSdfNode(C.Structure):
    _fields_ = [
        ("op", C.c_int32),
        ("count", C.c_int32),
        ("tau", C.c_double),
        ("eps1", C.c_double),
        ("eps2", C.c_double),
        ("axes", C.c_double * 3),
        ("pose", C.c_double * 6),
        ("normals", C.POINTER(C.c_double)),
        ("points", C.POINTER(C.c_double)),
        ("lengthscales", C.POINTER(C.c_double)),
    ]


class CmgbSurfaceInfo(C.Structure):
    _fields_ = [
        (n, C.c_int32)
        for n in (
            "n_vertices", "n_edges", "n_faces", "leaf_count", "vertex_topk", "edge_topk",
            "effective_vertex_topk", "effective_edge_topk", "n_warnings", "n_nodes",
        )
    ]


class CmgbLayout(C.Structure):
    _fields_ = [
        (n, C.c_int32)
        for n in ("n1", "n2", "m1", "m2", "mode", "n_contacts", "dynamic_src", "reserved")
    ]


class CmgbManifoldOut(C.Structure):
    _fields_ = [
        ("contacts", C.c_void_p),
        ("src", C.c_void_p),
        ("ee", C.c_void_p),
        ("mean_dist", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
        ("active_mask", C.c_void_p),
        ("active_count", C.c_void_p),
        ("active_threshold", C.c_float),
        ("reserved", C.c_int32),
    ]


class CmgbCompactOut(C.Structure):
    _fields_ = [
        ("contacts", C.c_void_p),
        ("slot", C.c_void_p),
        ("src", C.c_void_p),
        ("env_offset", C.c_void_p),
        ("env_count", C.c_void_p),
        ("total", C.c_void_p),
        ("capacity", C.c_int64),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
    ]


class CmgbManifoldJvpOut(C.Structure):
    _fields_ = [
        ("contacts", C.c_void_p),
        ("tangents", C.c_void_p),
        ("src", C.c_void_p),
        ("mean_dist", C.c_void_p),
        ("mean_dist_grad", C.c_void_p),
        ("mean_dist_f64", C.c_void_p),
        ("mean_dist_grad_f64", C.c_void_p),
    ]


class CmgbDemoParams(C.Structure):
    """cmgb_demo_params == cmg::PenaltyParams (demosim.hpp:24-31)."""

    _fields_ = [
        ("stiffness", C.c_double),
        ("damping", C.c_double),
        ("friction", C.c_double),
        ("friction_viscous", C.c_double),
        ("tau_force", C.c_double),
        ("gravity", C.c_double * 3),
    ]


class CmgbDemoBody(C.Structure):
    _fields_ = [
        ("surface", C.c_void_p),
        ("mass", C.c_double),
        ("inertia_diag", C.c_double * 3),
        ("is_static", C.c_int32),
        ("reserved", C.c_int32),
    ]


# Every exported symbol of include/cmgb.h with its ctypes signature.
_P = C.c_void_p
_I = C.c_int
SIGNATURES = {
    "cmgb_last_error": (C.c_char_p, []),
    "cmgb_abi_version": (C.c_int32, []),
    "cmgb_config_default": (None, [C.POINTER(CmgbConfig)]),
    "cmgb_config_no_smoothing": (None, [C.POINTER(CmgbConfig)]),
    "cmgb_config_validate": (_I, [C.POINTER(CmgbConfig)]),
    "cmgb_config_for_variant": (_I, [C.c_char_p, C.POINTER(CmgbConfig), C.POINTER(CmgbConfig)]),
    "cmgb_mesh_box": (_I, [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.POINTER(_P)]),
    "cmgb_mesh_parse_obj": (_I, [C.c_char_p, C.c_size_t, C.POINTER(_P), C.POINTER(C.c_int32)]),
    "cmgb_mesh_from_arrays": (
        _I,
        [_P, C.c_int32, _P, C.c_int32, _P, C.c_int32, C.POINTER(_P)],
    ),
    "cmgb_mesh_sizes": (
        _I,
        [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    ),
    "cmgb_mesh_read": (_I, [_P, _P, _P, _P]),
    "cmgb_mesh_warning": (C.c_char_p, [_P, C.c_int32]),
    "cmgb_mesh_destroy": (None, [_P]),
    "cmgb_surface_create": (
        _I,
        [_P, C.POINTER(CmgbSdfNode), C.c_int32, C.c_int32, C.c_int32, C.c_double, C.POINTER(_P)],
    ),
    "cmgb_surface_destroy": (None, [_P]),
    "cmgb_surface_get_info": (_I, [_P, C.POINTER(CmgbSurfaceInfo)]),
    "cmgb_surface_warning": (C.c_char_p, [_P, C.c_int32]),
    "cmgb_layout_query": (_I, [_P, _P, C.POINTER(CmgbConfig), C.POINTER(CmgbLayout)]),
    "cmgb_layout_metadata": (_I, [_P, _P, C.POINTER(CmgbConfig), _P, _P, _P, _P]),
    "cmgb_manifold_batch": (
        _I,
        [_P, _P, _P, C.c_int32, _P, C.c_int32, C.c_int64, C.POINTER(CmgbConfig),
         C.POINTER(CmgbManifoldOut), _P],
    ),
    "cmgb_manifold_batch_host": (
        _I,
        [_P, _P, _P, C.c_int32, _P, C.c_int32, C.c_int64, C.POINTER(CmgbConfig), _P, _P, _P],
    ),
    "cmgb_ee_witness_batch": (
        _I,
        [_P, C.c_int32, C.c_int64, C.POINTER(CmgbConfig), _P, _P, _P, _P],
    ),
    "cmgb_vf_witness_batch": (
        _I,
        [_P, C.c_int32, C.c_int64, C.POINTER(CmgbConfig), _P, _P, _P],
    ),
    "cmgb_device_count": (_I, [C.POINTER(C.c_int32)]),
    "cmgb_sdf_query": (_I, [_P, C.c_int32, _P, C.c_int64, _P, _P]),
    "cmgb_sphere_trace": (_I, [_P, _P, _P, C.c_int64, C.c_int32, C.c_double, _P, _P]),
    "cmgb_ee_witness_batch_f64": (_I, [_P, C.c_int64, C.POINTER(CmgbConfig), _P, _P, _P, _P]),
    "cmgb_rotating_edge_sweep": (_I, [C.c_int32, C.c_int32, _P]),
    "cmgb_manifold_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32, C.c_int32]),
    "cmgb_manifold_jvp_batch": (
        _I,
        [_P, _P, _P, C.c_int32, _P, C.c_int32, C.c_int64, C.POINTER(CmgbConfig),
         C.POINTER(CmgbManifoldJvpOut), _P],
    ),
    "cmgb_manifold_scene_jvp_batch": (
        _I,
        [C.POINTER(_P), C.c_int32, _P, C.c_int32, _P, C.c_int64, C.POINTER(CmgbConfig),
         C.POINTER(CmgbManifoldJvpOut), _P],
    ),
    "cmgb_demo_params_default": (None, [C.POINTER(CmgbDemoParams)]),
    "cmgb_demo_workspace_bytes": (C.c_size_t, [C.POINTER(CmgbDemoBody), C.c_int32, C.POINTER(CmgbConfig),
                                               C.c_int64]),
    "cmgb_demo_step_batch": (
        _I,
        [C.POINTER(CmgbDemoBody), C.c_int32, C.POINTER(CmgbConfig), C.POINTER(CmgbDemoParams), C.c_double,
         C.c_int64, _P, _P, _P, _P, _P, C.c_size_t, _P],
    ),
    "cmgb_scene_pairs": (_I, [_P, C.c_int32, _P, C.POINTER(C.c_int32)]),
    "cmgb_manifold_batch_host_ex": (
        _I,
        [_P, _P, _P, C.c_int32, _P, C.c_int32, C.c_int64, C.POINTER(CmgbConfig), C.POINTER(CmgbManifoldOut), _P],
    ),
    "cmgb_manifold_jvp_batch_host": (
        _I,
        [_P, _P, _P, C.c_int32, _P, C.c_int32, C.c_int64, C.POINTER(CmgbConfig),
         C.POINTER(CmgbManifoldJvpOut), _P],
    ),
    "cmgb_ee_witness_batch_host": (_I, [_P, C.c_int64, C.POINTER(CmgbConfig), _P, _P, _P]),
    "cmgb_vf_witness_batch_host": (_I, [_P, C.c_int64, C.POINTER(CmgbConfig), _P, _P, _P]),
    "cmgb_compact_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32]),
    "cmgb_compact_masked_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "cmgb_compact_masked": (_I, [_P, _P, C.c_int64, C.c_int32, _P, _P, C.POINTER(CmgbCompactOut), _P]),
    "cmgb_compact_contacts": (
        _I,
        [_P, _P, C.c_int64, C.c_int32, C.c_float, C.POINTER(CmgbCompactOut), _P],
    ),
    "cmgb_manifold_scene_batch": (
        _I,
        [C.POINTER(_P), C.c_int32, _P, C.c_int32, _P, C.c_int64, C.POINTER(CmgbConfig),
         C.POINTER(CmgbManifoldOut), _P],
    ),
    "cmgb_manifold_scene_batch_host": (
        _I,
        [C.POINTER(_P), C.c_int32, _P, C.c_int32, _P, C.c_int64, C.POINTER(CmgbConfig), _P, _P],
    ),
}

_lib = None


class CmgbError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


def load() -> C.CDLL:
    """Load libcmgb.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the contact-manifold path)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != CMGB_OK:
        msg = load().cmgb_last_error()
        raise CmgbError(status, msg.decode() if msg else "")
