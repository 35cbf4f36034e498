"""CPU: the C-ABI library loads, exports every symbol include/cmgb.h declares,
and its host-side logic (mesh ingest, surface build checks, config, layout)
matches the reference (golden fixtures). No compute calls: no GPU here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from cases import BOX_MESHES, OBJ_ERRORS, OBJ_TEXTS, manifold_cases
from paper_2602_20304_b200 import abi, api
from paper_2602_20304_b200.scene import SmoothingConfig, Superquadric, box_planes, ConvexPolyhedron, Union

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def gold(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"), allow_pickle=False)


def header_symbols():
    text = open(os.path.join(ROOT, "include", "cmgb.h")).read()
    return sorted(set(re.findall(r"\b(cmgb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = abi.load()
    syms = header_symbols()
    assert len(syms) >= 24
    for s in syms:
        assert hasattr(lib, s), f"libcmgb.so does not export {s}"
    assert set(syms) == set(abi.SIGNATURES), "ctypes mirror out of sync with include/cmgb.h"
    assert lib.cmgb_abi_version() == 2


def test_library_is_native_cuda_for_sm100a():
    """The product is the in-tree sm_100a library (no CPU fallback exists)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_config_matches_reference_defaults():
    lib = abi.load()
    c = abi.CmgbConfig()
    lib.cmgb_config_default(C.byref(c))
    ref = SmoothingConfig().to_c()  # config.hpp:17-46
    for f, _ in abi.CmgbConfig._fields_:
        assert getattr(c, f) == getattr(ref, f), f
    lib.cmgb_config_no_smoothing(C.byref(c))
    assert c.lambda_ == 1e-6 and c.hard_ops == 1


@pytest.mark.parametrize("variant", ["ours", "ours_ns", "ours_ne", "ours_ne_s"])
def test_config_for_variant(variant):
    lib = abi.load()
    base = SmoothingConfig().to_c()
    out = abi.CmgbConfig()
    assert lib.cmgb_config_for_variant(variant.encode(), C.byref(base), C.byref(out)) == 0
    ref = SmoothingConfig().for_variant(variant).to_c()
    for f, _ in abi.CmgbConfig._fields_:
        assert getattr(out, f) == getattr(ref, f)


def test_config_validation_messages():
    lib = abi.load()
    c = SmoothingConfig(tau_nn=0.0).to_c()
    assert lib.cmgb_config_validate(C.byref(c)) == abi.CMGB_OK + 1
    assert lib.cmgb_last_error().decode() == "smoothing: tau_nn must be > 0"
    c = SmoothingConfig(sphere_trace_iters=-1).to_c()
    assert lib.cmgb_config_validate(C.byref(c)) == 1
    assert lib.cmgb_last_error().decode() == "smoothing: sphere_trace_iters >= 0"
    out = abi.CmgbConfig()
    assert lib.cmgb_config_for_variant(b"nope", C.byref(c), C.byref(out)) == 1
    assert "unknown variant: nope" in lib.cmgb_last_error().decode()


@pytest.mark.parametrize("i", range(len(BOX_MESHES)))
def test_box_mesh_matches_reference(i):
    g = gold("meshes")
    half, sub, quad = BOX_MESHES[i]
    m = api.Mesh.box(half, sub, quad)
    assert np.array_equal(m.vertices, g[f"box{i}_v"])
    assert np.array_equal(m.faces, g[f"box{i}_f"])
    assert np.array_equal(m.edges, g[f"box{i}_e"])  # candidate (src) order


@pytest.mark.parametrize("name", sorted(OBJ_TEXTS))
def test_obj_ingest_matches_reference(name):
    g = gold("meshes")
    m = api.Mesh.parse_obj(OBJ_TEXTS[name])
    assert np.array_equal(m.vertices, g[f"obj_{name}_v"])
    assert np.array_equal(m.faces, g[f"obj_{name}_f"])
    assert np.array_equal(m.edges, g[f"obj_{name}_e"])
    assert m.warnings == list(g[f"obj_{name}_w"])


@pytest.mark.parametrize("name", sorted(OBJ_ERRORS))
def test_obj_errors_match_reference(name):
    g = gold("meshes")
    want, line = str(g[f"err_{name}"]).rsplit("|", 1)  # MeshParseError what() | line_number
    with pytest.raises(api.MeshParseError) as e:
        api.Mesh.parse_obj(OBJ_ERRORS[name])
    assert str(e.value) == want
    assert e.value.line_number == int(line)


def test_surface_validation_messages():
    box = api.Mesh.box((0.5, 0.5, 0.5))
    with pytest.raises(ValueError, match=r"superquadric: eps1, eps2 must lie in \(0, 2\]"):
        api.Surface(box, Superquadric(2.5, 1.0, (1, 1, 1)))
    with pytest.raises(ValueError, match="superquadric: axis lengths must be positive"):
        api.Surface(box, Superquadric(1.0, 1.0, (1, 0, 1)))
    with pytest.raises(ValueError, match="must lie in \\[1, V\\]"):
        api.Surface(box, Superquadric(), vertex_topk=9)
    with pytest.raises(ValueError, match="must lie in \\[1, E\\]"):
        api.Surface(box, Superquadric(), edge_topk=13)
    with pytest.raises(ValueError, match="convex polyhedron: normals must be unit length"):
        api.Surface(box, ConvexPolyhedron(np.array([[0, 0, 2.0]]), np.zeros((1, 3))))
    with pytest.raises(ValueError, match="smooth_union: tau > 0"):
        api.Surface(box, Union([Superquadric()], 0.0))
    bad = api.Mesh.from_arrays(box.vertices, box.faces, np.array([[0, 9]]))
    with pytest.raises(ValueError, match="surface: edge index out of range"):
        api.Surface(bad, Superquadric())


@pytest.mark.parametrize("case", [c[0] for c in manifold_cases()])
def test_layout_and_warnings_match_reference(case):
    g = gold(f"manifold_{case}")
    _, ws, cfg, _ = [c for c in manifold_cases() if c[0] == case][0]
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies[:2])
    L = api.layout(s1, s2, cfg)
    assert [L["n1"], L["n2"], L["m1"], L["m2"], L["n_contacts"]] == list(g["layout"])
    meta = api.layout_metadata(s1, s2, cfg)
    ref = g["meta"][0]
    assert np.array_equal(meta[:, :2], ref[:, :2])  # kinds and sides are static
    static = meta[:, 2:] >= 0
    assert np.array_equal(meta[:, 2:][static], ref[:, 2:][static])
    assert (s1.build_warnings + ["|"] + s2.build_warnings) == list(g["warnings"])


def test_effective_budgets():
    box = api.Mesh.box((0.5, 0.5, 0.5))
    s = api.Surface(box, Superquadric())  # edge_topk 0 -> leaf count (surface.hpp:28-32)
    assert s.effective_vertex_topk() == 8 and s.effective_edge_topk() == 1
    s = api.Surface(box, Union([Superquadric(), Superquadric(), box_planes((0.5, 0.5, 0.5))], 0.01))
    assert s.info["leaf_count"] == 3 and s.effective_edge_topk() == 3


def test_host_buffer_calls_validate_before_touching_the_device():
    """The pipelined host-buffer calls (witness batches, scene batch) reject bad
    arguments with the library's messages before any CUDA work; empty batches
    are no-ops."""
    lib = abi.load()
    good = SmoothingConfig().to_c()
    pairs = np.zeros((4, 12))
    out = np.zeros((4, 6))
    for fn, name in ((lib.cmgb_ee_witness_batch_host, "ee"), (lib.cmgb_vf_witness_batch_host, "vf")):
        assert fn(pairs.ctypes.data, -1, C.byref(good), out.ctypes.data, None, None) != 0
        assert lib.cmgb_last_error().decode() == f"{name}_witness_batch_host: n >= 0"
        assert fn(None, 4, C.byref(good), out.ctypes.data, None, None) != 0
        assert lib.cmgb_last_error().decode() == f"{name}_witness_batch_host: null buffer"
        bad = SmoothingConfig(tau_nn=0.0).to_c()
        assert fn(pairs.ctypes.data, 4, C.byref(bad), out.ctypes.data, None, None) != 0
        assert lib.cmgb_last_error().decode() == "smoothing: tau_nn must be > 0"
        assert fn(None, 0, C.byref(good), None, None, None) == 0
    mean = np.zeros((1, 4), np.float32)
    pr = np.array([[0, 1]], np.int32)
    poses = np.zeros((4, 2, 6))
    assert lib.cmgb_manifold_scene_batch_host(None, 2, pr.ctypes.data, 1, poses.ctypes.data, 4, C.byref(good),
                                              mean.ctypes.data, None) != 0
    assert lib.cmgb_last_error().decode() == "manifold_scene_batch_host: bad argument"
    handles = (C.c_void_p * 2)(None, None)
    assert lib.cmgb_manifold_scene_batch_host(handles, 2, pr.ctypes.data, 1, poses.ctypes.data, 0, C.byref(good),
                                              mean.ctypes.data, None) == 0
    assert lib.cmgb_manifold_scene_batch_host(handles, 2, pr.ctypes.data, 1, poses.ctypes.data, 4, C.byref(good),
                                              mean.ctypes.data, None) != 0
    assert lib.cmgb_last_error().decode() == "manifold_scene_batch: pair index out of range"
