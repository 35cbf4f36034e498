"""Scene documents and text outputs vs the compiled reference (CPU): parse_scene
/ load_scene (src/scene.cpp), write_manifold_csv / manifold_to_json
(src/manifold_io.cpp), write_sweep_csv (src/sweep.cpp) -- same bodies, same
smoothing block, same manifolds, byte-identical text for the same numbers."""
import io
import json
import os

import numpy as np
import pytest

from oracle import Oracle, Ref
from paper_2602_20304_b200 import scene_io

SCENES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenes")
NAMES = ["box_on_plane", "capsule_vs_hollow"]

pytestmark = pytest.mark.skipif(not Ref.available(), reason="compiled reference (oracle/_ref) not built")


def load_both(name):
    path = os.path.join(SCENES, f"{name}.json")
    return scene_io.load_scene(path), Ref.SceneHandle(open(path).read(), SCENES)


@pytest.mark.parametrize("name", NAMES)
def test_parse_scene_matches_reference(name):
    ours, ref = load_both(name)
    assert len(ours.bodies) == len(ref.bodies)
    for b, r in zip(ours.bodies, ref.bodies):
        assert b.name == r["name"] and b.is_static == r["is_static"]
        assert np.array_equal(b.pose, r["pose"]) and b.mass == r["mass"]
        assert np.array_equal(b.inertia_diag, r["inertia"])
        assert (b.vertex_topk, b.edge_topk) == (r["vertex_topk"], r["edge_topk"])
    c = ours.smoothing.to_c()
    for f, _ in c._fields_:
        assert getattr(c, f) == getattr(ref.smoothing, f), f
    # same geometry + SDF program + budgets: the C oracle on our parsed bodies
    # reproduces the reference's manifold of the parsed scene
    o = [Oracle.Surface(b.surface.mesh.vertices, b.surface.mesh.edges, b.sdf, b.vertex_topk, b.edge_topk)
         for b in ours.bodies]
    got = Oracle.manifold(o[0], o[1], ours.bodies[0].pose, ours.bodies[1].pose, ours.smoothing)
    want = Ref.manifold(ref.bodies[0]["surface"], ref.bodies[1]["surface"], ref.bodies[0]["pose"],
                        ref.bodies[1]["pose"], ref.smoothing)
    assert np.array_equal(got["meta"], want["meta"])
    assert np.allclose(got["contacts"], want["contacts"], rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("doc, msg", [
    ('{"bodies": []}', "scene: needs a non-empty 'bodies' array"),
    ('{"smoothing": {"mode": "sideways"}, "bodies": [{}]}', "mode must be one of: full, no-ee, one-sided"),
    ('{"bodies": [{"mesh": {"box": {"half_extents": [1, 1, 1]}}, "sdf": {"type": "blob"}, "pose": [0,0,0,0,0,0]}]}',
     "unknown sdf node type: blob"),
    ('{"bodies": [{"mesh": {"box": {"half_extents": [1, 1, 1]}}, "pose": [0,0,0,0,0,0], "mass": -1,'
     ' "sdf": {"type": "superquadric", "eps1": 1, "eps2": 1, "axes": [1, 1, 1]}}]}', "body mass must be positive"),
    ('{"bodies": [{"mesh": {"sphere": 1}, "pose": [0,0,0,0,0,0],'
     ' "sdf": {"type": "superquadric", "eps1": 1, "eps2": 1, "axes": [1, 1, 1]}}]}',
     "mesh: expected an 'obj' path or a 'box' generator"),
])
def test_scene_errors_match_reference(doc, msg):
    with pytest.raises(ValueError) as ours:
        scene_io.parse_scene(doc)
    with pytest.raises(ValueError) as ref:
        Ref.SceneHandle(doc)
    assert str(ours.value) == msg and msg in str(ref.value)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("as_json", [False, True])
def test_manifold_text_byte_identical(name, as_json):
    """Our writers on the reference's own manifold numbers give the reference's text."""
    _, ref = load_both(name)
    r0, r1 = ref.bodies[0], ref.bodies[1]
    want = Ref.manifold_text(r0["surface"], r1["surface"], r0["pose"], r1["pose"], ref.smoothing, as_json)
    m = Ref.manifold(r0["surface"], r1["surface"], r0["pose"], r1["pose"], ref.smoothing)
    if as_json:
        L = m["layout"]
        got = scene_io.manifold_to_json(m["contacts"], m["meta"],
                                        dict(n1=L[0], n2=L[1], m1=L[2], m2=L[3], mode=ref.smoothing.mode)) + "\n"
        assert json.loads(got) == json.loads(want)
    else:
        f = io.StringIO()
        scene_io.write_manifold_csv(f, m["contacts"], m["meta"])
        got = f.getvalue()
    assert got == want


def test_sweep_csv_byte_identical():
    n = 101
    f = io.StringIO()
    scene_io.write_sweep_csv(f, Ref.sweep(0, n), Ref.sweep(1, n), Ref.sweep(2, n))
    assert f.getvalue() == Ref.sweep_csv(n)
