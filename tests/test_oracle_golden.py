"""CPU: pin the oracle (oracle/cmg_oracle.c) to the compiled reference's golden
vectors (tests/golden, made by tests/golden/make_golden.py) and to the
reference's own known-answer examples (SPEC.md, proj/tests/*.cpp)."""
import math
import os

import numpy as np
import pytest

from cases import SDF_PROGRAMS, manifold_cases
from oracle import Oracle
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.scene import SmoothingConfig, Superquadric, box_planes

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"), allow_pickle=False)


def close(a, b, rtol=1e-10, atol=1e-12):
    return np.allclose(a, b, rtol=rtol, atol=atol)


@pytest.mark.parametrize("var", ["ours", "ours_ns"])
def test_ee_witness_matches_reference(var):
    g = gold("witness")
    out, _ = Oracle.ee_witness(g["pairs"], SmoothingConfig().for_variant(var))
    assert close(out, g[f"ee_{var}"])
    assert math.isclose(out[:, :6].sum(), float(g[f"ee_checksum_{var}"]), rel_tol=1e-12)


@pytest.mark.parametrize("var", ["ours", "ours_ns"])
def test_vf_witness_matches_reference(var):
    g = gold("witness")
    out, _ = Oracle.vf_witness(g["pairs"], SmoothingConfig().for_variant(var))
    assert close(out, g[f"vf_{var}"])


@pytest.mark.parametrize("var", ["ours", "ours_ns"])
def test_box_qp_matches_reference(var):
    g = gold("box_qp")
    assert close(Oracle.box_qp(g["qp"], SmoothingConfig().for_variant(var)), g[var])


@pytest.mark.parametrize("name", sorted(SDF_PROGRAMS))
def test_sdf_fields_match_reference(name):
    g = gold("sdf")
    box = api.Mesh.box((0.5, 0.5, 0.5))
    s = Oracle.Surface(box.vertices, box.edges, SDF_PROGRAMS[name])
    for fl in (0, 1, 2):
        got = s.sdf_query(fl, g["points"])
        ref = g[f"{name}_f{fl}"]
        # analytic gradients vs the reference's nested Dual<3>: same expression graph
        assert np.allclose(got, ref, rtol=1e-9, atol=1e-11), (name, fl, np.abs(got - ref).max())
    tr = s.sphere_trace([0.1, -0.2, 0.3, 0.2, 0.1, -0.3], g["points"][:50], 5)
    assert np.allclose(tr, g[f"{name}_trace5"], rtol=1e-8, atol=1e-10)


def test_soft_topk_matches_reference():
    g = gold("soft_topk")
    for i, x in enumerate(g["xs"]):
        assert close(Oracle.soft_topk(x, 4, 0.1), g[f"w{i}"])


@pytest.mark.parametrize("case", [c[0] for c in manifold_cases()])
def test_manifold_matches_reference(case):
    g = gold(f"manifold_{case}")
    name, ws, cfg, n = [c for c in manifold_cases() if c[0] == case][0]
    meshes = [api.surface_from_spec(b).mesh for b in ws.bodies[:2]]
    s = [Oracle.Surface(m.vertices, m.edges, b.sdf, b.vertex_topk, b.edge_topk)
         for m, b in zip(meshes, ws.bodies[:2])]
    r = Oracle.manifold_batch(s[0], s[1], g["poses1"], g["poses2"], cfg, threads=2)
    assert np.array_equal(r["layout"], g["layout"])
    assert np.array_equal(r["meta"], g["meta"])  # kinds, sides, provenance: bit-exact
    assert np.allclose(r["contacts"], g["contacts"], rtol=1e-9, atol=1e-10), np.abs(r["contacts"] - g["contacts"]).max()
    assert np.allclose(r["mean_dist"], g["mean_dist"], rtol=1e-12, atol=1e-14)
    one = Oracle.manifold(s[0], s[1], g["poses1"][0], g["poses2"][0], cfg)
    assert np.allclose(one["ee"], g["ee0"], rtol=1e-9, atol=1e-10)


# ---- known answers (SPEC.md; proj/tests/*.cpp) --------------------------------
def test_spec_witness_examples():
    c = SmoothingConfig()
    # Q = I, c = (-1/2, -1/2): alpha = (1/2, 1/2), gamma_con = 0.973496
    a = Oracle.box_qp([[1, 0, 1, -0.5, -0.5]], c)[0]
    assert np.allclose(a[:2], [0.5, 0.5], atol=1e-12) and abs(a[2] - 0.973496) < 1e-6
    # hard: Q = I, c = (-2, -1/2) -> (1, 1/2)
    a = Oracle.box_qp([[1, 0, 1, -2.0, -0.5]], c.for_variant("ours_ns"))[0]
    assert np.allclose(a[:2], [1.0, 0.5], atol=1e-12)
    # perpendicular crossing edges -> p1 = (0,0,0), p2 = (0,0,1), alpha = (1/2, 1/2)
    out, _ = Oracle.ee_witness([[-1, 0, 0, 1, 0, 0, 0, -1, 1, 0, 1, 1]], c)
    assert np.allclose(out[0, :6], [0, 0, 0, 0, 0, 1], atol=1e-12)
    # parallel edges: lambda > 0 pins alpha to (1/2, 1/2)
    out, _ = Oracle.ee_witness([[0, 0, 0, 1, 0, 0, 0, 0, 1, 1, 0, 1]], c)
    assert np.allclose(out[0, 6:8], [0.5, 0.5], atol=1e-9)
    # V-F: above the interior -> orthogonal projection; beyond the hypotenuse (hard)
    out, _ = Oracle.vf_witness([[0.25, 0.25, 1, 0, 0, 0, 1, 0, 0, 0, 1, 0]], c.for_variant("ours_ns"))
    assert np.allclose(out[0], [0.25, 0.25, 0.0], atol=1e-9)
    out, _ = Oracle.vf_witness([[2, 2, 0, 0, 0, 0, 1, 0, 0, 0, 1, 0]], c.for_variant("ours_ns"))
    assert np.allclose(out[0], [0.5, 0.5, 0.0], atol=1e-9)


def test_spec_sdf_examples():
    box = api.Mesh.box((1.0, 1.0, 1.0))
    sph = Oracle.Surface(box.vertices, box.edges, Superquadric(1.0, 1.0, (1.0, 1.0, 1.0)))
    v = sph.sdf_query(0, [[0, 0, 1], [0, 0, 2], [0, 0, 0.5]])[:, 0]
    assert np.allclose(v, [0.0, 0.25, -2.0], atol=1e-12)  # SPEC.md sq_sdf examples
    cube = Oracle.Surface(box.vertices, box.edges, box_planes((0.5, 0.5, 0.5), tau=1e-6))
    v = cube.sdf_query(0, [[0, 0, 0], [2, 0, 0]])[:, 0]
    assert abs(v[0] + 0.5) < 1e-5 and abs(v[1] - 1.5) < 1e-5


def test_spec_soft_topk_examples():
    w = Oracle.soft_topk([3.0, 1.0, 2.0], 2, 1e-6)
    assert np.allclose(w, [[1, 0, 0], [0, 0, 1]], atol=1e-12)
    assert np.allclose(Oracle.soft_topk([0.0, 0.0], 1, 0.1), [[0.5, 0.5]])
    with pytest.raises(ValueError):
        Oracle.soft_topk([1.0, 2.0], 3, 0.1)


def _box_qp_bruteforce(q, grid=201):
    """box_qp_oracle (proj/tests/test_helpers.hpp:50-70): grid seed + exact
    coordinate descent."""
    q11, q12, q22, c1, c2 = q
    a = np.linspace(0, 1, grid)
    A, B = np.meshgrid(a, a, indexing="ij")
    cost = 0.5 * (q11 * A * A + 2 * q12 * A * B + q22 * B * B) + c1 * A + c2 * B
    i, j = np.unravel_index(np.argmin(cost), cost.shape)
    x, y = a[i], a[j]
    for _ in range(200):
        x = min(max(-(c1 + q12 * y) / q11, 0.0), 1.0)
        y = min(max(-(c2 + q12 * x) / q22, 0.0), 1.0)
    return x, y


def test_acceptance_hard_qp_vs_bruteforce():
    """SPEC acceptance #1 (hard QP vs brute force), on 300 random PD QPs."""
    rng = np.random.default_rng(1)
    cfg = SmoothingConfig(lambda_=1e-6, hard_ops=True)
    qps = []
    for _ in range(300):
        A = rng.normal(size=(2, 2))
        Q = A @ A.T + 1e-2 * np.eye(2)
        c = rng.normal(size=2)
        qps.append([Q[0, 0], Q[0, 1], Q[1, 1], c[0], c[1]])
    got = Oracle.box_qp(np.array(qps), cfg)
    for q, g in zip(qps, got):
        x, y = _box_qp_bruteforce(q)
        f = lambda a, b: 0.5 * (q[0] * a * a + 2 * q[1] * a * b + q[2] * b * b) + q[3] * a + q[4] * b
        assert f(g[0], g[1]) - f(x, y) < 1e-6


def test_mt19937_matches_reference_generator():
    g = gold("witness")
    from paper_2602_20304_b200.workloads import mt19937_64_uniform
    assert np.array_equal(mt19937_64_uniform(0, 24000, 0.0, 1.0), g["pairs"].reshape(-1))
    assert np.array_equal(Oracle.uniform(0, 24000), g["pairs"].reshape(-1))


def test_scene_pairs_match_reference():
    """Config D: every body pair of the multi-body drop scene (DemoSim::step
    pair loop, src/demosim.cpp:88-104)."""
    from paper_2602_20304_b200 import workloads as W
    g = gold("scene_drop")
    sc = W.drop_scene(4)
    assert np.array_equal(api.scene_pairs(len(sc.bodies), sc.is_static()), g["pairs"])
    meshes = [api.surface_from_spec(b).mesh for b in sc.bodies]
    s = [Oracle.Surface(m.vertices, m.edges, b.sdf, b.vertex_topk, b.edge_topk)
         for m, b in zip(meshes, sc.bodies)]
    P = g["poses"]
    for q, (i, j) in enumerate(g["pairs"]):
        r = Oracle.manifold_batch(s[i], s[j], P[:, i], P[:, j], SmoothingConfig(), threads=2)
        assert np.array_equal(r["meta"], g[f"meta{q}"])
        assert np.allclose(r["contacts"], g[f"contacts{q}"], rtol=1e-9, atol=1e-10)
