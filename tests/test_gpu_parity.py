"""GPU parity: the sm_100a path through the C ABI vs (a) the compiled
reference's golden fixtures and (b) the C oracle on the same seeded inputs;
plus size-independent properties at BASELINE sizes (65,536 envs).

Tolerance (north star, tests/helpers.py): 1e-6 absolute + 1e-5 relative on
points, distances, normals (3-vectors compared as vectors) and activities;
provenance (src_a/src_b) and active-set labels bit-exact except at documented
near-ties."""
import os

import numpy as np
import pytest
import torch

from cases import manifold_cases
from helpers import assert_parity, scalar_close, surfaces
from oracle import Oracle
from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FLT_EPS = np.finfo(np.float32).eps


def gold(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"), allow_pickle=False)


def run_gpu(ws, cfg, p1, p2, **kw):
    a1, a2 = (api.surface_from_spec(b) for b in ws.bodies[:2])
    r = api.generate_manifold_batch(a1, a2, torch.as_tensor(p1, device="cuda"),
                                    torch.as_tensor(p2, device="cuda"), cfg, want_src=True,
                                    want_ee=True, **kw)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in r.items()}


CASES = {c[0]: c for c in manifold_cases()}


@pytest.mark.parametrize("case", sorted(CASES))
def test_manifold_vs_reference_golden(cuda, case):
    g = gold(f"manifold_{case}")
    _, ws, cfg, _ = CASES[case]
    r = run_gpu(ws, cfg, g["poses1"], g["poses2"])
    assert_parity(r["contacts"], g["contacts"], what=f"{case} vs reference")
    assert np.array_equal(r["src"], g["meta"][..., 2:]), "provenance differs from the reference"
    assert scalar_close(r["mean_dist"], g["mean_dist"]).all()


@pytest.mark.parametrize("case,n", [("box_box_ours", 512), ("box_box_ours_ns", 512),
                                    ("box_on_plane_ours", 256), ("box_box_topk", 256),
                                    ("mixed_rounded_box", 128), ("mixed_cylinder", 128),
                                    ("mixed_ellipsoid", 128), ("mixed_capsule", 128),
                                    ("opc_vs_box", 128), ("subtraction_vs_box", 128),
                                    ("box_box_containment", 128), ("box_box_ours_ne", 1024)])
def test_manifold_vs_oracle(cuda, case, n):
    _, ws, cfg, _ = CASES[case]
    (_, _), (o1, o2) = surfaces(ws)
    p1, p2 = ws.poses(n)
    ref = Oracle.manifold_batch(o1, o2, p1, p2, cfg, want_ee=True)
    r = run_gpu(ws, cfg, p1, p2)
    assert_parity(r["contacts"], ref["contacts"], what=f"{case} vs oracle")
    assert np.array_equal(r["src"], ref["meta"][..., 2:])
    assert scalar_close(r["mean_dist"], ref["mean_dist"]).all()
    if ref["ee"] is not None and ref["ee"].shape[-1]:
        assert scalar_close(r["ee"], ref["ee"]).all(), "EE indicator matrices differ"


def test_full_size_properties(cuda):
    """Config B at its full size: 65,536 envs (304 contacts each)."""
    n = 65536
    ws = W.box_box(n)
    p1, p2 = ws.poses(n)
    cfg = SmoothingConfig()
    full = run_gpu(ws, cfg, p1, p2)
    c = full["contacts"]
    assert c.shape == (n, 304, 8) and np.isfinite(c).all()
    assert (c[..., 7] >= 0).all() and (c[..., 7] <= 1).all()
    assert (np.linalg.norm(c[..., 4:7], axis=-1) <= 1 + 1e-6).all()
    # prefix property: the first N envs of the batch equal the N-env batch (bitwise)
    head = run_gpu(ws, cfg, p1, p2[:300])
    assert np.array_equal(head["contacts"], c[:300])
    # sharding: two contiguous halves reproduce the full batch bitwise
    h0 = run_gpu(ws, cfg, p1, p2[: n // 2])
    h1 = run_gpu(ws, cfg, p1, p2[n // 2:])
    assert np.array_equal(np.concatenate([h0["contacts"], h1["contacts"]]), c)
    # determinism
    again = run_gpu(ws, cfg, p1, p2)
    assert np.array_equal(again["contacts"], c)
    # oracle spot check on a scattered sample of envs across the batch
    idx = np.linspace(0, n - 1, 64).astype(int)
    (_, _), (o1, o2) = surfaces(ws)
    ref = Oracle.manifold_batch(o1, o2, p1, p2[idx], cfg)
    assert_parity(c[idx], ref["contacts"], what="65536-env sample vs oracle")


def test_shared_pose_broadcast_equals_explicit(cuda):
    ws = W.box_box(64)
    p1, p2 = ws.poses(64)
    a = run_gpu(ws, SmoothingConfig(), p1, p2)  # body-1 pose stride 0
    b = run_gpu(ws, SmoothingConfig(), np.repeat(p1, 64, axis=0), p2)
    assert np.array_equal(a["contacts"], b["contacts"])


def test_host_api_matches_device_api(cuda):
    ws = W.box_box(1000)
    p1, p2 = ws.poses(1000)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    dev = run_gpu(ws, SmoothingConfig(), p1, p2)
    contacts = np.empty_like(dev["contacts"])
    mean = api.generate_manifold_batch_host(s1, s2, p1, p2, SmoothingConfig(), contacts_out=contacts)
    assert np.array_equal(mean, dev["mean_dist"]) and np.array_equal(contacts, dev["contacts"])


@pytest.mark.parametrize("n", [4095, 4099, 20001, 33333])
def test_host_api_pipelined_chunks(cuda, n):
    """The host-buffer call pipelines a lead chunk (1/8 of the envs, at least
    2,048) and the rest over two streams (one chunk below 4,096 envs): results
    equal the device call bit for bit."""
    ws = W.box_box(n)
    p1, p2 = ws.poses(n)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    dev = run_gpu(ws, SmoothingConfig(), p1, p2)
    contacts = np.empty_like(dev["contacts"])
    mean = api.generate_manifold_batch_host(s1, s2, p1, p2, SmoothingConfig(), contacts_out=contacts)
    assert np.array_equal(mean, dev["mean_dist"]) and np.array_equal(contacts, dev["contacts"])
    mean2 = api.generate_manifold_batch_host(s1, s2, np.repeat(p1, n, axis=0), p2, SmoothingConfig())
    assert np.array_equal(mean2, dev["mean_dist"])


def test_single_env_reference_api(cuda):
    """generate_manifold (one env) returns the reference-shaped manifold."""
    g = gold("manifold_box_on_plane_ours")
    ws = W.box_on_plane()
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    m = api.generate_manifold(s1, s2, g["poses1"][0], g["poses2"][0], SmoothingConfig())
    assert np.array_equal(m["meta"], g["meta"][0])
    assert_parity(m["contacts"], g["contacts"][0], what="single env")


# ---- witness batches (K6) ------------------------------------------------------
def _ee_near_tie(pairs, cfg):
    """Near-tie set for E-E labels: argmin gap or box-edge
    margin within 64 FLT_EPSILON (1 + scale), recomputed in FP64."""
    e1a, e1b, e2a, e2b = pairs[:, 0:3], pairs[:, 3:6], pairs[:, 6:9], pairs[:, 9:12]
    t1, t2n, b = e1b - e1a, e2a - e2b, e1a - e2a
    q1 = (t1 * t1).sum(1) + cfg.lambda_
    q2 = (t1 * t2n).sum(1)
    q3 = (t2n * t2n).sum(1) + cfg.lambda_
    c1 = (b * t1).sum(1) - 0.5 * cfg.lambda_
    c2 = (b * t2n).sum(1) - 0.5 * cfg.lambda_
    a1u = (q2 * (c2 / q3) - c1) / (q1 - q2 * (q2 / q3))
    a2u = (q2 * (c1 / q1) - c2) / (q3 - q2 * (q2 / q1))
    cl = lambda x: np.clip(x, 0, 1)
    x11, x10 = cl(-(q2 / q3 + c2 / q3)), cl(-c2 / q3)
    x21, x20 = cl(-(q2 / q1 + c1 / q1)), cl(-c1 / q1)
    cost = np.stack([0.5 * (q1 + 2 * q2 * x11 + q3 * x11 ** 2) + c1 + c2 * x11, 0.5 * q3 * x10 ** 2 + c2 * x10,
                     0.5 * (q1 * x21 ** 2 + 2 * q2 * x21 + q3) + c1 * x21 + c2, 0.5 * q1 * x20 ** 2 + c1 * x20], 1)
    s = np.sort(cost, 1)
    tie = (s[:, 1] - s[:, 0]) <= 64 * FLT_EPS * (1 + np.abs(cost).max(1))
    for a in (a1u, a2u):
        tie |= (np.abs(a) <= 64 * FLT_EPS * (1 + np.abs(a))) | (np.abs(a - 1) <= 64 * FLT_EPS * (1 + np.abs(a)))
    return tie


def _vf_near_tie(pairs):
    """Hard V-F label near-ties: equal clipped-edge distances (vertex regions)."""
    v, t0, t1, t2 = pairs[:, 0:3], pairs[:, 3:6], pairs[:, 6:9], pairs[:, 9:12]
    costs = []
    for a, bb in ((t0, t1), (t1, t2), (t0, t2)):
        d = bb - a
        ln = np.sqrt((d * d).sum(1) + 1e-12)
        u = d / ln[:, None]
        s = np.clip(((v - a) * u).sum(1), 0, ln)
        costs.append(np.linalg.norm(v - (a + u * s[:, None]), axis=1))
    cost = np.stack(costs, 1)
    s = np.sort(cost, 1)
    return (s[:, 1] - s[:, 0]) <= 64 * FLT_EPS * (1 + cost.max(1))


@pytest.mark.parametrize("var", ["ours", "ours_ns"])
def test_ee_witness_vs_reference_golden(cuda, var):
    g = gold("witness")
    cfg = SmoothingConfig().for_variant(var)
    r = api.run_ee_batch(torch.as_tensor(g["pairs"], device="cuda"), cfg, want_alpha=True)
    torch.cuda.synchronize()
    ref = g[f"ee_{var}"]
    got = r["out"].cpu().numpy()
    for k in (0, 3):
        err = np.linalg.norm(got[:, k:k + 3] - ref[:, k:k + 3], axis=1)
        assert (err <= 1e-6 + 1e-5 * np.linalg.norm(ref[:, k:k + 3], axis=1)).all()
    assert scalar_close(r["alpha_gamma"].cpu().numpy(), ref[:, 6:9]).all()


@pytest.mark.parametrize("var", ["ours", "ours_ns"])
def test_vf_witness_vs_reference_golden(cuda, var):
    g = gold("witness")
    r = api.run_vf_batch(torch.as_tensor(g["pairs"], device="cuda"), SmoothingConfig().for_variant(var))
    got = r["out"].cpu().numpy()
    ref = g[f"vf_{var}"]
    err = np.linalg.norm(got - ref, axis=1)
    assert (err <= 1e-6 + 1e-5 * np.linalg.norm(ref, axis=1)).all()


@pytest.mark.parametrize("var", ["ours", "ours_ns"])
@pytest.mark.parametrize("fp64", [True, False])
def test_witness_batches_vs_oracle(cuda, var, fp64):
    n = 200_000
    cfg = SmoothingConfig().for_variant(var)
    pairs = W.mt19937_64_uniform(1, 12 * n, 0.0, 1.0).reshape(n, 12)
    if not fp64:
        pairs = pairs.astype(np.float32).astype(np.float64)  # same values, FP32 storage
    dev = torch.as_tensor(pairs if fp64 else pairs.astype(np.float32), device="cuda")
    ee = api.run_ee_batch(dev, cfg, want_labels=True)
    vf = api.run_vf_batch(dev, cfg, want_labels=True)
    ref_ee, lab_ee = Oracle.ee_witness(pairs, cfg)
    ref_vf, lab_vf = Oracle.vf_witness(pairs, cfg)
    got = ee["out"].cpu().numpy()
    for k in (0, 3):
        err = np.linalg.norm(got[:, k:k + 3] - ref_ee[:, k:k + 3], axis=1)
        assert (err <= 1e-6 + 1e-5 * np.linalg.norm(ref_ee[:, k:k + 3], axis=1)).all()
    err = np.linalg.norm(vf["out"].cpu().numpy() - ref_vf, axis=1)
    assert (err <= 1e-6 + 1e-5 * np.linalg.norm(ref_vf, axis=1)).all()
    # active-set labels: bit-exact outside documented near-ties
    bad = ee["labels"].cpu().numpy() != lab_ee
    assert not (bad & ~_ee_near_tie(pairs, cfg)).any(), int((bad & ~_ee_near_tie(pairs, cfg)).sum())
    bad = vf["labels"].cpu().numpy() != lab_vf
    tie = _vf_near_tie(pairs) if cfg.hard_ops else np.zeros(n, bool)
    assert not (bad & ~tie).any(), int((bad & ~tie).sum())


def test_invalid_config_fails_loudly(cuda):
    ws = W.box_box(4)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p = torch.zeros((4, 6), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="smoothing: tau_pen must be > 0"):
        api.generate_manifold_batch(s1, s2, p, p, SmoothingConfig(tau_pen=-1.0))


def test_scene_batch_all_pairs(cuda):
    """Config D shape: all body pairs of the drop scene in one scene call,
    vs the reference (golden) and the oracle at a larger batch."""
    g = gold("scene_drop")
    sc = W.drop_scene(4)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    res = api.generate_manifold_scene_batch(bodies, torch.as_tensor(g["poses"], device="cuda"), SmoothingConfig(),
                                            is_static=sc.is_static(), want_src=True)
    torch.cuda.synchronize()
    assert [r["pair"] for r in res] == [tuple(p) for p in g["pairs"]]
    for q, r in enumerate(res):
        assert_parity(r["contacts"].cpu().numpy(), g[f"contacts{q}"], what=f"scene pair {r['pair']}")
        assert np.array_equal(r["src"].cpu().numpy(), g[f"meta{q}"][..., 2:])
    n = 512
    P = sc.poses(n)
    res = api.generate_manifold_scene_batch(bodies, torch.as_tensor(P, device="cuda"), SmoothingConfig(),
                                            is_static=sc.is_static(), want_src=True)
    torch.cuda.synchronize()
    meshes = [b.mesh for b in bodies]
    o = [Oracle.Surface(m.vertices, m.edges, b.sdf, b.vertex_topk, b.edge_topk) for m, b in zip(meshes, sc.bodies)]
    for r in res:
        i, j = r["pair"]
        ref = Oracle.manifold_batch(o[i], o[j], P[:, i], P[:, j], SmoothingConfig())
        assert_parity(r["contacts"].cpu().numpy(), ref["contacts"], what=f"scene pair {(i, j)} vs oracle")
        assert np.array_equal(r["src"].cpu().numpy(), ref["meta"][..., 2:])


@pytest.mark.parametrize("name", list(__import__("cases").SDF_PROGRAMS))
def test_sdf_queries_vs_reference_golden(cuda, name):
    """The device field code directly: values, true
    gradients and normal sources of every SDF program, and 5-step sphere traces
    of a posed surface, vs the reference's (tests/golden/sdf.npz)."""
    from cases import SDF_PROGRAMS
    g = gold("sdf")
    s = api.Surface(api.Mesh.box((0.5, 0.5, 0.5)), SDF_PROGRAMS[name])
    pts = torch.as_tensor(g["points"], device="cuda")
    for fl in (0, 1, 2):
        got = api.sdf_query(s, pts, fl).cpu().numpy()
        ref = g[f"{name}_f{fl}"]
        err = np.abs(got - ref) / (1e-11 + 1e-9 * np.abs(ref))
        assert err.max() <= 1.0, (name, fl, float(err.max()))
    tr = api.sphere_trace(s, [0.1, -0.2, 0.3, 0.2, 0.1, -0.3], pts[:50], 5).cpu().numpy()
    assert np.allclose(tr, g[f"{name}_trace5"], rtol=1e-8, atol=1e-10), np.abs(tr - g[f"{name}_trace5"]).max()
