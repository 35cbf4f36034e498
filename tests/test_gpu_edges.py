"""Edge cases of the batched path (GPU): empty batches on every entry point,
ragged batch sizes around the CTA packing, pass-through budgets (K = D) at the
largest shared-memory working set, and the documented limit failing loudly."""
import numpy as np
import pytest
import torch

from helpers import assert_parity, surfaces
from oracle import Oracle
from paper_2602_20304_b200 import abi, api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import PenaltyParams, Superquadric, SmoothingConfig

pytestmark = pytest.mark.gpu


def test_empty_batches_everywhere(cuda):
    ws = W.box_box()
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    z = torch.zeros((0, 6), dtype=torch.float64, device="cuda")
    r = api.generate_manifold_batch(s1, s2, z, z, SmoothingConfig(), want_src=True, want_ee=True)
    assert r["contacts"].shape == (0, 304, 8)
    j = api.generate_manifold_jvp_batch(s1, s2, z, z, SmoothingConfig())
    assert j["tangents"].shape == (0, 304, 8, 12)
    assert api.generate_manifold_batch_host(s1, s2, np.zeros((0, 6)), np.zeros((0, 6))).shape == (0,)
    e = api.run_ee_batch(torch.zeros((0, 12), dtype=torch.float64, device="cuda"))
    assert e["out"].shape == (0, 6)
    v = api.run_vf_batch(torch.zeros((0, 12), dtype=torch.float64, device="cuda"))
    assert v["out"].shape == (0, 3)
    sc = W.drop_scene(0)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    P = torch.zeros((0, len(bodies), 6), dtype=torch.float64, device="cuda")
    assert all(x["contacts"].shape[0] == 0 for x in
               api.generate_manifold_scene_batch(bodies, P, SmoothingConfig(), is_static=sc.is_static()))
    d = api.DemoBatch(bodies, np.ones(len(bodies)), is_static=sc.is_static(), n_env=0)
    d.step(1e-3)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n", [1, 2, 3, 145, 1001])
def test_ragged_batch_sizes(cuda, n):
    """Batch sizes that leave the last CTA partly empty (2 box-box envs per CTA)
    and a mixed-family case (top-K, 4 envs per CTA)."""
    for ws in (W.box_box(n), W.mixed_bucket("capsule", n)):
        (a1, a2), (o1, o2) = surfaces(ws)
        p1, p2 = ws.poses(n)
        ref = Oracle.manifold_batch(o1, o2, p1, p2, SmoothingConfig())
        r = api.generate_manifold_batch(a1, a2, torch.as_tensor(p1, device="cuda"),
                                        torch.as_tensor(p2, device="cuda"), SmoothingConfig(), want_src=True)
        torch.cuda.synchronize()
        assert_parity(r["contacts"].cpu().numpy(), ref["contacts"], what=f"{ws.name} n={n}")
        assert np.array_equal(r["src"].cpu().numpy(), ref["meta"][..., 2:])


def big_boxes(m):
    """Two subdivided boxes with pass-through edge budgets (K = D): m edges each."""
    ws = W.box_box(64)
    for b in ws.bodies:
        b.mesh.subdivisions = 2
        b.edge_topk = m
    return ws


def test_pass_through_large_pair_sets(cuda):
    """All 48 edges of two subdivided boxes (pass-through K = D, P = 2,304 pairs:
    the pair records exceed shared memory and live in the global workspace,
    processed in env chunks) vs the oracle."""
    ws = big_boxes(0)
    a1 = api.surface_from_spec(ws.bodies[0])
    m = a1.mesh.edges.shape[0]
    for b in ws.bodies:
        b.edge_topk = m
    (a1, a2), (o1, o2) = surfaces(ws)
    L = api.layout(a1, a2, SmoothingConfig())
    assert L["m1"] == m and L["m1"] * L["m2"] > 2000
    p1, p2 = ws.poses(16)
    ref = Oracle.manifold_batch(o1, o2, p1, p2, SmoothingConfig())
    r = api.generate_manifold_batch(a1, a2, torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda"),
                                    SmoothingConfig())
    torch.cuda.synchronize()
    assert_parity(r["contacts"].cpu().numpy(), ref["contacts"], what=f"pass-through P={L['m1'] * L['m2']}")


def test_working_set_limit_fails_loudly(cuda):
    """A per-env working set whose slots alone exceed the shared-memory budget
    (2 x 2,352 pass-through edges) is refused with CMGB_ERR_UNSUPPORTED
    (DESIGN.md §3), never silently truncated."""
    ws = W.box_box(4)
    for b in ws.bodies:
        b.mesh.subdivisions = 14
    e = api.surface_from_spec(ws.bodies[0]).mesh.edges.shape[0]
    for b in ws.bodies:
        b.edge_topk = e  # pass-through: all edges (budgets are validated to lie in [1, E])
    a1, a2 = (api.surface_from_spec(b) for b in ws.bodies)
    p = torch.zeros((4, 6), dtype=torch.float64, device="cuda")
    with pytest.raises(abi.CmgbError, match="UNSUPPORTED"):
        api.generate_manifold_batch(a1, a2, p, p, SmoothingConfig())


def test_config_e_size_batch(cuda):
    """1,048,576 envs in one call (config E's size on one GPU, ~10 GB of
    contacts): 64-bit indexing end to end -- the first 4,096 envs and the last
    env equal separate smaller batches bit for bit, everything finite."""
    n = 1 << 20
    ws = W.box_box(n)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n)
    t1, t2 = torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda")
    big = api.generate_manifold_batch(s1, s2, t1, t2, SmoothingConfig())
    head = api.generate_manifold_batch(s1, s2, t1, t2[:4096].contiguous(), SmoothingConfig())
    last = api.generate_manifold_batch(s1, s2, t1, t2[n - 1:].contiguous(), SmoothingConfig())
    torch.cuda.synchronize()
    assert torch.equal(big["contacts"][:4096], head["contacts"])
    assert torch.equal(big["contacts"][n - 1:], last["contacts"])
    assert torch.equal(big["mean_dist"][:4096], head["mean_dist"])
    assert bool(torch.isfinite(big["mean_dist"]).all())
    del big
    torch.cuda.empty_cache()


def _topk_parity(ws, n, what):
    (a1, a2), (o1, o2) = surfaces(ws)
    p1, p2 = ws.poses(n)
    ref = Oracle.manifold_batch(o1, o2, p1, p2, SmoothingConfig())
    r = api.generate_manifold_batch(a1, a2, torch.as_tensor(p1, device="cuda"),
                                    torch.as_tensor(p2, device="cuda"), SmoothingConfig(), want_src=True)
    torch.cuda.synchronize()
    assert_parity(r["contacts"].cpu().numpy(), ref["contacts"], what=what)
    assert np.array_equal(r["src"].cpu().numpy(), ref["meta"][..., 2:]), f"{what}: provenance"


@pytest.mark.parametrize("subdiv,vk,ek", [(6, 16, 8), (6, 3, 40), (3, 50, 3)])
def test_soft_topk_both_order_schemes(cuda, subdiv, vk, ek):
    """Soft top-K over large candidate sets: a finely subdivided plate (218
    vertices, 432 edges: above the warp extraction's 128, so the rank count
    orders them) and small / large K against the primitive's sets (warp
    extraction when K x 104 < D^2), vs the C oracle incl. provenance."""
    ws = W.mixed_bucket("rounded_box", 64)
    ws.bodies[0].mesh.subdivisions = subdiv
    ws.bodies[0].vertex_topk, ws.bodies[0].edge_topk = vk, ek
    ws.bodies[1].vertex_topk, ws.bodies[1].edge_topk = min(vk, 30), min(ek, 60)
    _topk_parity(ws, 64, f"top-K subdiv {subdiv} K {vk}/{ek}")


def test_soft_topk_exact_ties(cuda):
    """Unjittered, axis-aligned box on a subdivided plate: many candidate
    scores are exactly equal, so the order's index tie-break and the first-
    argmax provenance are exercised (both order schemes)."""
    ws = W.box_on_plane(8)
    ws.jitter = 0.0
    ws.bodies[1].mesh.subdivisions = 2
    for b in ws.bodies:
        b.vertex_topk, b.edge_topk = 5, 7
    _topk_parity(ws, 8, "top-K exact ties")


def _blob(n_leaves, seed=5):
    """Smooth union of n small spheres (one flat union: wider than the
    interpreter's stack, and above the parameter block's 16 nodes)."""
    from paper_2602_20304_b200.scene import Union
    rng = np.random.default_rng(seed)
    leaves = [Superquadric(1.0, 1.0, (0.15, 0.15, 0.15), tuple(rng.uniform(-0.15, 0.15, 3)) + (0.0, 0.0, 0.0))
              for _ in range(n_leaves)]
    return Union(leaves, 0.02)


@pytest.mark.parametrize("n_leaves", [12, 40])
def test_large_sdf_programs(cuda, n_leaves):
    """Programs beyond the parameter block (n_leaves + 1 > 16 nodes: the node
    array in device memory) and unions wider than the interpreter's stack
    (emitted as chains of binary unions, the same smooth minimum): manifold
    and field values vs the C oracle, which evaluates the n-ary union directly."""
    blob = W.BodySpec("blob", W.MeshSpec(obj_text=W.sq_obj_text(1.0, 1.0, (0.3, 0.3, 0.3))), _blob(n_leaves),
                      [0.0, 0.0, 0.0, 0.0, 0.0, 0.0], 8, 6)
    box = W.BodySpec("box", W.MeshSpec(box_half=(0.5, 0.5, 0.5)), W.BOX_SQ, [0.05, -0.02, 0.78, 0.1, 0.2, 0.3], 0, 6)
    ws = W.Workload("blob-vs-box", [blob, box], 32)
    _topk_parity(ws, 32, f"union of {n_leaves} spheres")
    (a1, _), (o1, _) = surfaces(ws)
    pts = np.random.default_rng(1).uniform(-0.5, 0.5, (512, 3))
    ref = o1.sdf_query(1, pts)  # value + gradient
    got = api.sdf_query(a1, torch.as_tensor(pts, device="cuda"), 1).cpu().numpy()
    assert np.allclose(got, ref, rtol=1e-9, atol=1e-12), float(np.abs(got - ref).max())


def test_sdf_nesting_limit_is_loud(cuda):
    """Nesting deeper than the interpreter's stack cannot be chained: refused."""
    from paper_2602_20304_b200.scene import Subtraction
    s = Superquadric(1.0, 1.0, (0.3, 0.3, 0.3))
    for _ in range(9):  # right-deep: each subtraction holds its minuend while the subtrahend nests
        s = Subtraction(Superquadric(1.0, 1.0, (0.3, 0.3, 0.3)), s, 0.01)
    b = W.BodySpec("deep", W.MeshSpec(box_half=(0.3, 0.3, 0.3)), s, [0.0] * 6, 0, 0)
    with pytest.raises(Exception, match="nesting"):
        api.surface_from_spec(b)
        api.generate_manifold_batch(api.surface_from_spec(b), api.surface_from_spec(b),
                                    torch.zeros((1, 6), dtype=torch.float64, device="cuda"),
                                    torch.zeros((1, 6), dtype=torch.float64, device="cuda"), SmoothingConfig())


def test_scene_batch_under_cuda_graph_capture(cuda):
    """The scene call's fork onto side streams and join back (events) plus its
    stream-ordered scratch are capturable: a captured CUDA graph replays to the
    same manifolds as the direct call."""
    sc = W.drop_scene(64)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    P = torch.as_tensor(sc.poses(64), device="cuda")
    ref = api.generate_manifold_scene_batch(bodies, P, SmoothingConfig(), is_static=sc.is_static())
    ref = [r["contacts"].clone() for r in ref]
    s = torch.cuda.Stream()
    outs = None
    with torch.cuda.stream(s):  # warm-up on the capture stream (first-use setup outside the capture)
        outs = api.generate_manifold_scene_batch(bodies, P, SmoothingConfig(), is_static=sc.is_static(), outs=outs)
    s.synchronize()
    for r in outs:
        r["contacts"].zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        api.generate_manifold_scene_batch(bodies, P, SmoothingConfig(), is_static=sc.is_static(), outs=outs)
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a["contacts"], b)
