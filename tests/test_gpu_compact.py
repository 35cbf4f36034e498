"""GPU: active-contact compaction (cmgb_compact_contacts) — an extra output
beside the fixed layout (include/cmg/manifold.hpp:62-72, 303-330, which it
never replaces). The bar: BIT-EQUAL to a numpy filter of the fixed layout
(activity > thr, fixed-layout order, env after env), with exact per-env offsets
/ counts, slot indices and provenance; ragged / empty / capacity-limited /
unstaged (large C) cases; and batch independence at BASELINE size."""
import numpy as np
import pytest
import torch

from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig

pytestmark = pytest.mark.gpu


def numpy_filter(contacts, thr, src=None):
    c = np.asarray(contacts)
    keep = c[..., 7] > thr                                   # [n, C]
    rows = c[keep]                                           # row-major: env after env, layout order
    slot = np.nonzero(keep)[1].astype(np.int32)
    cnt = keep.sum(axis=1).astype(np.int32)
    off = np.concatenate([[0], np.cumsum(cnt, dtype=np.int64)])
    s = np.asarray(src)[keep] if src is not None else None
    return rows, slot, cnt, off, s


def check(res, contacts, thr, src=None, capacity=None):
    rows, slot, cnt, off, s = numpy_filter(contacts, thr, src)
    tot = int(res["total"].item())
    assert tot == len(rows)
    got_off = res["env_offset"].cpu().numpy()
    assert np.array_equal(got_off, off)
    assert np.array_equal(res["env_count"].cpu().numpy(), cnt)
    k = len(rows) if capacity is None else min(len(rows), capacity)
    got = res["contacts"][:k].cpu().numpy()
    assert np.array_equal(got.view(np.uint32), rows[:k].view(np.uint32)), "compacted contacts not bit-equal"
    assert np.array_equal(res["slot"][:k].cpu().numpy(), slot[:k])
    if s is not None:
        assert np.array_equal(res["src"][:k].cpu().numpy(), s[:k])


def box_box(n, cfg=None):
    ws = W.box_box(n)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n)
    r = api.generate_manifold_batch(s1, s2, torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda"),
                                    cfg or SmoothingConfig(), want_src=True)
    return r


@pytest.mark.parametrize("thr", [-1.0, 0.0, 1e-3, 0.01, 0.5, 2.0])
def test_compact_box_box_bit_equal(cuda, thr):
    r = box_box(1001)  # ragged: not a multiple of the 4-env tile
    res = api.compact_contacts(r["contacts"], thr, src=r["src"])
    torch.cuda.synchronize()
    check(res, r["contacts"].cpu().numpy(), thr, r["src"].cpu().numpy())


def test_compact_topk_provenance(cuda):
    ws = W.mixed_bucket("capsule", 333)
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(333)
    r = api.generate_manifold_batch(s1, s2, torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda"),
                                    SmoothingConfig(), want_src=True)
    res = api.compact_contacts(r["contacts"], 1e-2, src=r["src"])
    torch.cuda.synchronize()
    check(res, r["contacts"].cpu().numpy(), 1e-2, r["src"].cpu().numpy())


def test_compact_capacity_and_edges(cuda):
    r = box_box(64)
    c = r["contacts"]
    full = api.compact_contacts(c, -1.0)
    torch.cuda.synchronize()
    assert int(full["total"].item()) == c.shape[0] * c.shape[1]
    cap = 1000
    res = api.compact_contacts(c, -1.0, capacity=cap)
    torch.cuda.synchronize()
    check(res, c.cpu().numpy(), -1.0, capacity=cap)
    one = api.compact_contacts(c[:1].contiguous(), 0.01)
    torch.cuda.synchronize()
    check(one, c[:1].cpu().numpy(), 0.01)
    empty = api.compact_contacts(c[:0].contiguous(), 0.01)
    torch.cuda.synchronize()
    assert int(empty["total"].item()) == 0 and empty["env_offset"].cpu().tolist() == [0]
    with pytest.raises(ValueError):  # not [n, C, 8]
        api.compact_contacts(c[..., :7].contiguous(), 0.0)
    with pytest.raises(ValueError):  # 8-byte aligned view: the TMA staging needs 16
        api.compact_contacts(c.reshape(-1)[2:2 + 80].view(1, 10, 8), 0.0)


@pytest.mark.parametrize("n,C", [(1, 1), (7, 3), (1000, 48), (257, 600), (3, 6000), (3, 7000), (2, 30000)])
def test_compact_random_shapes(cuda, n, C):
    """Synthetic fixed layouts of every size class: many envs per tile (C=48),
    one env per tile (C=600, and C=6000: a 192 KB stage), and envs too large
    to stage (C=7000: 224 KB, C=30000: the unstaged two-read path)."""
    g = torch.Generator(device="cuda").manual_seed(n * 1000 + C)
    c = torch.rand((n, C, 8), generator=g, device="cuda", dtype=torch.float32)
    src = torch.randint(-1, 100, (n, C, 2), generator=g, device="cuda", dtype=torch.int32)
    res = api.compact_contacts(c, 0.7, src=src)
    torch.cuda.synchronize()
    check(res, c.cpu().numpy(), 0.7, src.cpu().numpy())


def test_compact_full_size_batch_independence(cuda):
    """BASELINE size (65,536 box-box envs): the compacted output equals the
    numpy filter, and the first 4,096 envs compact exactly as a 4,096-env
    batch does (offsets are a prefix; rows identical)."""
    r = box_box(65536)
    res = api.compact_contacts(r["contacts"], 0.01, src=r["src"])
    torch.cuda.synchronize()
    c = r["contacts"].cpu().numpy()
    check(res, c, 0.01, r["src"].cpu().numpy())
    small = api.compact_contacts(r["contacts"][:4096].contiguous(), 0.01)
    torch.cuda.synchronize()
    k = int(small["total"].item())
    assert np.array_equal(small["env_offset"].cpu().numpy(), res["env_offset"][:4097].cpu().numpy())
    assert torch.equal(small["contacts"][:k], res["contacts"][:k])


def numpy_masks(contacts, thr):
    c = np.asarray(contacts)
    keep = c[..., 7] > thr
    n, C = keep.shape
    words = (C + 31) // 32
    pad = np.zeros((n, words * 32), bool)
    pad[:, :C] = keep
    bits = pad.reshape(n, words, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)
    return bits.sum(axis=2).astype(np.uint32).view(np.int32), keep.sum(axis=1).astype(np.int32)


def masked_case(ws, n, cfg, thr):
    s1, s2 = (api.surface_from_spec(b) for b in ws.bodies)
    p1, p2 = ws.poses(n)
    r = api.generate_manifold_batch(s1, s2, torch.as_tensor(p1, device="cuda"), torch.as_tensor(p2, device="cuda"),
                                    cfg, want_src=True, active_threshold=thr)
    torch.cuda.synchronize()
    c = r["contacts"].cpu().numpy()
    m, k = numpy_masks(c, thr)
    assert np.array_equal(r["active_mask"].cpu().numpy(), m), "activity masks differ from the fixed layout"
    assert np.array_equal(r["active_count"].cpu().numpy(), k)
    res = api.compact_contacts(r["contacts"], src=r["src"], mask=r["active_mask"], count=r["active_count"])
    torch.cuda.synchronize()
    check(res, c, thr, r["src"].cpu().numpy())


@pytest.mark.parametrize("thr", [-1.0, 0.0, 0.01, 0.5, 2.0])
def test_masks_box_box(cuda, thr):
    """kVsX kernel pair (V-S bits from vs_kernel, E-E bits from the manifold kernel)."""
    masked_case(W.box_box(1001), 1001, SmoothingConfig(), thr)


@pytest.mark.parametrize("case", ["box_box_topk", "mixed_capsule", "mixed_rounded_box", "box_box_ours_ne",
                                  "box_box_ours_ne_s", "box_on_plane_ours", "subtraction_vs_box"])
def test_masks_every_kernel_shape(cuda, case):
    """In-kernel V-S paths (phase E on the 10-warp shape, phase F on the
    9-warp shape), no-EE / one-sided modes, generic interpreter."""
    from cases import manifold_cases
    _, ws, cfg, _ = [c for c in manifold_cases() if c[0] == case][0]
    masked_case(ws, 777, cfg, 0.01)


def test_masks_global_pair_records(cuda):
    """The global-memory pair-record instantiation: two subdivided boxes with
    all 48 edges pass-through (P = 2,304 pairs, tests/test_gpu_edges.py)."""
    ws = W.box_box(64)
    for b in ws.bodies:
        b.mesh.subdivisions = 2
    m = api.surface_from_spec(ws.bodies[0]).mesh.edges.shape[0]
    for b in ws.bodies:
        b.edge_topk = m
    masked_case(ws, 16, SmoothingConfig(), 0.01)
