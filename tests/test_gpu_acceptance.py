"""GPU: SPEC acceptance criteria #1 and #2 on the K6 witness
kernels, with the reference's own independent oracles re-stated in numpy
(proj/tests/test_helpers.hpp:50-105):

  #1 hard box QP: the objective at the GPU witness parameters is within 1e-6
     of the brute-force minimum (dense 201 x 201 grid seed + 200 rounds of exact
     coordinate descent) on make_random_ee_pairs(10^4, seed 0), ours_ns;
  #2 hard V-F: the GPU closest point is within 1e-4 of the Voronoi-region
     closest point on make_random_vf_pairs(10^4, seed 0), ours_ns.

Both kernels are exercised: the FP32-output batch kernel (cmgb_ee_witness_batch /
cmgb_vf_witness_batch, what run_*_batch uses) and, for #1, the FP64-output
solver (cmgb_ee_witness_batch_f64)."""
import numpy as np
import pytest
import torch

from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import SmoothingConfig

pytestmark = pytest.mark.gpu
N = 10_000


def box_qps(pairs, lam):
    """Q = A^T A + lambda I, c = b^T A - lambda / 2 with A = [t1, -t2] (witness.hpp:137-158)."""
    e1a, e1b, e2a, e2b = pairs[:, 0:3], pairs[:, 3:6], pairs[:, 6:9], pairs[:, 9:12]
    t1 = e1b - e1a
    t2n = e2a - e2b
    b = e1a - e2a
    q11 = (t1 * t1).sum(1) + lam
    q12 = (t1 * t2n).sum(1)
    q22 = (t2n * t2n).sum(1) + lam
    c1 = (b * t1).sum(1) - 0.5 * lam
    c2 = (b * t2n).sum(1) - 0.5 * lam
    return q11, q12, q22, c1, c2


def qp_cost(q, a, b):
    q11, q12, q22, c1, c2 = q
    return 0.5 * (q11 * a * a + 2 * q12 * a * b + q22 * b * b) + c1 * a + c2 * b


def box_qp_oracle(q, grid=201, chunk=256):
    """box_qp_oracle (test_helpers.hpp:50-70), vectorised over QPs."""
    q11, q12, q22, c1, c2 = q
    g = np.linspace(0.0, 1.0, grid)
    A, B = np.meshgrid(g, g, indexing="ij")
    A, B = A.ravel(), B.ravel()
    x = np.empty(len(q11))
    y = np.empty(len(q11))
    for lo in range(0, len(q11), chunk):
        sl = slice(lo, lo + chunk)
        cost = 0.5 * (q11[sl, None] * A * A + 2 * q12[sl, None] * A * B + q22[sl, None] * B * B) \
            + c1[sl, None] * A + c2[sl, None] * B
        k = np.argmin(cost, axis=1)
        x[sl], y[sl] = A[k], B[k]
    for _ in range(200):
        x = np.clip(-(c1 + q12 * y) / q11, 0.0, 1.0)
        y = np.clip(-(c2 + q12 * x) / q22, 0.0, 1.0)
    return x, y


def closest_point_triangle(p, a, b, c):
    """closest_point_triangle_oracle (test_helpers.hpp:76-105): Voronoi regions,
    evaluated per point (a route separate from the clipped-projection solver)."""
    out = np.empty_like(p)
    for i in range(len(p)):
        P, A, B, Cc = p[i], a[i], b[i], c[i]
        ab, ac, ap = B - A, Cc - A, P - A
        d1, d2 = ab @ ap, ac @ ap
        if d1 <= 0 and d2 <= 0:
            out[i] = A
            continue
        bp = P - B
        d3, d4 = ab @ bp, ac @ bp
        if d3 >= 0 and d4 <= d3:
            out[i] = B
            continue
        vc = d1 * d4 - d3 * d2
        if vc <= 0 and d1 >= 0 and d3 <= 0:
            out[i] = A + ab * (d1 / (d1 - d3))
            continue
        cp = P - Cc
        d5, d6 = ab @ cp, ac @ cp
        if d6 >= 0 and d5 <= d6:
            out[i] = Cc
            continue
        vb = d5 * d2 - d1 * d6
        if vb <= 0 and d2 >= 0 and d6 <= 0:
            out[i] = A + ac * (d2 / (d2 - d6))
            continue
        va = d3 * d6 - d5 * d4
        if va <= 0 and (d4 - d3) >= 0 and (d5 - d6) >= 0:
            w = (d4 - d3) / ((d4 - d3) + (d5 - d6))
            out[i] = B + (Cc - B) * w
            continue
        den = 1.0 / (va + vb + vc)
        out[i] = A + ab * (vb * den) + ac * (vc * den)
    return out


@pytest.fixture(scope="module")
def random_pairs():
    return W.mt19937_64_uniform(0, 12 * N, 0.0, 1.0).reshape(N, 12)  # make_random_*_pairs(N, seed 0)


def test_acceptance_1_hard_qp_vs_bruteforce(cuda, random_pairs):
    cfg = SmoothingConfig().for_variant("ours_ns")  # lambda 1e-6, hard operators
    q = box_qps(random_pairs, cfg.lambda_)
    xo, yo = box_qp_oracle(q)
    best = qp_cost(q, xo, yo)
    D = torch.as_tensor(random_pairs, device="cuda")
    r32 = api.run_ee_batch(D, cfg, want_alpha=True)
    r64 = api.run_ee_batch_f64(D, cfg, want_alpha=True)
    torch.cuda.synchronize()
    for name, r, tol in (("fp64-output solver", r64, 1e-6), ("fp32-output batch kernel", r32, 1e-6)):
        ag = r["alpha_gamma"].cpu().numpy().astype(np.float64)
        gap = qp_cost(q, ag[:, 0], ag[:, 1]) - best
        bad = int((gap > tol).sum())
        print(f"acceptance #1 ({name}): {bad}/{N} gaps > {tol:g}, worst {gap.max():.3g}")
        assert bad == 0, (name, float(gap.max()))


def test_acceptance_2_hard_vf_vs_voronoi(cuda, random_pairs):
    cfg = SmoothingConfig().for_variant("ours_ns")
    p = random_pairs
    ref = closest_point_triangle(p[:, 0:3], p[:, 3:6], p[:, 6:9], p[:, 9:12])
    r = api.run_vf_batch(torch.as_tensor(p, device="cuda"), cfg)
    torch.cuda.synchronize()
    err = np.linalg.norm(r["out"].cpu().numpy().astype(np.float64) - ref, axis=1)
    bad = int((err > 1e-4).sum())
    print(f"acceptance #2: {bad}/{N} errors > 1e-4, worst {err.max():.3g}")
    assert bad == 0, float(err.max())
