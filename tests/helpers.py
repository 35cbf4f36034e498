"""Shared test helpers: surfaces for both backends, parity comparison.

Parity rule (BASELINE.json north star, "1e-5 relative / 1e-6 absolute in
FP32"): for every contact,
    |point_gpu  - point_ref|  <= 1e-6 + 1e-5 |point_ref|     (Euclidean, 3-vector)
    |normal_gpu - normal_ref| <= 1e-6 + 1e-5 |normal_ref|    (Euclidean, 3-vector)
    |dist_gpu - dist_ref|     <= 1e-6 + 1e-5 |dist_ref|
    |act_gpu - act_ref|       <= 1e-6 + 1e-5 |act_ref|
Vectors are compared as vectors: "relative" is relative to the vector's
magnitude (a per-component relative bound on a near-zero component of a unit
normal is not a property of the normal).
"""
from __future__ import annotations

import numpy as np

from oracle import Oracle
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.workloads import Workload

RTOL = 1e-5
ATOL = 1e-6
QUANTITIES = {"point": slice(0, 3), "dist": slice(3, 4), "normal": slice(4, 7), "activity": slice(7, 8)}


def surfaces(ws: Workload):
    """(api surfaces, oracle surfaces) for the first two bodies of a workload."""
    a = [api.surface_from_spec(b) for b in ws.bodies[:2]]
    o = [Oracle.Surface(s.mesh.vertices, s.mesh.edges, b.sdf, b.vertex_topk, b.edge_topk)
         for s, b in zip(a, ws.bodies[:2])]
    return a, o


def parity_report(got: np.ndarray, ref: np.ndarray, rtol=RTOL, atol=ATOL):
    """Per-quantity failure counts over contacts [..., 8]."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    rep = {}
    bad_any = np.zeros(got.shape[:-1], dtype=bool)
    for name, sl in QUANTITIES.items():
        err = np.linalg.norm(got[..., sl] - ref[..., sl], axis=-1)
        bound = atol + rtol * np.linalg.norm(ref[..., sl], axis=-1)
        bad = ~(err <= bound)
        bad_any |= bad
        rep[name] = dict(fails=int(bad.sum()), n=int(bad.size), max_err=float(err.max()) if err.size else 0.0,
                         max_ratio=float((err / bound).max()) if err.size else 0.0)
    return rep, bad_any


def assert_parity(got, ref, what="", rtol=RTOL, atol=ATOL, allow=0):
    rep, bad = parity_report(got, ref, rtol, atol)
    nfail = int(bad.sum())
    if nfail > allow:
        lines = [f"{what}: {nfail} contacts outside {atol:g} + {rtol:g}|ref| (allowed {allow})"]
        for f, r in rep.items():
            if r["fails"]:
                lines.append(f"  {f}: {r['fails']}/{r['n']} max_err={r['max_err']:.3g} max_ratio={r['max_ratio']:.3g}")
        for i in np.argwhere(bad)[:6]:
            t = tuple(int(x) for x in i)
            lines.append(f"  at {t}: got={np.asarray(got)[t]!r}\n           ref={np.asarray(ref)[t]!r}")
        raise AssertionError("\n".join(lines))
    return rep


def scalar_close(got, ref, rtol=RTOL, atol=ATOL):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.abs(got - ref) <= atol + rtol * np.abs(ref)
