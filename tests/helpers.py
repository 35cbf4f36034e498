"""Shared test helpers: surfaces for both backends, parity comparison."""
from __future__ import annotations

import numpy as np

from oracle import Oracle
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.workloads import Workload

# North-star tolerance (BASELINE.json): 1e-5 relative / 1e-6 absolute in FP32.
RTOL = 1e-5
ATOL = 1e-6
FIELDS = ["px", "py", "pz", "dist", "nx", "ny", "nz", "activity"]


def surfaces(ws: Workload):
    """(api surfaces, oracle surfaces) for the first two bodies of a workload."""
    a = [api.surface_from_spec(b) for b in ws.bodies[:2]]
    o = [Oracle.Surface(s.mesh.vertices, s.mesh.edges, b.sdf, b.vertex_topk, b.edge_topk)
         for s, b in zip(a, ws.bodies[:2])]
    return a, o


def parity_report(got: np.ndarray, ref: np.ndarray, rtol=RTOL, atol=ATOL):
    """Per-field failure counts of |got - ref| <= atol + rtol |ref| over [..., 8]."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(got - ref)
    bound = atol + rtol * np.abs(ref)
    bad = ~(err <= bound)
    rep = {}
    for k, f in enumerate(FIELDS[: got.shape[-1]]):
        b = bad[..., k]
        rep[f] = dict(fails=int(b.sum()), n=int(b.size), max_err=float(err[..., k].max()),
                      max_ratio=float((err[..., k] / bound[..., k]).max()))
    return rep, bad


def assert_parity(got, ref, what="", rtol=RTOL, atol=ATOL, allow=0):
    rep, bad = parity_report(got, ref, rtol, atol)
    nfail = int(bad.sum())
    if nfail > allow:
        idx = np.argwhere(bad)[:8]
        lines = [f"{what}: {nfail} components outside {atol:g} + {rtol:g}|ref| (allowed {allow})"]
        for f, r in rep.items():
            if r["fails"]:
                lines.append(f"  {f}: {r['fails']}/{r['n']} max_err={r['max_err']:.3g} max_ratio={r['max_ratio']:.3g}")
        for i in idx:
            t = tuple(int(x) for x in i)
            lines.append(f"  at {t}: got={got[t]!r} ref={ref[t]!r}")
        raise AssertionError("\n".join(lines))
    return rep
