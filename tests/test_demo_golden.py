"""Checks the DemoSim golden rollouts (CPU): invariants of the reference's
integrator (src/demosim.cpp:81-138) and DemoSim::kinetic_energy (140-155),
restated by api.kinetic_energy_np.
The GPU integrator is checked against the same fixtures in tests/test_gpu_demo.py."""
import os

import numpy as np

from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_rollout_invariants():
    """Static bodies never move (demosim.cpp:107), deepest_penetration <= 0
    (initialised to 0, min over active contacts), every step finite. (Free fall
    is not closed-form here: the smoothed E-E activities let separated boxes
    exchange small penalty forces, which the GPU port reproduces.)"""
    g = np.load(os.path.join(GOLD, "demo.npz"))
    sc = W.demo_scene(2)
    st = np.flatnonzero(sc.is_static().astype(bool))
    for e in range(2):
        P, V, D = g[f"poses{e}"], g[f"velocities{e}"], g[f"deepest{e}"]
        assert len(P) == 300 and np.isfinite(P).all() and np.isfinite(V).all()
        assert np.array_equal(P[:, st], np.broadcast_to(g["init_poses"][e, st], P[:, st].shape))
        assert (V[:, st] == 0).all()
        assert (D <= 0).all() and (D < 0).any()


def test_kinetic_energy_restatement():
    g = np.load(os.path.join(GOLD, "demo.npz"))
    sc = W.demo_scene(2)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    masses = np.ones(len(bodies))
    inertia = np.array([api._box_inertia(1.0, b.mesh.vertices) for b in bodies])
    for e in range(2):
        ke = api.kinetic_energy_np(g[f"poses{e}"], g[f"velocities{e}"], masses, inertia, sc.is_static())
        assert np.allclose(ke, g[f"kinetic_energy{e}"], rtol=1e-10, atol=1e-12)
