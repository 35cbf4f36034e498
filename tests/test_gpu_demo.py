"""GPU parity of the batched demo integrator (cmgb_demo_step_batch: DemoSim::step,
src/demosim.cpp:81-138) against the reference's DemoSim rollouts
(tests/golden/demo.npz).

The GPU path consumes the ABI's FP32 contacts (the reference's are FP64), so a
single step from a reference state is compared with a state tolerance
(1e-7 absolute + 1e-6 relative on poses and velocities: a 100 N contact force
with FP32-rounded normals / points moves a 1 ms velocity update by ~1e-8) and
the free rollout
within a bound that widens as contact events amplify the difference."""
import os

import numpy as np
import pytest
import torch

from cases import DEMO_DT, DEMO_STEPS
from paper_2602_20304_b200 import api
from paper_2602_20304_b200 import workloads as W
from paper_2602_20304_b200.scene import PenaltyParams, SmoothingConfig

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def make_batch(n_env, poses, vels=None):
    sc = W.demo_scene(n_env)
    bodies = [api.surface_from_spec(b) for b in sc.bodies]
    return api.DemoBatch(bodies, np.ones(len(bodies)), is_static=sc.is_static(), cfg=SmoothingConfig(),
                         params=PenaltyParams(), poses=poses, velocities=vels, n_env=n_env)


def state_err(got, ref):
    return float(np.max(np.abs(got - ref) / (1e-7 + 1e-6 * np.abs(ref))))


def test_one_step_from_reference_states(cuda):
    """From reference states inside contact events, one GPU step equals the
    reference's next state."""
    g = np.load(os.path.join(GOLD, "demo.npz"))
    steps = [100, 150, 170, 200, 250, 298]
    P = np.stack([g[f"poses{e}"][s] for e in range(2) for s in steps])
    V = np.stack([g[f"velocities{e}"][s] for e in range(2) for s in steps])
    b = make_batch(len(P), P, V)
    b.step(DEMO_DT)
    torch.cuda.synchronize()
    ref_P = np.stack([g[f"poses{e}"][s + 1] for e in range(2) for s in steps])
    ref_V = np.stack([g[f"velocities{e}"][s + 1] for e in range(2) for s in steps])
    ref_D = np.array([g[f"deepest{e}"][s + 1] for e in range(2) for s in steps])
    ep, ev = state_err(b.poses.cpu().numpy(), ref_P), state_err(b.velocities.cpu().numpy(), ref_V)
    print("one-step error ratios: poses", ep, "velocities", ev, "abs",
          np.abs(b.poses.cpu().numpy() - ref_P).max(), np.abs(b.velocities.cpu().numpy() - ref_V).max())
    assert ep <= 1.0 and ev <= 1.0
    assert np.allclose(b.deepest.cpu().numpy(), ref_D, rtol=1e-5, atol=1e-6)
    assert (b.ok.cpu().numpy() == 1).all()


def test_rollout_tracks_reference(cuda):
    """Free rollouts from the initial states: the stacked scene (envs 0, 1) and
    16 single-box drops stay on the reference trajectory to 1e-6 over the first
    150 / 200 steps (measured ~1e-9; later the impacts amplify the FP32-contact
    differences chaotically, as they would any perturbation)."""
    g = np.load(os.path.join(GOLD, "demo.npz"))
    b = make_batch(2, g["init_poses"], None)
    for s in range(150):
        b.step(DEMO_DT)
    ref = np.stack([g[f"poses{e}"][149] for e in range(2)])
    err3 = float(np.abs(b.poses.cpu().numpy() - ref).max())
    sc = W.demo_scene(16, n_boxes=1)
    bodies = [api.surface_from_spec(x) for x in sc.bodies]
    b1 = api.DemoBatch(bodies, np.ones(2), is_static=sc.is_static(), cfg=SmoothingConfig(), params=PenaltyParams(),
                       poses=g["box1_init_poses"], n_env=16)
    b1.step(DEMO_DT, 100)
    e100 = max(float(np.abs(b1.poses.cpu().numpy()[e] - g[f"box1_{e}_s100"]).max()) for e in range(16))
    b1.step(DEMO_DT, 100)
    e200 = max(float(np.abs(b1.poses.cpu().numpy()[e] - g[f"box1_{e}_s200"]).max()) for e in range(16))
    print("rollout max |pose - ref|: stack@150", err3, "box@100", e100, "box@200", e200)
    assert err3 < 1e-6 and e100 < 1e-6 and e200 < 1e-6


def world_translation(pose):
    """t of se3_exp(pose) (pose.hpp:65-76): V(w) rho, V = I + [w]x B + [w]x^2 C."""
    rho, w = pose[:3], pose[3:]
    th2 = float(w @ w)
    if th2 < 1e-8:
        b, c = 0.5 - th2 / 24 + th2 * th2 / 720, 1 / 6 - th2 / 120 + th2 * th2 / 5040
    else:
        th = np.sqrt(th2)
        b, c = (1 - np.cos(th)) / th2, (1 - np.sin(th) / th) / th2
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    return (np.eye(3) + W * b + (W @ W) * c) @ rho


def test_batch_rollout_finite(cuda):
    """4,096 jittered single-box drops, 1,000 steps: every env finite (the
    reference's step() never fails here) and no box over the ground plate has
    sunk through it (edge-first landings can launch a box off the plate, in the
    reference too)."""
    sc = W.demo_scene(4096, n_boxes=1)
    bodies = [api.surface_from_spec(x) for x in sc.bodies]
    b = api.DemoBatch(bodies, np.ones(2), is_static=sc.is_static(), cfg=SmoothingConfig(), params=PenaltyParams(),
                      poses=sc.poses(4096), n_env=4096)
    b.step(DEMO_DT, 1000)
    torch.cuda.synchronize()
    assert (b.ok.cpu().numpy() == 1).all()
    P = b.poses.cpu().numpy()
    assert np.isfinite(P).all()
    t = np.array([world_translation(p) for p in P[:, 1]])
    over = (np.abs(t[:, 0]) < 1.5) & (np.abs(t[:, 1]) < 1.5)  # still above the 4 x 4 m plate
    assert over.mean() > 0.5 and (t[over, 2] > 0.3).all(), (over.mean(), t[over, 2].min())
    assert (b.deepest.cpu().numpy() > -0.05).all()
