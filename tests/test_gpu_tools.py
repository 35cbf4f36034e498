"""GPU checks of the reference tool surface (proj/tools/main.cpp) on this
package: the Fig. 4 sweep (src/sweep.cpp) and FP64 witnesses vs the
reference, and every CLI command end to end on the scene files."""
import csv
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from helpers import assert_parity
from paper_2602_20304_b200 import api
from paper_2602_20304_b200.scene import SmoothingConfig

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
SCENES = os.path.join(HERE, "scenes")
ROOT = os.path.dirname(HERE)


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_rotating_edge_sweep_matches_reference(cuda, variant):
    g = np.load(os.path.join(GOLD, "tools.npz"))[f"sweep{variant}"]
    s = api.rotating_edge_sweep(variant, len(g))
    assert np.array_equal(s[:, 0], g[:, 0])
    assert np.abs(s[:, 1:4] - g[:, 1:4]).max() < 1e-9
    # central differences at h = 1e-7 amplify the 1e-12 witness differences;
    # a jump of the hard solver's active set inside [t - h, t + h] is a tie
    d = np.abs(s[:, 4:7] - g[:, 4:7]) / (1e-4 + 1e-4 * np.abs(g[:, 4:7]))
    assert (d.max(axis=1) > 1).sum() <= 2, np.argwhere(d > 1)[:5]


@pytest.mark.parametrize("var", ["ours", "ours_ns"])
def test_ee_witness_f64_matches_reference(cuda, var):
    g = np.load(os.path.join(GOLD, "witness.npz"))
    pairs = torch.as_tensor(g["pairs"], device="cuda")
    r = api.run_ee_batch_f64(pairs, SmoothingConfig().for_variant(var), want_alpha=True)
    ref = g[f"ee_{var}"]  # p1, p2, alpha1, alpha2, gamma
    got = r["out"].cpu().numpy()
    assert np.abs(got - ref[:, :6]).max() < 1e-9
    assert np.abs(r["alpha_gamma"].cpu().numpy() - ref[:, 6:9]).max() < 1e-9


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2602_20304_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=600)


@pytest.mark.parametrize("name", ["box_on_plane", "capsule_vs_hollow"])
def test_cli_manifold(cuda, tmp_path, name):
    out = tmp_path / "m.csv"
    r = run_cli("manifold", "--scene", os.path.join(SCENES, f"{name}.json"), "--out", str(out))
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(out)))
    assert rows[0] == "index,kind,side,src_a,src_b,px,py,pz,dist,nx,ny,nz,activity".split(",")
    g = np.load(os.path.join(GOLD, "tools.npz"))
    contacts = np.array([[float(x) for x in r[5:]] for r in rows[1:]])
    meta = np.array([[0 if r[1] == "VS" else 1, int(r[2]), int(r[3]), int(r[4])] for r in rows[1:]])
    assert np.array_equal(meta, g[f"{name}_meta"])
    assert_parity(contacts, g[f"{name}_contacts"], what=f"cli manifold {name}")
    rj = run_cli("manifold", "--scene", os.path.join(SCENES, f"{name}.json"), "--out", str(tmp_path / "m.json"),
                 "--json")
    assert rj.returncode == 0, rj.stderr


def test_cli_gradcheck_sweep_bench_sim(cuda, tmp_path):
    r = run_cli("gradcheck", "--scene", os.path.join(SCENES, "box_on_plane.json"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "max relative error" in r.stdout
    r = run_cli("sweep-edges", "--out", str(tmp_path / "s.csv"), "--samples", "257")
    assert r.returncode == 0 and len(open(tmp_path / "s.csv").read().splitlines()) == 258
    r = run_cli("bench", "--kind", "ee", "--batch", "1000,4096", "--out", str(tmp_path / "b.csv"), "--repetitions", "3")
    assert r.returncode == 0, r.stderr
    lines = open(tmp_path / "b.csv").read().splitlines()
    assert lines[0] == "# cmg-bench-csv v1" and len(lines) == 2 + 4
    r = run_cli("bench", "--kind", "manifold", "--scene", os.path.join(SCENES, "box_on_plane.json"), "--batch",
                "512", "--variants", "ours", "--out", str(tmp_path / "bm.csv"), "--repetitions", "3")
    assert r.returncode == 0, r.stderr
    r = run_cli("sim", "--scene", os.path.join(SCENES, "box_on_plane.json"), "--duration", "0.05", "--out",
                str(tmp_path / "sim.csv"))
    assert r.returncode == 0, r.stderr
    assert len(open(tmp_path / "sim.csv").read().splitlines()) == 1 + 6


@pytest.mark.parametrize("ground", ["box_planes", "sq"])
def test_cli_gradcheck_posed_primitives(cuda, tmp_path, ground):
    """Pose Jacobians with rotated / offset primitives inside the bodies (the
    SQ leaf's body_from_prim frame, sdf.cpp:9): the analytic-Hessian paths of
    the JVP kernel vs central differences of its own FP64 mean (the
    reference's gradcheck, main.cpp:190-235)."""
    import json
    g = ({"type": "box_planes", "half_extents": [2.0, 2.0, 0.1]} if ground == "box_planes" else
         {"type": "superquadric", "eps1": 0.1, "eps2": 0.1, "axes": [2.0, 2.0, 0.1],
          "pose": [0.0, 0.01, 0.0, 0.0, 0.0, 0.3]})
    scene = {
        "smoothing": {"sphere_trace_iters": 5, "mode": "full"},
        "bodies": [
            {"name": "box", "mesh": {"box": {"half_extents": [0.5, 0.5, 0.5]}},
             "sdf": {"type": "superquadric", "eps1": 0.1, "eps2": 0.1, "axes": [0.5, 0.5, 0.5],
                     "pose": [0.01, -0.02, 0.005, 0.05, -0.04, 0.2]},
             "pose": [0.01, -0.02, 0.49, 0.02, -0.01, 0.05], "edge_topk": 12},
            {"name": "ground", "mesh": {"box": {"half_extents": [2.0, 2.0, 0.1]}}, "sdf": g,
             "pose": [0.0, 0.0, -0.1, 0.0, 0.0, 0.0], "edge_topk": 4},
        ],
    }
    path = tmp_path / "posed.json"
    path.write_text(json.dumps(scene))
    r = run_cli("gradcheck", "--scene", str(path))
    assert r.returncode == 0, r.stdout + r.stderr
