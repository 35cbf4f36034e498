"""The C++ drop-in boundary (include/cmgb_cmg.hpp + include/cmg/*.hpp): a C++
caller written against the REFERENCE's API switches to the B200 path by
changing its include path.

* tests/cpp/dropin_main.cpp is one source that builds against the reference
  (its golden: tests/golden/dropin_ref.json, make_dropin_golden.sh) and against
  this repo's headers + libcmgb.so; on the GPU its output must match the
  reference's within the parity rule (tests/helpers.py), provenance / kinds /
  sides exactly, run_ee_batch checksums to the FP64 solver's precision.
* The reference's own dev probe (proj/tests/probe.cpp), UNMODIFIED, is built
  against the drop-in headers (oracle/Makefile `probe` -> oracle/_ref/
  probe_cmgb) and must print what the reference build prints
  (tests/golden/probe_ref*.txt).
"""
import json
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_main.cpp")
LIBDIR = os.path.join(ROOT, "paper_2602_20304_b200")
REF_INC = "/root/reference/proj/include"


def build_ours(out):
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lcmgb", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)


def test_dropin_source_builds_against_this_library(tmp_path):
    build_ours(str(tmp_path / "dropin"))


@pytest.mark.skipif(not os.path.isdir(REF_INC) or not os.path.exists(os.path.join(ROOT, "oracle/_ref/libcmgref.so")),
                    reason="needs the reference sources (dev container)")
def test_dropin_source_builds_against_the_reference(tmp_path):
    """The same caller compiles unchanged against the reference's headers."""
    subprocess.run(["g++", "-std=c++20", "-O0", "-fsyntax-only", "-I", REF_INC, SRC], check=True)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="needs the reference sources (dev container)")
def test_reference_probe_builds_against_dropin_headers(tmp_path):
    """proj/tests/probe.cpp, unmodified, against include/cmg/*.hpp."""
    subprocess.run(["g++", "-std=c++17", "-O0", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                    "/root/reference/proj/tests/probe.cpp"], check=True)


def _close(got, ref, rtol=1e-5, atol=1e-6):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return np.abs(got - ref) <= atol + rtol * np.abs(ref)


@pytest.mark.gpu
def test_dropin_caller_matches_reference_on_gpu(cuda, tmp_path):
    exe = str(tmp_path / "dropin")
    build_ours(exe)
    out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    got = json.loads(out)
    ref = json.load(open(os.path.join(GOLD, "dropin_ref.json")))
    for case in ("box_box_ours", "box_box_ours_ns", "box_box_ours_ne", "box_on_plane", "box_on_plane_topk",
                 "tet_vs_box"):
        g, r = got[case], ref[case]
        for k in ("n1", "n2", "m1", "m2", "size"):
            assert g[k] == r[k], (case, k)
        gc = np.array(g["contacts"], np.float64)
        rc = np.array(r["contacts"], np.float64)
        assert gc.shape == rc.shape, case
        assert np.array_equal(gc[:, 8:], rc[:, 8:]), f"{case}: kind / side / provenance differ"
        for sl in (slice(0, 3), slice(3, 4), slice(4, 7), slice(7, 8)):  # vector-wise parity rule
            err = np.linalg.norm(gc[:, sl] - rc[:, sl], axis=1)
            bound = 1e-6 + 1e-5 * np.linalg.norm(rc[:, sl], axis=1)
            assert (err <= bound).all(), (case, sl, float((err / bound).max()))
        for k in ("ee_act1", "ee_dist"):
            assert len(g[k]) == len(r[k]) and _close(g[k], r[k]).all(), (case, k)
        assert _close(g["mean"], r["mean"])
    gm, rm = np.array(got["grad_mean"]), np.array(ref["grad_mean"])
    assert abs(gm[0] - rm[0]) <= 1e-6 + 1e-5 * abs(rm[0])
    assert np.abs(gm[1:] - rm[1:]).max() <= 1e-4 * np.abs(rm[1:]).max() + 1e-7, "pose gradient of the mean"
    cs_g, cs_r = np.array(got["checksums"]), np.array(ref["checksums"])
    assert abs(cs_g[0] - cs_r[0]) <= 1e-9 * abs(cs_r[0]), "run_ee_batch checksum (FP64 solver)"
    assert abs(cs_g[1] - cs_r[1]) <= 1e-9 * abs(cs_r[1]), "run_ee_batch checksum, ours_ns"
    assert abs(cs_g[2] - cs_r[2]) <= 1e-5 * abs(cs_r[2]), "run_vf_batch checksum (FP32 solver, widened)"
    assert np.abs(np.array(got["ee_out"]) - np.array(ref["ee_out"])).max() <= 1e-9
    assert _close(got["vf_out"], ref["vf_out"]).all()
    assert got["bench"] == ref["bench"]


def _numbers(text):
    return [float(x) for x in re.findall(r"[-+]?\d+\.\d+|[-+]?\d+", text)]


@pytest.mark.gpu
@pytest.mark.parametrize("args,golden", [((), "probe_ref.txt"),
                                         (("0.06", "0.0", "0.0", "0.01", "0.005", "0.02", "5", "0.05", "-0.03"),
                                          "probe_ref_tilt.txt")])
def test_reference_probe_on_gpu(cuda, args, golden):
    exe = os.path.join(ROOT, "oracle", "_ref", "probe_cmgb")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/probe_cmgb not built (needs the reference sources at build time)")
    out = subprocess.run([exe, *args], check=True, capture_output=True, text=True).stdout
    ref = open(os.path.join(GOLD, golden)).read()
    assert out.count("\n") == ref.count("\n"), f"probe prints a different set of contacts:\n{out}\n---\n{ref}"
    g, r = np.array(_numbers(out)), np.array(_numbers(ref))
    assert g.shape == r.shape
    # printed with 1-4 decimals: one unit in the last printed place (plus FP32 output rounding)
    assert np.abs(g - r).max() <= 0.11, np.abs(g - r).max()
    frac = [ln for ln in zip(out.splitlines(), ref.splitlines()) if ln[0] != ln[1]]
    assert len(frac) <= 2, f"more than two printed lines differ: {frac}"


@pytest.mark.gpu
@pytest.mark.parametrize("scene", ["box_on_plane", "capsule_vs_hollow"])
def test_dropin_scene_and_writers_on_gpu(cuda, tmp_path, scene):
    """cmd_manifold's path through the drop-in: load_scene (the reference's
    JSON schema) -> generate_manifold -> write_manifold_csv / manifold_to_json,
    against the same caller built on the reference (tests/golden/
    dropin_<scene>_ref.*): metadata columns identical, numbers within the
    parity rule, JSON text identical once numbers are masked (key order,
    indentation, layout block)."""
    exe = str(tmp_path / "dropin")
    build_ours(exe)
    csv_p, js_p = str(tmp_path / "m.csv"), str(tmp_path / "m.json")
    subprocess.run([exe, os.path.join(ROOT, "tests", "scenes", f"{scene}.json"), csv_p, js_p], check=True)
    got = [ln.split(",") for ln in open(csv_p).read().splitlines()]
    ref = [ln.split(",") for ln in open(os.path.join(GOLD, f"dropin_{scene}_ref.csv")).read().splitlines()]
    assert got[0] == ref[0] and len(got) == len(ref)
    for g, r in zip(got[1:], ref[1:]):
        assert g[:5] == r[:5], (g[:5], r[:5])
    g = np.array([[float(x) for x in row[5:]] for row in got[1:]])
    r = np.array([[float(x) for x in row[5:]] for row in ref[1:]])
    assert _close(g, r).all(), float((np.abs(g - r) / (1e-6 + 1e-5 * np.abs(r))).max())
    mask = re.compile(r"-?\d+\.\d+(e[-+]?\d+)?|-?\d+e[-+]?\d+")
    gj, rj = open(js_p).read(), open(os.path.join(GOLD, f"dropin_{scene}_ref.json")).read()
    assert mask.sub("N", gj) == mask.sub("N", rj), "manifold_to_json layout differs from the reference's"
    assert json.loads(gj)["layout"] == json.loads(rj)["layout"]
