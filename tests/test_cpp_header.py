"""CPU: a C++ caller of the reference API builds against include/cmgb.hpp and
links libcmgb.so; host-side calls (mesh, surface, layout, config errors) run
without a GPU and reproduce the reference's counts and messages."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r"""
#include <cstdio>
#include "cmgb.hpp"
int main(int argc, char** argv) {
  (void)argv;
  const double half[3] = {0.5, 0.5, 0.5};
  cmgb::Mesh box = cmgb::Mesh::box(half);
  cmgb_sdf_node sq{};
  sq.op = CMGB_SDF_SUPERQUADRIC;
  sq.eps1 = sq.eps2 = 0.1;
  sq.axes[0] = sq.axes[1] = sq.axes[2] = 0.5;
  cmgb::Surface s(box, {sq}, 0, 12);
  cmgb::SmoothingConfig cfg;
  cmgb_layout L = cmgb::layout(s, s, cfg);
  std::printf("contacts %d warnings %zu\n", L.n_contacts, s.build_warnings().size());
  cmgb::SmoothingConfig bad;
  bad.tau_pen = 0.0;
  try { bad.validate(); } catch (const std::invalid_argument& e) { std::printf("err %s\n", e.what()); }
  try { cmgb::Mesh::parse_obj("v 0 0 0\nf 1 2 3\n"); }
  catch (const cmgb::MeshParseError& e) { std::printf("parse %d %s\n", e.line_number, e.what()); }
  const cmgb_demo_params pp = cmgb::default_penalty_params();
  std::printf("penalty %g %g %g\n", pp.stiffness, pp.tau_force, pp.gravity[2]);
  std::printf("pairs %zu\n", cmgb::scene_pairs({1, 0, 0, 0, 0}).size() / 2);
  if (argc > 99) {  // device entry points: compiled and linked here, exercised by the GPU suites
    double* d = nullptr;
    cmgb::sdf_query(s, 1, d, 0, d);
    const double pose[6] = {0, 0, 0, 0, 0, 0};
    cmgb::sphere_trace(s, pose, d, 0, 5, 1e-9, d);
    cmgb::rotating_edge_sweep(2, 16);
    cmgb_demo_body b{s.handle(), 1.0, {0, 0, 0}, 0, 0};
    cmgb::demo_step({b, b}, cfg, pp, 1e-3, 0, d, d);
    cmgb::run_ee_batch_f64(d, 0, cfg, d);
    cmgb_manifold_jvp_out jo{};
    cmgb::generate_manifold_jvp_batch(s, s, d, 1, d, 1, 0, cfg, jo);
  }
  return 0;
}
"""


def test_cpp_header_host_api(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(SRC)
    exe = tmp_path / "t"
    lib_dir = os.path.join(ROOT, "paper_2602_20304_b200")
    r = subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", f"-I{ROOT}/include", str(src), "-o", str(exe),
                        f"-L{lib_dir}", "-lcmgb", f"-Wl,-rpath,{lib_dir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.splitlines()
    assert lines[0] == "contacts 304 warnings 1"
    assert lines[1] == "err smoothing: tau_pen must be > 0"
    assert lines[2] == "parse 2 face index out of range (line 2)"
    assert lines[3] == "penalty 10000 0.0001 -9.81"  # PenaltyParams{} (demosim.hpp:24-31)
    assert lines[4] == "pairs 10"  # DemoSim::step's pairs of a 5-body scene with one static body
