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
int main() {
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
