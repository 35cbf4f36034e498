// cmgb.hpp — thin RAII C++ wrapper over the C ABI (include/cmgb.h) for callers
// that manage DEVICE buffers and streams themselves (batched calls on device
// pointers, throwing on error). It does NOT have the reference's signatures:
// the reference-signature drop-in (namespace cmg: generate_manifold<T>,
// ContactManifold, run_ee_batch(problems, cfg, workers, out) -> checksum,
// bench_manifold(scene, ...), ...) is include/cmgb_cmg.hpp, reached through the
// forwarding headers include/cmg/*.hpp by swapping the include path.
//
//   cmg::make_box_mesh / parse_obj        -> cmgb::Mesh::box / Mesh::parse_obj
//   cmg::build_surface                     -> cmgb::Surface
//   cmg::SmoothingConfig (+ variants)      -> cmgb::SmoothingConfig
//   bench_manifold's per-env loop          -> cmgb::generate_manifold_batch (device poses / outputs)
//   cmg::run_ee_batch / run_vf_batch       -> cmgb::run_ee_batch / run_vf_batch (device pairs / outputs)
//
// Errors: std::invalid_argument / MeshParseError / std::runtime_error with the
// library's message.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "cmgb.h"

namespace cmgb {

struct MeshParseError : std::runtime_error {
  MeshParseError(const std::string& what, int line) : std::runtime_error(what), line_number(line) {}
  int line_number;
};

inline void check(int status) {
  if (status == CMGB_OK) return;
  const std::string msg = cmgb_last_error();
  if (status == CMGB_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct SmoothingConfig : cmgb_config {
  SmoothingConfig() { cmgb_config_default(this); }
  static SmoothingConfig no_smoothing() {
    SmoothingConfig c;
    cmgb_config_no_smoothing(&c);
    return c;
  }
  void validate() const { check(cmgb_config_validate(this)); }
  SmoothingConfig for_variant(const std::string& v) const {
    SmoothingConfig out;
    check(cmgb_config_for_variant(v.c_str(), this, &out));
    return out;
  }
};

class Mesh {
 public:
  static Mesh box(const double half[3], int subdivisions = 1, bool quad_edges = true) {
    cmgb_mesh m = nullptr;
    check(cmgb_mesh_box(half, subdivisions, quad_edges ? 1 : 0, &m));
    return Mesh(m);
  }
  static Mesh parse_obj(const std::string& text) {
    cmgb_mesh m = nullptr;
    int32_t line = 0;
    const int st = cmgb_mesh_parse_obj(text.data(), text.size(), &m, &line);
    if (st == CMGB_ERR_PARSE) throw MeshParseError(cmgb_last_error(), line);
    check(st);
    return Mesh(m);
  }
  Mesh(Mesh&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Mesh(const Mesh&) = delete;
  ~Mesh() { cmgb_mesh_destroy(h_); }
  cmgb_mesh handle() const { return h_; }

 private:
  explicit Mesh(cmgb_mesh h) : h_(h) {}
  cmgb_mesh h_;
};

class Surface {
 public:
  // build_surface(mesh, sdf, vertex_topk, edge_topk, tolerance_fraction)
  Surface(const Mesh& mesh, const std::vector<cmgb_sdf_node>& sdf_postfix, int vertex_topk = 0,
          int edge_topk = 0, double tolerance_fraction = 1e-2) {
    check(cmgb_surface_create(mesh.handle(), sdf_postfix.data(), (int32_t)sdf_postfix.size(),
                              vertex_topk, edge_topk, tolerance_fraction, &h_));
  }
  Surface(Surface&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Surface(const Surface&) = delete;
  ~Surface() { cmgb_surface_destroy(h_); }
  cmgb_surface handle() const { return h_; }
  cmgb_surface_info info() const {
    cmgb_surface_info i{};
    check(cmgb_surface_get_info(h_, &i));
    return i;
  }
  std::vector<std::string> build_warnings() const {
    std::vector<std::string> w;
    for (int i = 0; i < info().n_warnings; ++i) w.emplace_back(cmgb_surface_warning(h_, i));
    return w;
  }

 private:
  cmgb_surface h_ = nullptr;
};

inline cmgb_layout layout(const Surface& a, const Surface& b, const SmoothingConfig& c) {
  cmgb_layout L{};
  check(cmgb_layout_query(a.handle(), b.handle(), &c, &L));
  return L;
}

// Every env of a batch: device poses [n][6] (stride 0 = one pose for all),
// device outputs (cmgb_manifold_out); stream-ordered on `stream`.
inline void generate_manifold_batch(const Surface& a, const Surface& b, const double* poses1,
                                    int pose1_stride, const double* poses2, int pose2_stride,
                                    int64_t n_env, const SmoothingConfig& c,
                                    const cmgb_manifold_out& out, void* stream = nullptr) {
  check(cmgb_manifold_batch(a.handle(), b.handle(), poses1, pose1_stride, poses2, pose2_stride, n_env,
                            &c, &out, stream));
}

// Host buffers in and out (copies inside the call).
inline void generate_manifold_batch_host(const Surface& a, const Surface& b, const double* poses1,
                                         int pose1_stride, const double* poses2, int pose2_stride,
                                         int64_t n_env, const SmoothingConfig& c, float* mean_dist,
                                         float* contacts = nullptr, void* stream = nullptr) {
  check(cmgb_manifold_batch_host(a.handle(), b.handle(), poses1, pose1_stride, poses2, pose2_stride,
                                 n_env, &c, mean_dist, contacts, stream));
}

// generate_manifold<Dual12> with seed_pose_tangents (dual.hpp:249-263) for every
// env: primal contacts + their 12 pose tangents (smooth mode only).
inline void generate_manifold_jvp_batch(const Surface& a, const Surface& b, const double* poses1,
                                        int pose1_stride, const double* poses2, int pose2_stride,
                                        int64_t n_env, const SmoothingConfig& c,
                                        const cmgb_manifold_jvp_out& out, void* stream = nullptr) {
  check(cmgb_manifold_jvp_batch(a.handle(), b.handle(), poses1, pose1_stride, poses2, pose2_stride, n_env,
                                &c, &out, stream));
}

// DemoSim::step's pair loop (demosim.cpp:88-104): every non-static body pair.
inline std::vector<int32_t> scene_pairs(const std::vector<int32_t>& is_static) {
  int32_t n = 0;
  check(cmgb_scene_pairs(is_static.data(), (int32_t)is_static.size(), nullptr, &n));
  std::vector<int32_t> pairs(2 * (size_t)n);
  check(cmgb_scene_pairs(is_static.data(), (int32_t)is_static.size(), pairs.data(), &n));
  return pairs;
}

// poses: device [n_env][n_bodies][6]; outs[q] for pair q of `pairs`.
inline void generate_scene_batch(const std::vector<cmgb_surface>& bodies, const std::vector<int32_t>& pairs,
                                 const double* poses, int64_t n_env, const SmoothingConfig& c,
                                 const std::vector<cmgb_manifold_out>& outs, void* stream = nullptr) {
  check(cmgb_manifold_scene_batch(bodies.data(), (int32_t)bodies.size(), pairs.data(),
                                  (int32_t)(pairs.size() / 2), poses, n_env, &c, outs.data(), stream));
}

// SmoothSdf queries / sphere_trace_project on one surface (device buffers).
inline void sdf_query(const Surface& s, int flavor, const double* points, int64_t n, double* out,
                      void* stream = nullptr) {
  check(cmgb_sdf_query(s.handle(), flavor, points, n, out, stream));
}
inline void sphere_trace(const Surface& s, const double pose[6], const double* points, int64_t n, int iters,
                         double tau, double* out, void* stream = nullptr) {
  check(cmgb_sphere_trace(s.handle(), pose, points, n, iters, tau, out, stream));
}

// rotating_edge_sweep (src/sweep.cpp): rows of theta, p1 (3), dp1/dtheta (3).
inline std::vector<double> rotating_edge_sweep(int variant, int n_samples) {
  std::vector<double> out(7 * (size_t)n_samples);
  check(cmgb_rotating_edge_sweep(variant, n_samples, out.data()));
  return out;
}

// PenaltyParams{} and one DemoSim::step for a batch of scenes (device state,
// [n_env][n_bodies][6] poses / velocities updated in place).
inline cmgb_demo_params default_penalty_params() {
  cmgb_demo_params p;
  cmgb_demo_params_default(&p);
  return p;
}
inline void demo_step(const std::vector<cmgb_demo_body>& bodies, const SmoothingConfig& c,
                      const cmgb_demo_params& params, double dt, int64_t n_env, double* poses, double* velocities,
                      double* deepest = nullptr, int32_t* ok = nullptr, void* stream = nullptr) {
  check(cmgb_demo_step_batch(bodies.data(), (int32_t)bodies.size(), &c, &params, dt, n_env, poses, velocities,
                             deepest, ok, nullptr, 0, stream));
}

inline void run_ee_batch_f64(const double* pairs_device, int64_t n, const SmoothingConfig& c, double* out_device,
                             void* stream = nullptr) {
  check(cmgb_ee_witness_batch_f64(pairs_device, n, &c, out_device, nullptr, nullptr, stream));
}

inline void run_ee_batch(const double* pairs_device, int64_t n, const SmoothingConfig& c,
                         float* out_device, void* stream = nullptr) {
  check(cmgb_ee_witness_batch(pairs_device, 1, n, &c, out_device, nullptr, nullptr, stream));
}

inline void run_vf_batch(const double* pairs_device, int64_t n, const SmoothingConfig& c,
                         float* out_device, void* stream = nullptr) {
  check(cmgb_vf_witness_batch(pairs_device, 1, n, &c, out_device, nullptr, stream));
}

}  // namespace cmgb
