// TEST INFRASTRUCTURE — not product code.
//
// Two more extern "C" entry points over the UNMODIFIED reference, compiled into
// oracle/_ref/libcmgref.so beside ref_harness.cpp (surfaces come from
// cmgref_surface_create there):
//
//   cmgref_opcount_manifold   SURVEY.md Appendix B's op counter: the reference's
//                             own generate_manifold<T> (proj/include/cmg/
//                             manifold.hpp:336-377) instantiated with a counting
//                             scalar (one add/sub/mul/div = 1 arith op; every
//                             transcendental = 1 op of its kind). Optionally
//                             generate_manifold<Dual<12, Counted>> with
//                             seed_pose_tangents (dual.hpp:249-262), the
//                             reference's own Jacobian formulation. This is how
//                             bench.py's algorithmic work per manifold W is
//                             defined for every configuration.
//   cmgref_scene_bench        the CPU reference of config D: every scene pair
//                             (DemoSim::step's enumeration, src/demosim.cpp:
//                             88-104) of every env through generate_manifold<
//                             double> or generate_manifold<Dual12> (main.cpp:
//                             202-205's gradcheck pattern), chunked over
//                             std::threads like parallel_for (batch.cpp:27-41)
//                             and timed by the reference's own time_run
//                             (batch.cpp:100-120).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "cmg/batch.hpp"
#include "cmg/dual.hpp"
#include "cmg/manifold.hpp"
#include "cmg/surface.hpp"
#include "cmgb.h"

namespace opcount {

struct Counts {
  int64_t arith = 0, pow = 0, sqrt = 0, exp = 0, log = 0, tanh = 0, other = 0;
};
inline Counts g;  // single-threaded counting only

struct Cnt {
  double v = 0.0;
  Cnt() = default;
  Cnt(double x) : v(x) {}  // NOLINT: implicit like a double
  Cnt(int x) : v(x) {}     // NOLINT
  Cnt& operator+=(const Cnt& o) { ++g.arith; v += o.v; return *this; }
  Cnt& operator-=(const Cnt& o) { ++g.arith; v -= o.v; return *this; }
  Cnt& operator*=(const Cnt& o) { ++g.arith; v *= o.v; return *this; }
  Cnt& operator/=(const Cnt& o) { ++g.arith; v /= o.v; return *this; }
};
inline Cnt operator+(const Cnt& a, const Cnt& b) { ++g.arith; return a.v + b.v; }
inline Cnt operator-(const Cnt& a, const Cnt& b) { ++g.arith; return a.v - b.v; }
inline Cnt operator*(const Cnt& a, const Cnt& b) { ++g.arith; return a.v * b.v; }
inline Cnt operator/(const Cnt& a, const Cnt& b) { ++g.arith; return a.v / b.v; }
inline Cnt operator+(const Cnt& a, double b) { ++g.arith; return a.v + b; }
inline Cnt operator-(const Cnt& a, double b) { ++g.arith; return a.v - b; }
inline Cnt operator*(const Cnt& a, double b) { ++g.arith; return a.v * b; }
inline Cnt operator/(const Cnt& a, double b) { ++g.arith; return a.v / b; }
inline Cnt operator+(double a, const Cnt& b) { ++g.arith; return a + b.v; }
inline Cnt operator-(double a, const Cnt& b) { ++g.arith; return a - b.v; }
inline Cnt operator*(double a, const Cnt& b) { ++g.arith; return a * b.v; }
inline Cnt operator/(double a, const Cnt& b) { ++g.arith; return a / b.v; }
inline Cnt operator-(const Cnt& a) { return -a.v; }
inline Cnt operator+(const Cnt& a) { return a; }
inline bool operator<(const Cnt& a, const Cnt& b) { return a.v < b.v; }
inline bool operator>(const Cnt& a, const Cnt& b) { return a.v > b.v; }
inline bool operator<=(const Cnt& a, const Cnt& b) { return a.v <= b.v; }
inline bool operator>=(const Cnt& a, const Cnt& b) { return a.v >= b.v; }
inline bool operator==(const Cnt& a, const Cnt& b) { return a.v == b.v; }
inline bool operator!=(const Cnt& a, const Cnt& b) { return a.v != b.v; }
inline double primal(const Cnt& x) { return x.v; }
inline Cnt exp(const Cnt& x) { ++g.exp; return std::exp(x.v); }
inline Cnt log(const Cnt& x) { ++g.log; return std::log(x.v); }
inline Cnt log1p(const Cnt& x) { ++g.log; return std::log1p(x.v); }
inline Cnt expm1(const Cnt& x) { ++g.exp; return std::expm1(x.v); }
inline Cnt sqrt(const Cnt& x) { ++g.sqrt; return std::sqrt(x.v); }
inline Cnt tanh(const Cnt& x) { ++g.tanh; return std::tanh(x.v); }
inline Cnt sin(const Cnt& x) { ++g.other; return std::sin(x.v); }
inline Cnt cos(const Cnt& x) { ++g.other; return std::cos(x.v); }
inline Cnt pow(const Cnt& x, double p) { ++g.pow; return std::pow(x.v, p); }
inline Cnt pow(const Cnt& x, const Cnt& p) { ++g.pow; return std::pow(x.v, p.v); }
inline Cnt fabs(const Cnt& x) { return std::fabs(x.v); }
inline Cnt abs(const Cnt& x) { return std::fabs(x.v); }

}  // namespace opcount

namespace {

using cmg::Pose6;
using cmg::SmoothingConfig;
using cmg::SurfaceModel;

SmoothingConfig to_cfg2(const cmgb_config* c) {
  SmoothingConfig s;
  s.lambda = c->lambda;
  s.tau_clip = c->tau_clip;
  s.tau_min = c->tau_min;
  s.tau_comp = c->tau_comp;
  s.tau_sign = c->tau_sign;
  s.tau_pen = c->tau_pen;
  s.tau_nn = c->tau_nn;
  s.tau_clash = c->tau_clash;
  s.tau_cont = c->tau_cont;
  s.tau_topk_verts = c->tau_topk_verts;
  s.tau_topk_edges = c->tau_topk_edges;
  s.tau_normal = c->tau_normal;
  s.tau_union = c->tau_union;
  s.hard_ops = c->hard_ops != 0;
  s.sphere_trace = c->sphere_trace != 0;
  s.sphere_trace_iters = c->sphere_trace_iters;
  s.containment_safeguard = c->containment_safeguard != 0;
  s.mode = c->mode == 1 ? cmg::ContactMode::kNoEe
                        : (c->mode == 2 ? cmg::ContactMode::kOneSided : cmg::ContactMode::kFull);
  return s;
}

template <class T>
Pose6<T> pose_of(const double* p) {
  return {T(p[0]), T(p[1]), T(p[2]), T(p[3]), T(p[4]), T(p[5])};
}

void put(const opcount::Counts& c, int64_t* out) {
  out[0] = c.arith;
  out[1] = c.pow;
  out[2] = c.sqrt;
  out[3] = c.exp;
  out[4] = c.log;
  out[5] = c.tanh;
  out[6] = c.other;
}

}  // namespace

extern "C" {

// counts out[7]: arith, pow, sqrt, exp (+expm1), log (+log1p), tanh, other (sin/cos).
// jvp = 0: generate_manifold<Counted>; 1: generate_manifold<Dual<12, Counted>>
// seeded at the 12 pose coordinates (the reference's Jacobian formulation).
int cmgref_opcount_manifold(void* h1, void* h2, const double* pose1, const double* pose2,
                            const cmgb_config* c, int jvp, int64_t* out) {
  using opcount::Cnt;
  const SurfaceModel& s1 = *static_cast<SurfaceModel*>(h1);
  const SurfaceModel& s2 = *static_cast<SurfaceModel*>(h2);
  const SmoothingConfig cfg = to_cfg2(c);
  opcount::g = {};
  if (!jvp) {
    const auto m = cmg::generate_manifold<Cnt>(s1, s2, pose_of<Cnt>(pose1), pose_of<Cnt>(pose2), cfg);
    (void)m;
  } else {
    using D = cmg::Dual<12, Cnt>;
    Pose6<D> a, b;
    for (int k = 0; k < 6; ++k) {
      a[k] = D(0.0);
      a[k].v = Cnt(pose1[k]);
      a[k].d[k] = Cnt(1.0);
      b[k] = D(0.0);
      b[k].v = Cnt(pose2[k]);
      b[k].d[6 + k] = Cnt(1.0);
    }
    opcount::g = {};
    const auto m = cmg::generate_manifold<D>(s1, s2, a, b, cfg);
    (void)m;
  }
  put(opcount::g, out);
  return 0;
}

// Config D's CPU reference: poses [n_env][n_bodies][6]; pairs [n_pairs][2].
// jvp = 0: generate_manifold<double> per pair; 1: generate_manifold<Dual12>
// per pair (seed_pose_tangents on the pair's two poses). Timed by time_run
// (median / population std over reps after `warmups`).
int cmgref_scene_bench(void* const* surfaces, int n_bodies, const int32_t* pairs, int n_pairs,
                       const double* poses, int64_t n_env, const cmgb_config* c, int jvp, int reps,
                       int warmups, int workers, double* median_s, double* std_s, double* checksum) {
  const SmoothingConfig cfg = to_cfg2(c);
  std::vector<double> sums(static_cast<size_t>(n_env), 0.0);
  auto body = [&](int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      double acc = 0.0;
      for (int q = 0; q < n_pairs; ++q) {
        const int i = pairs[2 * q], j = pairs[2 * q + 1];
        const SurfaceModel& si = *static_cast<SurfaceModel*>(surfaces[i]);
        const SurfaceModel& sj = *static_cast<SurfaceModel*>(surfaces[j]);
        const double* pi = poses + (e * n_bodies + i) * 6;
        const double* pj = poses + (e * n_bodies + j) * 6;
        if (jvp) {
          const auto seeded = cmg::seed_pose_tangents(
              std::array<double, 6>{pi[0], pi[1], pi[2], pi[3], pi[4], pi[5]},
              std::array<double, 6>{pj[0], pj[1], pj[2], pj[3], pj[4], pj[5]});
          const auto m = cmg::generate_manifold(si, sj, seeded.first, seeded.second, cfg);
          acc += cmg::primal(cmg::mean_contact_distance(m));
        } else {
          const auto m = cmg::generate_manifold(si, sj, pose_of<double>(pi), pose_of<double>(pj), cfg);
          acc += cmg::mean_contact_distance(m);
        }
      }
      sums[static_cast<size_t>(e)] = acc;
    }
  };
  auto run = [&] {
    const int w = std::max(1, workers);
    std::vector<std::thread> pool;
    const int64_t chunk = (n_env + w - 1) / w;
    for (int k = 0; k < w; ++k) {
      const int64_t lo = std::min<int64_t>(n_env, k * chunk);
      const int64_t hi = std::min<int64_t>(n_env, lo + chunk);
      if (lo < hi) pool.emplace_back(body, lo, hi);
    }
    for (auto& t : pool) t.join();
  };
  const cmg::TimingStats st = cmg::time_run(run, std::max(1, reps), std::max(0, warmups));
  *median_s = st.median_s;
  *std_s = st.std_s;
  double cs = 0.0;
  for (double v : sums) cs += v;
  *checksum = cs;
  return 0;
}

}  // extern "C"
