// cmgb_cmg.hpp — the reference's C++ collision API (namespace cmg of
// /root/reference/proj/include/cmg) re-declared over the C ABI (cmgb.h), so a
// C++ caller of the reference switches to the B200 path by changing its
// include path: `-I<repo>/include` resolves "cmg/manifold.hpp" & co. to the
// forwarding headers in include/cmg/, which include this file. The reference
// names are declared in cmgb::ref and exposed as `namespace cmg` (define
// CMGB_NO_CMG_ALIAS to suppress the alias).
//
// Reference interface -> what runs here
//   Vec3 / Mat3 / Pose6 / Transform / se3_exp / so3_log (vec3.hpp, pose.hpp)   host math (setup only)
//   Dual<N> / seed_pose_tangents / extract_jacobian (dual.hpp:46-271)          forward-mode pose tangents
//   SmoothingConfig / ContactMode (config.hpp:8-74), config_for_variant         -> cmgb_config
//   CollisionMesh / make_box_mesh / parse_obj / load_obj (mesh.hpp:25-44)        -> cmgb_mesh_* (same vertex /
//                                                                                  edge order = same src_a/src_b)
//   SuperquadricParams / ConvexPolyhedronParams / OrientedPointcloudParams,
//   SmoothSdf factories (sdf.hpp:35-202)                                         -> postfix cmgb_sdf_node program
//   SurfaceModel / build_surface (surface.hpp:16-40)                             -> cmgb_surface (lazy, cached)
//   ContactPoint / EeIndicatorMatrices / ContactManifold (manifold.hpp:27-73)   same value types
//   generate_manifold<T> (manifold.hpp:336-377)                                  -> cmgb_manifold_batch_host_ex
//                                                                                  (T = double / float) or
//                                                                                  cmgb_manifold_jvp_batch_host
//                                                                                  (T = Dual<N>)
//   mean_contact_distance / activity_weighted_distance (manifold.hpp:379-391)   same
//   Scene / SceneBody (scene.hpp:15-27)                                          same value types
//   EeProblemSet / VfProblemSet / make_random_*_pairs / run_*_batch /
//   time_run / BenchRecord / write_bench_csv / bench_witness / bench_manifold
//   (batch.hpp:19-75)                                                            same signatures, GPU batches
//
// Results: contact fields are computed in FP64 on the device and returned as
// FP32 (the north star's output precision), widened to T; E-E witnesses of
// run_ee_batch come from the FP64-output solver. Errors throw the reference's
// exception types (std::invalid_argument, MeshParseError) with the library's
// messages. Differences (documented in INTEGRATION.md): the SDF tree is not
// queryable on its own (queries go through a surface: cmgb_sdf_query), the
// EeIndicatorMatrices of T = Dual are empty (the Jacobian kernel does not emit
// them), `workers` arguments are accepted and ignored (the GPU is the worker
// pool), and mutating a SurfaceModel's mesh / sdf after build_surface needs a
// new build_surface (budget changes are picked up).
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <functional>
#include <istream>
#include <iterator>
#include <memory>
#include <ostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include <filesystem>
#include <iomanip>

#include "cmgb.h"
#include "cmgb_json.hpp"

namespace cmgb {
namespace ref {

// ============================================================================ errors
struct MeshParseError : std::runtime_error {
  MeshParseError(const std::string& what, int line)
      : std::runtime_error(what + " (line " + std::to_string(line) + ")"), line_number(line) {}
  int line_number;
};

namespace detail {
[[noreturn]] inline void raise(int status) {
  const std::string msg = cmgb_last_error();
  if (status == CMGB_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline void ok(int status) {
  if (status != CMGB_OK) raise(status);
}
}  // namespace detail

// ============================================================================ scalars
// Forward-mode scalar with the reference's layout (dual.hpp:46-129): value v
// and N tangents d. Arithmetic is provided for caller-side reductions over
// returned manifolds (mean_contact_distance of a ContactManifold<Dual12>).
template <int N, class B = double>
struct Dual {
  static_assert(N >= 1, "Dual needs at least one tangent");
  using Base = B;
  static constexpr int tangent_width = N;
  B v{};
  std::array<B, N> d{};

  Dual() = default;
  template <class S, std::enable_if_t<std::is_arithmetic_v<S>, int> = 0>
  Dual(S s) : v(static_cast<B>(s)) {}  // NOLINT: implicit promotion as in the reference

  static Dual seeded(const B& value, int direction) {
    Dual r(value);
    r.d[direction] = B(1);
    return r;
  }
  friend Dual operator+(const Dual& a, const Dual& b) {
    Dual r;
    r.v = a.v + b.v;
    for (int i = 0; i < N; ++i) r.d[i] = a.d[i] + b.d[i];
    return r;
  }
  friend Dual operator-(const Dual& a, const Dual& b) {
    Dual r;
    r.v = a.v - b.v;
    for (int i = 0; i < N; ++i) r.d[i] = a.d[i] - b.d[i];
    return r;
  }
  friend Dual operator-(const Dual& a) {
    Dual r;
    r.v = -a.v;
    for (int i = 0; i < N; ++i) r.d[i] = -a.d[i];
    return r;
  }
  friend Dual operator*(const Dual& a, const Dual& b) {
    Dual r;
    r.v = a.v * b.v;
    for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
    return r;
  }
  friend Dual operator/(const Dual& a, const Dual& b) {
    Dual r;
    const B q = B(1) / b.v;
    r.v = a.v * q;
    for (int i = 0; i < N; ++i) r.d[i] = (a.d[i] - r.v * b.d[i]) * q;
    return r;
  }
  Dual& operator+=(const Dual& o) { return *this = *this + o; }
  Dual& operator-=(const Dual& o) { return *this = *this - o; }
  Dual& operator*=(const Dual& o) { return *this = *this * o; }
  Dual& operator/=(const Dual& o) { return *this = *this / o; }
  friend bool operator<(const Dual& a, const Dual& b) { return a.v < b.v; }
  friend bool operator>(const Dual& a, const Dual& b) { return a.v > b.v; }
  friend bool operator<=(const Dual& a, const Dual& b) { return a.v <= b.v; }
  friend bool operator>=(const Dual& a, const Dual& b) { return a.v >= b.v; }
  friend bool operator==(const Dual& a, const Dual& b) { return a.v == b.v; }
};
using Dual12 = Dual<12, double>;

inline double primal(double x) { return x; }
inline double primal(float x) { return x; }
template <int N, class B>
double primal(const Dual<N, B>& x) {
  return primal(x.v);
}

template <class T>
struct tangent_width {
  static constexpr int value = 0;
};
template <int N, class B>
struct tangent_width<Dual<N, B>> {
  static constexpr int value = N;
};

// Directions 0..5 track pose 1, 6..11 pose 2 (dual.hpp:252-262).
template <class D = Dual12>
std::pair<std::array<D, 6>, std::array<D, 6>> seed_pose_tangents(const std::array<double, 6>& pose1,
                                                                 const std::array<double, 6>& pose2) {
  static_assert(D::tangent_width >= 12, "need 12 tangent slots for two 6D poses");
  std::pair<std::array<D, 6>, std::array<D, 6>> out;
  for (int i = 0; i < 6; ++i) {
    out.first[i] = D::seeded(pose1[i], i);
    out.second[i] = D::seeded(pose2[i], 6 + i);
  }
  return out;
}

template <int N, class B>
std::vector<std::array<double, N>> extract_jacobian(const std::vector<Dual<N, B>>& outputs) {
  std::vector<std::array<double, N>> rows(outputs.size());
  for (size_t i = 0; i < outputs.size(); ++i)
    for (int j = 0; j < N; ++j) rows[i][j] = primal(outputs[i].d[j]);
  return rows;
}

// ============================================================================ geometry (host)
template <class T>
struct Vec3 {
  T x{}, y{}, z{};
  Vec3() = default;
  Vec3(T xx, T yy, T zz) : x(std::move(xx)), y(std::move(yy)), z(std::move(zz)) {}
  T& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  const T& operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  friend Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
  friend Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
  friend Vec3 operator-(const Vec3& a) { return {-a.x, -a.y, -a.z}; }
  friend Vec3 operator*(const Vec3& a, const T& k) { return {a.x * k, a.y * k, a.z * k}; }
  friend Vec3 operator*(const T& k, const Vec3& a) { return {a.x * k, a.y * k, a.z * k}; }
  friend Vec3 operator/(const Vec3& a, const T& k) { return {a.x / k, a.y / k, a.z / k}; }
  Vec3& operator+=(const Vec3& o) { return *this = *this + o; }
  Vec3& operator-=(const Vec3& o) { return *this = *this - o; }
};
using Vec3d = Vec3<double>;

template <class T>
T dot(const Vec3<T>& a, const Vec3<T>& b) {
  return a.x * b.x + a.y * b.y + a.z * b.z;
}
template <class T>
Vec3<T> cross(const Vec3<T>& a, const Vec3<T>& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class T>
T norm_sq(const Vec3<T>& a) {
  return dot(a, a);
}
template <class T>
T norm(const Vec3<T>& a) {
  using std::sqrt;
  return sqrt(norm_sq(a));
}
template <class T>
Vec3<T> normalize_smooth(const Vec3<T>& v, double tau) {
  using std::sqrt;
  return v * (T(1) / sqrt(T(tau) + norm_sq(v)));
}
template <class T, class U>
Vec3<T> vec_cast(const Vec3<U>& v) {
  return {T(v.x), T(v.y), T(v.z)};
}
template <class T>
Vec3<double> vec_primal(const Vec3<T>& v) {
  return {primal(v.x), primal(v.y), primal(v.z)};
}

// Row-major 3x3 (vec3.hpp:76-131).
template <class T>
struct Mat3 {
  std::array<T, 9> m{};
  static Mat3 identity() {
    Mat3 r;
    r.m[0] = r.m[4] = r.m[8] = T(1);
    return r;
  }
  T& operator()(int r, int c) { return m[3 * r + c]; }
  const T& operator()(int r, int c) const { return m[3 * r + c]; }
  friend Vec3<T> operator*(const Mat3& A, const Vec3<T>& v) {
    Vec3<T> r;
    for (int i = 0; i < 3; ++i) r[i] = A(i, 0) * v.x + A(i, 1) * v.y + A(i, 2) * v.z;
    return r;
  }
  friend Mat3 operator*(const Mat3& A, const Mat3& B) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        T acc = A(i, 0) * B(0, j);
        acc += A(i, 1) * B(1, j);
        acc += A(i, 2) * B(2, j);
        r(i, j) = acc;
      }
    return r;
  }
  friend Mat3 operator+(const Mat3& A, const Mat3& B) {
    Mat3 r;
    for (int k = 0; k < 9; ++k) r.m[k] = A.m[k] + B.m[k];
    return r;
  }
  friend Mat3 operator*(const Mat3& A, const T& k) {
    Mat3 r;
    for (int i = 0; i < 9; ++i) r.m[i] = A.m[i] * k;
    return r;
  }
  Mat3 transposed() const {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r(j, i) = (*this)(i, j);
    return r;
  }
  Vec3<T> t_mul(const Vec3<T>& v) const { return transposed() * v; }
};
using Mat3d = Mat3<double>;

template <class T>
using Pose6 = std::array<T, 6>;
using Pose6d = Pose6<double>;

template <class T>
struct Transform {
  Mat3<T> R = Mat3<T>::identity();
  Vec3<T> t{};
  Vec3<T> apply(const Vec3<T>& p) const { return R * p + t; }
  Vec3<T> apply_inverse(const Vec3<T>& p) const { return R.t_mul(p - t); }
};
using Transformd = Transform<double>;

inline Mat3d skew(const Vec3d& w) {
  Mat3d s;
  s(0, 1) = -w.z;
  s(0, 2) = w.y;
  s(1, 0) = w.z;
  s(1, 2) = -w.x;
  s(2, 0) = -w.y;
  s(2, 1) = w.x;
  return s;
}

namespace detail {
// Rodrigues coefficients sin(t)/t, (1 - cos t)/t^2, (1 - sin(t)/t)/t^2 with the
// reference's series branch below t^2 = 1e-8 (pose.hpp:45-65).
inline void rodrigues(double th2, double& a, double& b, double& c) {
  if (th2 < 1e-8) {
    a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    c = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
    return;
  }
  const double th = std::sqrt(th2);
  a = std::sin(th) / th;
  b = (1.0 - std::cos(th)) / th2;
  c = (1.0 - a) / th2;
}
}  // namespace detail

inline Mat3d so3_exp_d(const Vec3d& w) {
  double a, b, c;
  detail::rodrigues(norm_sq(w), a, b, c);
  const Mat3d W = skew(w);
  return Mat3d::identity() + W * a + (W * W) * b;
}

inline Transformd se3_exp(const Pose6d& xi) {
  const Vec3d w{xi[3], xi[4], xi[5]}, rho{xi[0], xi[1], xi[2]};
  double a, b, c;
  detail::rodrigues(norm_sq(w), a, b, c);
  const Mat3d W = skew(w), W2 = W * W;
  Transformd out;
  out.R = Mat3d::identity() + W * a + W2 * b;
  out.t = (Mat3d::identity() + W * b + W2 * c) * rho;
  return out;
}

// Log map for angles in [0, pi) (pose.hpp:93-98), near-pi axis from the
// dominant column of (R + I) / 2.
inline Vec3d so3_log(const Mat3d& r) {
  const double ct = std::min(1.0, std::max(-1.0, 0.5 * (r(0, 0) + r(1, 1) + r(2, 2) - 1.0)));
  const double th = std::acos(ct);
  const Vec3d v{r(2, 1) - r(1, 2), r(0, 2) - r(2, 0), r(1, 0) - r(0, 1)};
  if (th < 1e-8) return v * 0.5;
  if (th > M_PI - 1e-6) {
    int k = 0;
    for (int i = 1; i < 3; ++i)
      if (r(i, i) > r(k, k)) k = i;
    Vec3d axis{r(0, k), r(1, k), r(2, k)};
    axis[k] += 1.0;
    return axis * (th / norm(axis));
  }
  return v * (0.5 * th / std::sin(th));
}

inline Pose6d se3_log(const Transformd& tf) {
  const Vec3d w = so3_log(tf.R);
  const double th2 = norm_sq(w);
  double k;
  if (th2 < 1e-8) {
    k = 1.0 / 12.0;
  } else {
    const double th = std::sqrt(th2), h = 0.5 * th;
    k = (1.0 - h * std::cos(h) / std::sin(h)) / th2;
  }
  const Mat3d W = skew(w);
  const Vec3d rho = (Mat3d::identity() + W * (-0.5) + (W * W) * k) * tf.t;
  return {rho.x, rho.y, rho.z, w.x, w.y, w.z};
}

// ============================================================================ config
enum class ContactMode { kFull, kNoEe, kOneSided };

struct SmoothingConfig {
  double lambda = 0.01;
  double tau_clip = 0.1;
  double tau_min = 0.1;
  double tau_comp = 0.1;
  bool hard_ops = false;
  double tau_sign = 0.1;
  double tau_pen = 0.01;
  double tau_nn = 0.01;
  double tau_clash = 0.1;
  double tau_cont = 0.01;
  double tau_topk_verts = 0.01;
  double tau_topk_edges = 0.01;
  double tau_normal = 1e-9;
  double tau_union = 0.01;
  bool sphere_trace = true;
  int sphere_trace_iters = 5;
  bool containment_safeguard = false;
  ContactMode mode = ContactMode::kFull;
  static constexpr double kEdgeNormalEps = 1e-12;

  static SmoothingConfig no_smoothing() {
    SmoothingConfig c;
    c.lambda = 1e-6;
    c.hard_ops = true;
    return c;
  }
  cmgb_config to_c() const {
    cmgb_config c{};
    c.lambda = lambda;
    c.tau_clip = tau_clip;
    c.tau_min = tau_min;
    c.tau_comp = tau_comp;
    c.tau_sign = tau_sign;
    c.tau_pen = tau_pen;
    c.tau_nn = tau_nn;
    c.tau_clash = tau_clash;
    c.tau_cont = tau_cont;
    c.tau_topk_verts = tau_topk_verts;
    c.tau_topk_edges = tau_topk_edges;
    c.tau_normal = tau_normal;
    c.tau_union = tau_union;
    c.hard_ops = hard_ops ? 1 : 0;
    c.sphere_trace = sphere_trace ? 1 : 0;
    c.sphere_trace_iters = sphere_trace_iters;
    c.containment_safeguard = containment_safeguard ? 1 : 0;
    c.mode = mode == ContactMode::kFull ? CMGB_MODE_FULL
                                        : (mode == ContactMode::kNoEe ? CMGB_MODE_NO_EE : CMGB_MODE_ONE_SIDED);
    return c;
  }
  // Same checks and messages as config.hpp:55-73 (done by the library).
  void validate() const {
    const cmgb_config c = to_c();
    detail::ok(cmgb_config_validate(&c));
  }
};

inline SmoothingConfig config_for_variant(const std::string& variant, SmoothingConfig base) {
  const cmgb_config in = base.to_c();
  cmgb_config out{};
  detail::ok(cmgb_config_for_variant(variant.c_str(), &in, &out));
  base.hard_ops = out.hard_ops != 0;
  base.lambda = out.lambda;
  base.mode = out.mode == CMGB_MODE_FULL ? ContactMode::kFull
                                         : (out.mode == CMGB_MODE_NO_EE ? ContactMode::kNoEe : ContactMode::kOneSided);
  return base;
}

// ============================================================================ meshes
struct CollisionMesh {
  std::vector<Vec3d> vertices;
  std::vector<std::array<int, 3>> faces;
  std::vector<std::array<int, 2>> edges;
  std::vector<std::string> warnings;

  Vec3d aabb_min() const {
    Vec3d m = vertices.empty() ? Vec3d{} : vertices[0];
    for (const auto& v : vertices)
      for (int k = 0; k < 3; ++k) m[k] = std::min(m[k], v[k]);
    return m;
  }
  Vec3d aabb_max() const {
    Vec3d m = vertices.empty() ? Vec3d{} : vertices[0];
    for (const auto& v : vertices)
      for (int k = 0; k < 3; ++k) m[k] = std::max(m[k], v[k]);
    return m;
  }
  double bounding_diagonal() const { return norm(aabb_max() - aabb_min()); }
};

namespace detail {
// Library mesh handle -> value type (vertex / face / edge order preserved).
inline CollisionMesh read_mesh(cmgb_mesh h) {
  int32_t nv = 0, nf = 0, ne = 0, nw = 0;
  ok(cmgb_mesh_sizes(h, &nv, &nf, &ne, &nw));
  std::vector<double> v(3 * (size_t)nv);
  std::vector<int32_t> f(3 * (size_t)nf), e(2 * (size_t)ne);
  ok(cmgb_mesh_read(h, v.data(), f.data(), e.data()));
  CollisionMesh m;
  for (int i = 0; i < nv; ++i) m.vertices.push_back({v[3 * i], v[3 * i + 1], v[3 * i + 2]});
  for (int i = 0; i < nf; ++i) m.faces.push_back({f[3 * i], f[3 * i + 1], f[3 * i + 2]});
  for (int i = 0; i < ne; ++i) m.edges.push_back({e[2 * i], e[2 * i + 1]});
  for (int i = 0; i < nw; ++i) m.warnings.emplace_back(cmgb_mesh_warning(h, i));
  cmgb_mesh_destroy(h);
  return m;
}
inline cmgb_mesh mesh_handle(const CollisionMesh& m) {
  std::vector<double> v;
  std::vector<int32_t> f, e;
  for (const auto& x : m.vertices) v.insert(v.end(), {x.x, x.y, x.z});
  for (const auto& x : m.faces) f.insert(f.end(), {x[0], x[1], x[2]});
  for (const auto& x : m.edges) e.insert(e.end(), {x[0], x[1]});
  cmgb_mesh h = nullptr;
  ok(cmgb_mesh_from_arrays(v.data(), (int32_t)m.vertices.size(), f.data(), (int32_t)m.faces.size(), e.data(),
                           (int32_t)m.edges.size(), &h));
  return h;
}
}  // namespace detail

inline CollisionMesh make_box_mesh(const Vec3d& half_extents, int subdivisions = 1, bool quad_edges = true) {
  const double h[3] = {half_extents.x, half_extents.y, half_extents.z};
  cmgb_mesh m = nullptr;
  detail::ok(cmgb_mesh_box(h, subdivisions, quad_edges ? 1 : 0, &m));
  return detail::read_mesh(m);
}

inline CollisionMesh parse_obj(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  cmgb_mesh m = nullptr;
  int32_t line = 0;
  const int st = cmgb_mesh_parse_obj(text.data(), text.size(), &m, &line);
  if (st == CMGB_ERR_PARSE) {
    // the library message already carries " (line N)"; rebuild it the reference's way
    std::string msg = cmgb_last_error();
    const std::string tail = " (line " + std::to_string(line) + ")";
    if (msg.size() >= tail.size() && msg.compare(msg.size() - tail.size(), tail.size(), tail) == 0)
      msg.erase(msg.size() - tail.size());
    throw MeshParseError(msg, line);
  }
  detail::ok(st);
  return detail::read_mesh(m);
}

inline CollisionMesh load_obj(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("cannot open mesh file: " + path);
  return parse_obj(f);
}

// ============================================================================ SDF programs
inline constexpr double kSquaredCoordFloor = 1e-30;
inline constexpr double kRadiusGuard = 1e-20;
inline constexpr double kWeightFloor = 1e-30;

struct SuperquadricParams {
  double eps1 = 1.0;
  double eps2 = 1.0;
  Vec3d axes{1.0, 1.0, 1.0};
  Pose6d pose{0, 0, 0, 0, 0, 0};
};
struct ConvexPolyhedronParams {
  std::vector<Vec3d> normals;
  std::vector<Vec3d> points;
  double tau = 1e-3;
};
struct OrientedPointcloudParams {
  std::vector<Vec3d> points;
  std::vector<Vec3d> normals;
  std::vector<double> lengthscales;
};

// The reference's SmoothSdf tree (private nodes, sdf.hpp:160-202) as a value
// holding the public postfix program the ABI takes (cmgb_sdf_node); array
// payloads are owned here and re-pointed on every flatten.
class SmoothSdf {
 public:
  SmoothSdf() : SmoothSdf(superquadric(SuperquadricParams{})) {}  // unit sphere, as the reference

  static SmoothSdf superquadric(SuperquadricParams q) {
    SmoothSdf s(0);
    Node n;
    n.op = CMGB_SDF_SUPERQUADRIC;
    n.eps1 = q.eps1;
    n.eps2 = q.eps2;
    n.axes = {q.axes.x, q.axes.y, q.axes.z};
    n.pose = q.pose;
    s.nodes_.push_back(std::move(n));
    return s;
  }
  static SmoothSdf convex_polyhedron(ConvexPolyhedronParams cp) {
    SmoothSdf s(0);
    Node n;
    n.op = CMGB_SDF_CONVEX_POLYHEDRON;
    n.count = (int)cp.normals.size();
    n.tau = cp.tau;
    if (cp.normals.size() != cp.points.size())
      throw std::invalid_argument("convex polyhedron: need matching normals/points, N >= 1");
    for (size_t i = 0; i < cp.normals.size(); ++i) {
      n.normals.insert(n.normals.end(), {cp.normals[i].x, cp.normals[i].y, cp.normals[i].z});
      n.points.insert(n.points.end(), {cp.points[i].x, cp.points[i].y, cp.points[i].z});
    }
    s.nodes_.push_back(std::move(n));
    return s;
  }
  static SmoothSdf oriented_pointcloud(OrientedPointcloudParams pc) {
    SmoothSdf s(0);
    Node n;
    n.op = CMGB_SDF_ORIENTED_POINTCLOUD;
    n.count = (int)pc.points.size();
    if (pc.points.size() != pc.normals.size() || pc.points.size() != pc.lengthscales.size())
      throw std::invalid_argument("oriented pointcloud: need matching arrays, N >= 1");
    for (size_t i = 0; i < pc.points.size(); ++i) {
      n.points.insert(n.points.end(), {pc.points[i].x, pc.points[i].y, pc.points[i].z});
      n.normals.insert(n.normals.end(), {pc.normals[i].x, pc.normals[i].y, pc.normals[i].z});
    }
    n.lengthscales = pc.lengthscales;
    s.nodes_.push_back(std::move(n));
    return s;
  }
  static SmoothSdf smooth_union(std::vector<SmoothSdf> children, double tau) {
    if (children.empty()) throw std::invalid_argument("union: need at least one child");
    SmoothSdf s(0);
    for (auto& c : children) s.nodes_.insert(s.nodes_.end(), c.nodes_.begin(), c.nodes_.end());
    Node n;
    n.op = CMGB_SDF_UNION;
    n.count = (int)children.size();
    n.tau = tau;
    s.nodes_.push_back(std::move(n));
    return s;
  }
  static SmoothSdf subtraction(SmoothSdf positive, SmoothSdf negative, double tau) {
    SmoothSdf s(0);
    s.nodes_ = std::move(positive.nodes_);
    s.nodes_.insert(s.nodes_.end(), negative.nodes_.begin(), negative.nodes_.end());
    Node n;
    n.op = CMGB_SDF_SUBTRACTION;
    n.count = 2;
    n.tau = tau;
    s.nodes_.push_back(std::move(n));
    return s;
  }

  size_t leaf_count() const {
    size_t k = 0;
    for (const auto& n : nodes_) k += n.op <= CMGB_SDF_ORIENTED_POINTCLOUD;
    return k;
  }
  // The ABI's postfix program (pointers into this object; valid while it lives).
  std::vector<cmgb_sdf_node> program() const {
    std::vector<cmgb_sdf_node> out;
    for (const auto& n : nodes_) {
      cmgb_sdf_node c{};
      c.op = n.op;
      c.count = n.count;
      c.tau = n.tau;
      c.eps1 = n.eps1;
      c.eps2 = n.eps2;
      for (int k = 0; k < 3; ++k) c.axes[k] = n.axes[k];
      for (int k = 0; k < 6; ++k) c.pose[k] = n.pose[k];
      c.normals = n.normals.empty() ? nullptr : n.normals.data();
      c.points = n.points.empty() ? nullptr : n.points.data();
      c.lengthscales = n.lengthscales.empty() ? nullptr : n.lengthscales.data();
      out.push_back(c);
    }
    return out;
  }

 private:
  struct Node {
    int op = 0, count = 0;
    double tau = 0.0, eps1 = 1.0, eps2 = 1.0;
    std::array<double, 3> axes{1.0, 1.0, 1.0};
    std::array<double, 6> pose{0, 0, 0, 0, 0, 0};
    std::vector<double> normals, points, lengthscales;
  };
  explicit SmoothSdf(int) {}
  std::vector<Node> nodes_;
};

// ============================================================================ surfaces
struct SurfaceModel;
namespace detail {
struct SurfaceHandle {
  cmgb_surface h = nullptr;
  int vertex_topk = 0, edge_topk = 0;
  ~SurfaceHandle() {
    if (h) cmgb_surface_destroy(h);
  }
};
}  // namespace detail

struct SurfaceModel {
  CollisionMesh mesh;
  SmoothSdf sdf;
  int vertex_topk = 0;
  int edge_topk = 0;
  std::vector<std::string> build_warnings;

  int effective_vertex_topk() const {
    const int v = (int)mesh.vertices.size();
    return vertex_topk <= 0 ? v : std::min(vertex_topk, v);
  }
  int effective_edge_topk() const {
    const int e = (int)mesh.edges.size();
    return edge_topk <= 0 ? std::min((int)sdf.leaf_count(), e) : std::min(edge_topk, e);
  }
  // The library surface of this model (created by build_surface; re-created if
  // the budgets were changed since, as the reference CLI's top-K overrides do).
  cmgb_surface handle() const {
    if (!cache_ || cache_->vertex_topk != vertex_topk || cache_->edge_topk != edge_topk)
      cache_ = make_handle(tolerance_fraction_, nullptr);
    return cache_->h;
  }

 private:
  friend SurfaceModel build_surface(CollisionMesh, SmoothSdf, int, int, double);
  std::shared_ptr<detail::SurfaceHandle> make_handle(double tol, std::vector<std::string>* warnings) const {
    auto hd = std::make_shared<detail::SurfaceHandle>();
    cmgb_mesh m = detail::mesh_handle(mesh);
    const std::vector<cmgb_sdf_node> prog = sdf.program();
    const int st = cmgb_surface_create(m, prog.data(), (int32_t)prog.size(), vertex_topk, edge_topk, tol, &hd->h);
    cmgb_mesh_destroy(m);
    detail::ok(st);
    hd->vertex_topk = vertex_topk;
    hd->edge_topk = edge_topk;
    if (warnings) {
      cmgb_surface_info info{};
      detail::ok(cmgb_surface_get_info(hd->h, &info));
      for (int i = 0; i < info.n_warnings; ++i) warnings->emplace_back(cmgb_surface_warning(hd->h, i));
    }
    return hd;
  }
  double tolerance_fraction_ = 1e-2;
  mutable std::shared_ptr<detail::SurfaceHandle> cache_;
};

// Validation and the mesh/SDF agreement warning happen in the library with the
// reference's messages (surface.cpp:9-44).
inline SurfaceModel build_surface(CollisionMesh mesh, SmoothSdf sdf, int vertex_topk = 0, int edge_topk = 0,
                                  double tolerance_fraction = 1e-2) {
  SurfaceModel s;
  s.mesh = std::move(mesh);
  s.sdf = std::move(sdf);
  s.vertex_topk = vertex_topk;
  s.edge_topk = edge_topk;
  s.tolerance_fraction_ = tolerance_fraction;
  s.build_warnings = s.mesh.warnings;  // then the library's mesh/SDF discrepancy warning, if any
  s.cache_ = s.make_handle(tolerance_fraction, &s.build_warnings);
  return s;
}

// ============================================================================ manifolds
enum class ContactKind { kVertexSdf, kEdgeEdge };

template <class T>
struct ContactPoint {
  Vec3<T> point{};
  T dist{};
  Vec3<T> normal{};
  T activity{};
  ContactKind kind = ContactKind::kVertexSdf;
  int side = 1;
  int src_a = -1;
  int src_b = -1;
};

template <class T>
struct EeIndicatorMatrices {
  size_t m1 = 0, m2 = 0;
  std::vector<T> dist, con, pen1, pen2, nn1, nn2, clash, act1, act2;
  const T& at(const std::vector<T>& m, size_t k, size_t l) const { return m[k * m2 + l]; }
};

template <class T>
struct ContactManifold {
  int n1 = 0, n2 = 0;
  int m1 = 0, m2 = 0;
  ContactMode mode = ContactMode::kFull;
  std::vector<ContactPoint<T>> contacts;
  EeIndicatorMatrices<T> ee;

  size_t expected_size() const {
    switch (mode) {
      case ContactMode::kFull:
        return size_t(n1) + size_t(n2) + 2 * size_t(m1) * size_t(m2);
      case ContactMode::kNoEe:
        return size_t(n1) + size_t(n2);
      case ContactMode::kOneSided:
        return size_t(n1);
    }
    return 0;
  }
};

namespace detail {

template <class T>
struct is_dual : std::false_type {};
template <int N, class B>
struct is_dual<Dual<N, B>> : std::true_type {};

struct LayoutInfo {
  cmgb_layout L{};
  std::vector<int32_t> kind, side, src_a, src_b;
};
inline LayoutInfo layout_info(cmgb_surface a, cmgb_surface b, const cmgb_config& c) {
  LayoutInfo li;
  ok(cmgb_layout_query(a, b, &c, &li.L));
  const size_t n = (size_t)li.L.n_contacts;
  li.kind.resize(n);
  li.side.resize(n);
  li.src_a.resize(n);
  li.src_b.resize(n);
  ok(cmgb_layout_metadata(a, b, &c, li.kind.data(), li.side.data(), li.src_a.data(), li.src_b.data()));
  return li;
}

template <class T>
ContactManifold<T> shell(const LayoutInfo& li, ContactMode mode) {
  ContactManifold<T> m;
  m.n1 = li.L.n1;
  m.n2 = li.L.n2;
  m.m1 = li.L.m1;
  m.m2 = li.L.m2;
  m.mode = mode;
  m.contacts.resize((size_t)li.L.n_contacts);
  for (size_t i = 0; i < m.contacts.size(); ++i) {
    m.contacts[i].kind = li.kind[i] ? ContactKind::kEdgeEdge : ContactKind::kVertexSdf;
    m.contacts[i].side = li.side[i];
  }
  return m;
}

// Every env of a pose batch (poses [n][6] FP64, stride 0 = shared) -> value manifolds.
template <class T>
std::vector<ContactManifold<T>> manifolds_f(const SurfaceModel& s1, const SurfaceModel& s2, const double* p1,
                                            int st1, const double* p2, int st2, int64_t n,
                                            const SmoothingConfig& cfg, bool want_ee) {
  const cmgb_config c = cfg.to_c();
  const LayoutInfo li = layout_info(s1.handle(), s2.handle(), c);
  const size_t C = (size_t)li.L.n_contacts, P = (size_t)li.L.m1 * li.L.m2;
  const bool ee = want_ee && P > 0 && cfg.mode == ContactMode::kFull;
  std::vector<float> contacts((size_t)n * C * 8), eem(ee ? (size_t)n * 9 * P : 0);
  std::vector<int32_t> src((size_t)n * C * 2);
  cmgb_manifold_out o{contacts.data(), src.data(), ee ? eem.data() : nullptr, nullptr, nullptr, 0, nullptr, nullptr, 0.0f, 0};
  ok(cmgb_manifold_batch_host_ex(s1.handle(), s2.handle(), p1, st1, p2, st2, n, &c, &o, nullptr));
  std::vector<ContactManifold<T>> out;
  out.reserve((size_t)n);
  for (int64_t e = 0; e < n; ++e) {
    ContactManifold<T> m = shell<T>(li, cfg.mode);
    const float* ce = contacts.data() + (size_t)e * C * 8;
    const int32_t* se = src.data() + (size_t)e * C * 2;
    for (size_t i = 0; i < C; ++i) {
      ContactPoint<T>& cp = m.contacts[i];
      const float* f = ce + 8 * i;
      cp.point = {T(f[0]), T(f[1]), T(f[2])};
      cp.dist = T(f[3]);
      cp.normal = {T(f[4]), T(f[5]), T(f[6])};
      cp.activity = T(f[7]);
      cp.src_a = se[2 * i];
      cp.src_b = se[2 * i + 1];
    }
    if (P > 0 && cfg.mode == ContactMode::kFull) {
      m.ee.m1 = (size_t)li.L.m1;
      m.ee.m2 = (size_t)li.L.m2;
      if (ee) {
        const float* E = eem.data() + (size_t)e * 9 * P;
        std::vector<T>* rows[9] = {&m.ee.dist, &m.ee.con,   &m.ee.pen1, &m.ee.pen2, &m.ee.nn1,
                                   &m.ee.nn2,  &m.ee.clash, &m.ee.act1, &m.ee.act2};
        for (int r = 0; r < 9; ++r) rows[r]->assign(E + r * P, E + (r + 1) * P);
      }
    }
    out.push_back(std::move(m));
  }
  return out;
}

// Pose-Jacobian path: the device computes d(field)/d(pose coordinate) for the
// 12 coordinates; the caller's seeds (any Dual<N>) enter by the chain rule
// out.d[j] = sum_k J[k] dpose_k/d(direction j).
template <int N, class B>
std::vector<ContactManifold<Dual<N, B>>> manifolds_jvp(const SurfaceModel& s1, const SurfaceModel& s2,
                                                       const std::vector<Pose6<Dual<N, B>>>& q1,
                                                       const std::vector<Pose6<Dual<N, B>>>& q2,
                                                       const SmoothingConfig& cfg) {
  using D = Dual<N, B>;
  const cmgb_config c = cfg.to_c();
  const LayoutInfo li = layout_info(s1.handle(), s2.handle(), c);
  const int64_t n = (int64_t)std::max(q1.size(), q2.size());
  const int st1 = q1.size() == (size_t)n ? 1 : 0, st2 = q2.size() == (size_t)n ? 1 : 0;
  std::vector<double> p1(6 * q1.size()), p2(6 * q2.size());
  for (size_t e = 0; e < q1.size(); ++e)
    for (int k = 0; k < 6; ++k) p1[6 * e + k] = primal(q1[e][k]);
  for (size_t e = 0; e < q2.size(); ++e)
    for (int k = 0; k < 6; ++k) p2[6 * e + k] = primal(q2[e][k]);
  const size_t C = (size_t)li.L.n_contacts;
  std::vector<float> contacts((size_t)n * C * 8), tangents((size_t)n * C * 96);
  std::vector<int32_t> src((size_t)n * C * 2);
  cmgb_manifold_jvp_out o{contacts.data(), tangents.data(), src.data(), nullptr, nullptr, nullptr, nullptr};
  ok(cmgb_manifold_jvp_batch_host(s1.handle(), s2.handle(), p1.data(), st1, p2.data(), st2, n, &c, &o, nullptr));
  std::vector<ContactManifold<D>> out;
  for (int64_t e = 0; e < n; ++e) {
    const Pose6<D>& a = q1[st1 ? e : 0];
    const Pose6<D>& b = q2[st2 ? e : 0];
    ContactManifold<D> m = shell<D>(li, cfg.mode);
    if (li.L.m1 > 0 && li.L.m2 > 0 && cfg.mode == ContactMode::kFull) {
      m.ee.m1 = (size_t)li.L.m1;
      m.ee.m2 = (size_t)li.L.m2;
    }
    for (size_t i = 0; i < C; ++i) {
      D f[8];
      for (int q = 0; q < 8; ++q) {
        const size_t base = (((size_t)e * C + i) * 8 + q);
        f[q].v = B(contacts[base]);
        const float* J = tangents.data() + base * 12;
        for (int j = 0; j < N; ++j) {
          double acc = 0.0;
          for (int k = 0; k < 6; ++k) acc += (double)J[k] * primal(a[k].d[j]) + (double)J[6 + k] * primal(b[k].d[j]);
          f[q].d[j] = B(acc);
        }
      }
      ContactPoint<D>& cp = m.contacts[i];
      cp.point = {f[0], f[1], f[2]};
      cp.dist = f[3];
      cp.normal = {f[4], f[5], f[6]};
      cp.activity = f[7];
      cp.src_a = src[((size_t)e * C + i) * 2];
      cp.src_b = src[((size_t)e * C + i) * 2 + 1];
    }
    out.push_back(std::move(m));
  }
  return out;
}

}  // namespace detail

// generate_manifold<T> (manifold.hpp:336-377) for one pose pair.
template <class T>
ContactManifold<T> generate_manifold(const SurfaceModel& s1, const SurfaceModel& s2, const Pose6<T>& pose1,
                                     const Pose6<T>& pose2, const SmoothingConfig& cfg) {
  if constexpr (detail::is_dual<T>::value) {
    return std::move(detail::manifolds_jvp(s1, s2, std::vector<Pose6<T>>{pose1}, std::vector<Pose6<T>>{pose2},
                                           cfg)[0]);
  } else {
    static_assert(std::is_floating_point_v<T>, "generate_manifold: T = float, double or Dual<N>");
    double p1[6], p2[6];
    for (int k = 0; k < 6; ++k) {
      p1[k] = (double)pose1[k];
      p2[k] = (double)pose2[k];
    }
    return std::move(detail::manifolds_f<T>(s1, s2, p1, 1, p2, 1, 1, cfg, true)[0]);
  }
}

// Batched extension (the loop body of bench_manifold, batch.cpp:207-215, as
// one call): poses1 / poses2 hold one pose per env or a single shared pose.
template <class T>
std::vector<ContactManifold<T>> generate_manifolds(const SurfaceModel& s1, const SurfaceModel& s2,
                                                   const std::vector<Pose6<T>>& poses1,
                                                   const std::vector<Pose6<T>>& poses2,
                                                   const SmoothingConfig& cfg, bool want_ee = false) {
  const size_t n = std::max(poses1.size(), poses2.size());
  for (size_t r : {poses1.size(), poses2.size()})
    if (r != n && r != 1) throw std::invalid_argument("generate_manifolds: pose arrays need n or 1 entries");
  if (n == 0) return {};
  if constexpr (detail::is_dual<T>::value) {
    return detail::manifolds_jvp(s1, s2, poses1, poses2, cfg);
  } else {
    std::vector<double> p1, p2;
    for (const auto& p : poses1)
      for (int k = 0; k < 6; ++k) p1.push_back((double)p[k]);
    for (const auto& p : poses2)
      for (int k = 0; k < 6; ++k) p2.push_back((double)p[k]);
    const int st1 = poses1.size() == n && n > 1 ? 1 : (n == 1 ? 1 : 0);
    const int st2 = poses2.size() == n && n > 1 ? 1 : (n == 1 ? 1 : 0);
    return detail::manifolds_f<T>(s1, s2, p1.data(), st1, p2.data(), st2, (int64_t)n, cfg, want_ee);
  }
}

template <class T>
T mean_contact_distance(const ContactManifold<T>& m) {
  T acc = T(0);
  for (const auto& c : m.contacts) acc += c.dist;
  return acc / T(double(m.contacts.size()));
}

template <class T>
T activity_weighted_distance(const ContactManifold<T>& m) {
  T acc = T(0);
  for (const auto& c : m.contacts) acc += c.activity * c.dist;
  return acc;
}

// ============================================================================ scenes
struct SceneBody {
  std::string name;
  SurfaceModel surface;
  Pose6d pose{0, 0, 0, 0, 0, 0};
  double mass = 1.0;
  Vec3d inertia_diag{0, 0, 0};
  bool is_static = false;
};

struct Scene {
  std::vector<SceneBody> bodies;
  SmoothingConfig smoothing;
};

struct SceneError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ============================================================================ batches (batch.hpp)
struct EeProblemSet {
  size_t count = 0;
  std::vector<double> data;
};
struct VfProblemSet {
  size_t count = 0;
  std::vector<double> data;
};

namespace detail {
// std::mt19937_64(seed) + uniform_real_distribution(0, 1): the same standard
// library draws as the reference (batch.cpp:18-24).
inline std::vector<double> unit_cube(size_t n, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<double> v(n);
  for (auto& x : v) x = u(rng);
  return v;
}
}  // namespace detail

inline EeProblemSet make_random_ee_pairs(size_t n, uint64_t seed) { return {n, detail::unit_cube(12 * n, seed)}; }
inline VfProblemSet make_random_vf_pairs(size_t n, uint64_t seed) { return {n, detail::unit_cube(12 * n, seed)}; }

// Witness points of every pair (6 doubles / pair E-E, 3 V-F) into *out;
// returns the checksum over them (batch.cpp:53-98). `workers` is ignored.
inline double run_ee_batch(const EeProblemSet& problems, const SmoothingConfig& cfg, int workers = 1,
                           std::vector<double>* out = nullptr) {
  (void)workers;
  std::vector<double> local;
  std::vector<double>& r = out ? *out : local;
  r.assign(6 * problems.count, 0.0);
  const cmgb_config c = cfg.to_c();
  detail::ok(cmgb_ee_witness_batch_host(problems.data.data(), (int64_t)problems.count, &c, r.data(), nullptr,
                                        nullptr));
  double sum = 0.0;
  for (double v : r) sum += v;
  return sum;
}

inline double run_vf_batch(const VfProblemSet& problems, const SmoothingConfig& cfg, int workers = 1,
                           std::vector<double>* out = nullptr) {
  (void)workers;
  std::vector<double> local;
  std::vector<double>& r = out ? *out : local;
  r.assign(3 * problems.count, 0.0);
  const cmgb_config c = cfg.to_c();
  detail::ok(cmgb_vf_witness_batch_host(problems.data.data(), (int64_t)problems.count, &c, r.data(), nullptr,
                                        nullptr));
  double sum = 0.0;
  for (double v : r) sum += v;
  return sum;
}

struct TimingStats {
  double median_s = 0.0;
  double std_s = 0.0;
};

// Median and population std of `repetitions` timed calls after `warmups`
// untimed ones (batch.cpp:100-120).
inline TimingStats time_run(const std::function<void()>& fn, int repetitions, int warmups) {
  if (repetitions < 1) throw std::invalid_argument("time_run: repetitions >= 1");
  for (int i = 0; i < warmups; ++i) fn();
  std::vector<double> t((size_t)repetitions);
  for (auto& x : t) {
    const auto a = std::chrono::steady_clock::now();
    fn();
    x = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
  }
  std::sort(t.begin(), t.end());
  TimingStats st;
  st.median_s = t[t.size() / 2];
  double mean = 0.0, var = 0.0;
  for (double x : t) mean += x;
  mean /= (double)t.size();
  for (double x : t) var += (x - mean) * (x - mean);
  st.std_s = std::sqrt(var / (double)t.size());
  return st;
}

struct BenchRecord {
  std::string kind;
  std::string variant;
  size_t batch = 0;
  int repetitions = 0;
  TimingStats timing;
  double throughput_qps = 0.0;
};

inline constexpr const char* kBenchCsvVersion = "cmg-bench-csv v1";

inline void write_bench_csv(std::ostream& os, const std::vector<BenchRecord>& records) {
  os << "# " << kBenchCsvVersion << "\n";
  os << "kind,variant,batch,repetitions,median_s,std_s,throughput_qps\n";
  for (const auto& r : records)
    os << r.kind << ',' << r.variant << ',' << r.batch << ',' << r.repetitions << ',' << r.timing.median_s << ','
       << r.timing.std_s << ',' << r.throughput_qps << '\n';
}

inline std::vector<BenchRecord> bench_witness(const std::string& kind, const std::vector<size_t>& batch_sizes,
                                              const std::vector<std::string>& variants, uint64_t seed,
                                              int repetitions, int workers) {
  if (kind != "ee" && kind != "vf") throw std::invalid_argument("bench kind must be ee or vf");
  std::vector<BenchRecord> records;
  for (size_t batch : batch_sizes) {
    const EeProblemSet ee = kind == "ee" ? make_random_ee_pairs(batch, seed) : EeProblemSet{};
    const VfProblemSet vf = kind == "vf" ? make_random_vf_pairs(batch, seed) : VfProblemSet{};
    for (const auto& variant : variants) {
      const SmoothingConfig cfg = config_for_variant(variant, SmoothingConfig{});
      volatile double sink = 0.0;
      BenchRecord rec;
      rec.timing = time_run(
          [&] { sink = kind == "ee" ? run_ee_batch(ee, cfg, workers) : run_vf_batch(vf, cfg, workers); },
          repetitions, 3);
      (void)sink;
      rec.kind = kind;
      rec.variant = variant;
      rec.batch = batch;
      rec.repetitions = repetitions;
      rec.throughput_qps = (double)batch / std::max(rec.timing.median_s, 1e-12);
      records.push_back(rec);
    }
  }
  return records;
}

// bench_manifold (batch.cpp:184-228): the same pose jitter stream, one batched
// GPU call per repetition (host poses in, per-env mean contact distance out:
// the reference's sums[i]).
inline std::vector<BenchRecord> bench_manifold(const Scene& scene, const std::vector<size_t>& batch_sizes,
                                               const std::vector<std::string>& variants, uint64_t seed,
                                               int repetitions, int workers) {
  (void)workers;
  if (scene.bodies.size() < 2) throw std::invalid_argument("manifold benchmark needs a two-body scene");
  const SurfaceModel& s1 = scene.bodies[0].surface;
  const SurfaceModel& s2 = scene.bodies[1].surface;
  std::vector<BenchRecord> records;
  for (size_t batch : batch_sizes) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> jitter(-0.05, 0.05);
    std::vector<double> p1(scene.bodies[0].pose.begin(), scene.bodies[0].pose.end()), p2(6 * batch);
    for (size_t i = 0; i < batch; ++i)
      for (int k = 0; k < 6; ++k) p2[6 * i + k] = scene.bodies[1].pose[k] + jitter(rng);
    for (const auto& variant : variants) {
      const cmgb_config c = config_for_variant(variant, scene.smoothing).to_c();
      std::vector<float> sums(batch);
      BenchRecord rec;
      rec.timing = time_run(
          [&] {
            if (batch)
              detail::ok(cmgb_manifold_batch_host(s1.handle(), s2.handle(), p1.data(), batch > 1 ? 0 : 1, p2.data(),
                                                  1, (int64_t)batch, &c, sums.data(), nullptr, nullptr));
          },
          repetitions, std::min(3, repetitions));
      rec.kind = "manifold";
      rec.variant = variant;
      rec.batch = batch;
      rec.repetitions = repetitions;
      rec.throughput_qps = (double)batch / std::max(rec.timing.median_s, 1e-12);
      records.push_back(rec);
    }
  }
  return records;
}

// ============================================================================ scene documents (scene.hpp)
// parse_scene / load_scene (src/scene.cpp:130-182): the same schema, defaults
// and messages, on cmgb_json.hpp (the reference uses nlohmann::json).
namespace detail {

inline Vec3d scene_vec3(const json::Value& j, const char* what) {
  if (!j.is_array() || j.size() != 3) throw SceneError(std::string(what) + ": expected [x, y, z]");
  return {j[0].as_number(), j[1].as_number(), j[2].as_number()};
}

inline Pose6d scene_pose(const json::Value& j, const char* what) {
  if (!j.is_array() || j.size() != 6)
    throw SceneError(std::string(what) + ": expected a 6-vector [tx, ty, tz, rx, ry, rz]");
  Pose6d p;
  for (int i = 0; i < 6; ++i) p[i] = j[i].as_number();
  return p;
}

inline SmoothSdf scene_sdf_node(const json::Value& j, const SmoothingConfig& defaults);

inline SmoothSdf scene_sdf_primitive(const json::Value& j, const SmoothingConfig& defaults) {
  const std::string type = j.at("type").as_string();
  if (type == "superquadric") {
    SuperquadricParams q;
    q.eps1 = j.at("eps1").as_number();
    q.eps2 = j.at("eps2").as_number();
    q.axes = scene_vec3(j.at("axes"), "superquadric axes");
    if (j.contains("pose")) q.pose = scene_pose(j.at("pose"), "superquadric pose");
    return SmoothSdf::superquadric(q);
  }
  if (type == "convex_polyhedron" || type == "box_planes") {
    ConvexPolyhedronParams cp;
    cp.tau = j.value("tau", 1e-3);
    if (type == "convex_polyhedron") {
      for (const auto& plane : j.at("planes").arr) {
        cp.normals.push_back(scene_vec3(plane.at("normal"), "plane normal"));
        cp.points.push_back(scene_vec3(plane.at("point"), "plane point"));
      }
    } else {  // the six half-space planes of an axis-aligned box: +x, -x, +y, -y, +z, -z
      const Vec3d h = scene_vec3(j.at("half_extents"), "box_planes half_extents");
      for (int a = 0; a < 3; ++a)
        for (double sg : {1.0, -1.0}) {
          Vec3d n{0, 0, 0}, pt{0, 0, 0};
          n[a] = sg;
          pt[a] = sg * h[a];
          cp.normals.push_back(n);
          cp.points.push_back(pt);
        }
    }
    return SmoothSdf::convex_polyhedron(cp);
  }
  if (type == "oriented_pointcloud") {
    OrientedPointcloudParams pc;
    for (const auto& x : j.at("points").arr) pc.points.push_back(scene_vec3(x, "pointcloud point"));
    for (const auto& x : j.at("normals").arr) pc.normals.push_back(scene_vec3(x, "pointcloud normal"));
    for (const auto& x : j.at("lengthscales").arr) pc.lengthscales.push_back(x.as_number());
    return SmoothSdf::oriented_pointcloud(pc);
  }
  if (type == "union") {
    std::vector<SmoothSdf> children;
    for (const auto& c : j.at("children").arr) children.push_back(scene_sdf_node(c, defaults));
    return SmoothSdf::smooth_union(std::move(children), j.value("tau", defaults.tau_union));
  }
  if (type == "subtraction")
    return SmoothSdf::subtraction(scene_sdf_node(j.at("positive"), defaults),
                                  scene_sdf_node(j.at("negative"), defaults), j.value("tau", defaults.tau_union));
  throw SceneError("unknown sdf node type: " + type);
}

inline SmoothSdf scene_sdf_node(const json::Value& j, const SmoothingConfig& defaults) {
  if (j.is_array()) {  // array shorthand: implicit union, a single child collapses
    std::vector<SmoothSdf> children;
    for (const auto& c : j.arr) children.push_back(scene_sdf_node(c, defaults));
    if (children.size() == 1) return std::move(children.front());
    return SmoothSdf::smooth_union(std::move(children), defaults.tau_union);
  }
  return scene_sdf_primitive(j, defaults);
}

inline CollisionMesh scene_mesh(const json::Value& j, const std::string& base_dir) {
  if (j.contains("obj")) {
    std::filesystem::path p = j.at("obj").as_string();
    if (p.is_relative()) p = std::filesystem::path(base_dir) / p;
    return load_obj(p.string());
  }
  if (j.contains("box")) {
    const json::Value& b = j.at("box");
    return make_box_mesh(scene_vec3(b.at("half_extents"), "box half_extents"), b.value("subdivisions", 1),
                         b.value("quad_edges", true));
  }
  throw SceneError("mesh: expected an 'obj' path or a 'box' generator");
}

inline SmoothingConfig scene_smoothing(const json::Value& j) {
  SmoothingConfig c;
  if (!j.is_object()) return c;
  c.lambda = j.value("lambda", c.lambda);
  c.tau_clip = j.value("tau_clip", c.tau_clip);
  c.tau_min = j.value("tau_min", c.tau_min);
  c.tau_comp = j.value("tau_comp", c.tau_comp);
  c.tau_sign = j.value("tau_sign", c.tau_sign);
  c.tau_pen = j.value("tau_pen", c.tau_pen);
  c.tau_nn = j.value("tau_nn", c.tau_nn);
  c.tau_clash = j.value("tau_clash", c.tau_clash);
  c.tau_cont = j.value("tau_cont", c.tau_cont);
  c.tau_topk_verts = j.value("tau_topk_verts", c.tau_topk_verts);
  c.tau_topk_edges = j.value("tau_topk_edges", c.tau_topk_edges);
  c.tau_normal = j.value("tau_normal", c.tau_normal);
  c.tau_union = j.value("tau_union", c.tau_union);
  c.hard_ops = j.value("hard_ops", c.hard_ops);
  c.sphere_trace = j.value("sphere_trace", c.sphere_trace);
  c.sphere_trace_iters = j.value("sphere_trace_iters", c.sphere_trace_iters);
  c.containment_safeguard = j.value("containment_safeguard", c.containment_safeguard);
  if (j.contains("mode")) {
    const std::string m = j.at("mode").as_string();
    if (m == "full") c.mode = ContactMode::kFull;
    else if (m == "no-ee") c.mode = ContactMode::kNoEe;
    else if (m == "one-sided") c.mode = ContactMode::kOneSided;
    else throw SceneError("mode must be one of: full, no-ee, one-sided");
  }
  c.validate();
  return c;
}

}  // namespace detail

inline Scene parse_scene(const std::string& json_text, const std::string& base_dir) {
  json::Value doc;
  try {
    doc = json::parse(json_text);
  } catch (const json::ParseError& e) {
    throw SceneError(std::string("scene JSON parse error: ") + e.what());
  }
  Scene scene;
  try {
    scene.smoothing = detail::scene_smoothing(doc.contains("smoothing") ? doc.at("smoothing") : json::Value());
    if (!doc.contains("bodies") || !doc.at("bodies").is_array() || doc.at("bodies").size() == 0)
      throw SceneError("scene: needs a non-empty 'bodies' array");
    for (const auto& jb : doc.at("bodies").arr) {
      SceneBody body;
      body.name = jb.value("name", std::string("body") + std::to_string(scene.bodies.size()));
      CollisionMesh mesh = detail::scene_mesh(jb.at("mesh"), base_dir);
      SmoothSdf sdf = detail::scene_sdf_node(jb.at("sdf"), scene.smoothing);
      body.surface = build_surface(std::move(mesh), std::move(sdf), jb.value("vertex_topk", 0),
                                   jb.value("edge_topk", 0));
      body.pose = detail::scene_pose(jb.at("pose"), "body pose");
      body.mass = jb.value("mass", 1.0);
      if (!(body.mass > 0.0)) throw SceneError("body mass must be positive");
      if (jb.contains("inertia")) body.inertia_diag = detail::scene_vec3(jb.at("inertia"), "inertia");
      body.is_static = jb.value("static", false);
      scene.bodies.push_back(std::move(body));
    }
  } catch (const json::KeyError& e) {  // the reference catches json::exception here
    throw SceneError(std::string("scene schema error: ") + e.what());
  } catch (const json::TypeError& e) {
    throw SceneError(std::string("scene schema error: ") + e.what());
  }
  return scene;
}

inline Scene load_scene(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw SceneError("cannot open scene file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return parse_scene(ss.str(), std::filesystem::path(path).parent_path().string());
}

// ============================================================================ writers (manifold_io.hpp)
namespace detail {
inline const char* kind_name(ContactKind k) { return k == ContactKind::kVertexSdf ? "VS" : "EE"; }
inline const char* mode_name(ContactMode m) {
  return m == ContactMode::kNoEe ? "no-ee" : (m == ContactMode::kOneSided ? "one-sided" : "full");
}
}  // namespace detail

// CSV schema v1 (src/manifold_io.cpp:24-33).
inline void write_manifold_csv(std::ostream& os, const ContactManifold<double>& m) {
  os << "index,kind,side,src_a,src_b,px,py,pz,dist,nx,ny,nz,activity\n";
  const auto prec = os.precision(17);
  for (size_t i = 0; i < m.contacts.size(); ++i) {
    const auto& c = m.contacts[i];
    os << i << ',' << detail::kind_name(c.kind) << ',' << c.side << ',' << c.src_a << ',' << c.src_b << ','
       << c.point.x << ',' << c.point.y << ',' << c.point.z << ',' << c.dist << ',' << c.normal.x << ','
       << c.normal.y << ',' << c.normal.z << ',' << c.activity << '\n';
  }
  os.precision(prec);
}

// JSON mirror of the same records plus the layout (src/manifold_io.cpp:35-52).
inline std::string manifold_to_json(const ContactManifold<double>& m) {
  using json::Value;
  Value j = Value::object(), layout = Value::object(), rows = Value::array();
  layout.obj["n1"] = Value::integer(m.n1);
  layout.obj["n2"] = Value::integer(m.n2);
  layout.obj["m1"] = Value::integer(m.m1);
  layout.obj["m2"] = Value::integer(m.m2);
  layout.obj["mode"] = Value::string(detail::mode_name(m.mode));
  auto vec = [](const Vec3d& v) {
    Value a = Value::array();
    for (int k = 0; k < 3; ++k) a.arr.push_back(Value::number(v[k]));
    return a;
  };
  for (const auto& c : m.contacts) {
    Value r = Value::object();
    r.obj["kind"] = Value::string(detail::kind_name(c.kind));
    r.obj["side"] = Value::integer(c.side);
    r.obj["src_a"] = Value::integer(c.src_a);
    r.obj["src_b"] = Value::integer(c.src_b);
    r.obj["point"] = vec(c.point);
    r.obj["dist"] = Value::number(c.dist);
    r.obj["normal"] = vec(c.normal);
    r.obj["activity"] = Value::number(c.activity);
    rows.arr.push_back(std::move(r));
  }
  j.obj["layout"] = std::move(layout);
  j.obj["contacts"] = std::move(rows);
  return json::dump(j, 2);
}

}  // namespace ref
}  // namespace cmgb

#ifndef CMGB_NO_CMG_ALIAS
namespace cmg = cmgb::ref;
#endif
