// TEST INFRASTRUCTURE — not product code.
//
// extern "C" harness over the UNMODIFIED reference implementation
// (/root/reference/proj). It is compiled together with the reference's own
// sources by oracle/Makefile into oracle/_ref/libcmgref.so and is used only by
// tests/ (golden generation, parity checks) and by bench.py's reference /
// cpu_baseline arm. Nothing here is shipped in the product library.
//
// Every function forwards to the reference's public API:
//   build_surface            proj/src/surface.cpp:9-44
//   SmoothSdf factories      proj/src/sdf.cpp:5-50
//   make_box_mesh/parse_obj  proj/src/mesh.cpp:60-173
//   generate_manifold<T>     proj/include/cmg/manifold.hpp:336-377
//   run_ee/vf_batch          proj/src/batch.cpp:53-98
//   bench_manifold/_witness  proj/src/batch.cpp:152-228
//   ee_witness / vf_witness  proj/include/cmg/witness.hpp:137-227

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cmg/batch.hpp"
#include "cmg/demosim.hpp"
#include "cmg/manifold_io.hpp"
#include "cmg/sweep.hpp"
#include "cmg/manifold.hpp"
#include "cmg/mesh.hpp"
#include "cmg/pose.hpp"
#include "cmg/scene.hpp"
#include "cmg/sdf.hpp"
#include "cmg/smooth_ops.hpp"
#include "cmg/surface.hpp"
#include "cmg/witness.hpp"
#include "cmgb.h"

using namespace cmg;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

SmoothingConfig to_cfg(const cmgb_config* c) {
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
  s.mode = c->mode == 1 ? ContactMode::kNoEe
                        : (c->mode == 2 ? ContactMode::kOneSided : ContactMode::kFull);
  return s;
}

Vec3d v3(const double* p) { return {p[0], p[1], p[2]}; }

// Postfix program -> SmoothSdf via the reference's own factories.
SmoothSdf build_sdf(const cmgb_sdf_node* nodes, int n) {
  std::vector<SmoothSdf> stack;
  for (int i = 0; i < n; ++i) {
    const cmgb_sdf_node& nd = nodes[i];
    switch (nd.op) {
      case CMGB_SDF_SUPERQUADRIC: {
        SuperquadricParams q;
        q.eps1 = nd.eps1;
        q.eps2 = nd.eps2;
        q.axes = v3(nd.axes);
        for (int k = 0; k < 6; ++k) q.pose[k] = nd.pose[k];
        stack.push_back(SmoothSdf::superquadric(q));
        break;
      }
      case CMGB_SDF_CONVEX_POLYHEDRON: {
        ConvexPolyhedronParams cp;
        cp.tau = nd.tau;
        for (int k = 0; k < nd.count; ++k) {
          cp.normals.push_back(v3(nd.normals + 3 * k));
          cp.points.push_back(v3(nd.points + 3 * k));
        }
        stack.push_back(SmoothSdf::convex_polyhedron(cp));
        break;
      }
      case CMGB_SDF_ORIENTED_POINTCLOUD: {
        OrientedPointcloudParams pc;
        for (int k = 0; k < nd.count; ++k) {
          pc.points.push_back(v3(nd.points + 3 * k));
          pc.normals.push_back(v3(nd.normals + 3 * k));
          pc.lengthscales.push_back(nd.lengthscales[k]);
        }
        stack.push_back(SmoothSdf::oriented_pointcloud(pc));
        break;
      }
      case CMGB_SDF_UNION: {
        if (nd.count < 1 || static_cast<size_t>(nd.count) > stack.size())
          throw std::invalid_argument("harness: bad union arity");
        std::vector<SmoothSdf> ch(std::make_move_iterator(stack.end() - nd.count),
                                  std::make_move_iterator(stack.end()));
        stack.resize(stack.size() - nd.count);
        stack.push_back(SmoothSdf::smooth_union(std::move(ch), nd.tau));
        break;
      }
      case CMGB_SDF_SUBTRACTION: {
        if (stack.size() < 2) throw std::invalid_argument("harness: bad subtraction arity");
        SmoothSdf neg = std::move(stack.back());
        stack.pop_back();
        SmoothSdf pos = std::move(stack.back());
        stack.pop_back();
        stack.push_back(SmoothSdf::subtraction(std::move(pos), std::move(neg), nd.tau));
        break;
      }
      default:
        throw std::invalid_argument("harness: unknown sdf op");
    }
  }
  if (stack.size() != 1) throw std::invalid_argument("harness: program must leave one root");
  return std::move(stack.back());
}

struct MeshBox {
  CollisionMesh mesh;
};

void write_contacts(const ContactManifold<double>& m, double* contacts, int32_t* meta) {
  for (size_t i = 0; i < m.contacts.size(); ++i) {
    const auto& c = m.contacts[i];
    if (contacts) {
      double* o = contacts + 8 * i;
      o[0] = c.point.x;
      o[1] = c.point.y;
      o[2] = c.point.z;
      o[3] = c.dist;
      o[4] = c.normal.x;
      o[5] = c.normal.y;
      o[6] = c.normal.z;
      o[7] = c.activity;
    }
    if (meta) {
      int32_t* q = meta + 4 * i;
      q[0] = c.kind == ContactKind::kVertexSdf ? 0 : 1;
      q[1] = c.side;
      q[2] = c.src_a;
      q[3] = c.src_b;
    }
  }
}

void write_ee(const EeIndicatorMatrices<double>& e, double* ee) {
  if (!ee) return;
  const size_t n = e.m1 * e.m2;
  const std::vector<double>* mats[9] = {&e.dist, &e.con, &e.pen1, &e.pen2, &e.nn1,
                                        &e.nn2,  &e.clash, &e.act1, &e.act2};
  for (int f = 0; f < 9; ++f)
    for (size_t i = 0; i < n; ++i) ee[f * n + i] = (*mats[f])[i];
}

Pose6d pose6(const double* p) { return {p[0], p[1], p[2], p[3], p[4], p[5]}; }

}  // namespace

extern "C" {

const char* cmgref_last_error() { return g_err.c_str(); }

// ---- meshes ------------------------------------------------------------------
void* cmgref_mesh_box(const double* half, int subdiv, int quad) {
  try {
    auto* m = new MeshBox{make_box_mesh(v3(half), subdiv, quad != 0)};
    return m;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void* cmgref_mesh_parse_obj(const char* text, int32_t* error_line) {
  try {
    std::istringstream in(text);
    auto* m = new MeshBox{parse_obj(in)};
    return m;
  } catch (const MeshParseError& e) {
    if (error_line) *error_line = e.line_number;
    fail(e);
    return nullptr;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void* cmgref_mesh_arrays(const double* v, int nv, const int32_t* f, int nf, const int32_t* e,
                         int ne) {
  auto* m = new MeshBox;
  for (int i = 0; i < nv; ++i) m->mesh.vertices.push_back(v3(v + 3 * i));
  for (int i = 0; i < nf; ++i) m->mesh.faces.push_back({f[3 * i], f[3 * i + 1], f[3 * i + 2]});
  for (int i = 0; i < ne; ++i) m->mesh.edges.push_back({e[2 * i], e[2 * i + 1]});
  return m;
}

void cmgref_mesh_sizes(void* h, int32_t* nv, int32_t* nf, int32_t* ne, int32_t* nw) {
  auto* m = static_cast<MeshBox*>(h);
  *nv = static_cast<int32_t>(m->mesh.vertices.size());
  *nf = static_cast<int32_t>(m->mesh.faces.size());
  *ne = static_cast<int32_t>(m->mesh.edges.size());
  *nw = static_cast<int32_t>(m->mesh.warnings.size());
}

void cmgref_mesh_read(void* h, double* v, int32_t* f, int32_t* e) {
  auto* m = static_cast<MeshBox*>(h);
  for (size_t i = 0; i < m->mesh.vertices.size(); ++i) {
    v[3 * i] = m->mesh.vertices[i].x;
    v[3 * i + 1] = m->mesh.vertices[i].y;
    v[3 * i + 2] = m->mesh.vertices[i].z;
  }
  for (size_t i = 0; i < m->mesh.faces.size(); ++i)
    for (int k = 0; k < 3; ++k) f[3 * i + k] = m->mesh.faces[i][k];
  for (size_t i = 0; i < m->mesh.edges.size(); ++i)
    for (int k = 0; k < 2; ++k) e[2 * i + k] = m->mesh.edges[i][k];
}

const char* cmgref_mesh_warning(void* h, int i) {
  return static_cast<MeshBox*>(h)->mesh.warnings[i].c_str();
}

void cmgref_mesh_destroy(void* h) { delete static_cast<MeshBox*>(h); }

// ---- surfaces ----------------------------------------------------------------
void* cmgref_surface_create(void* mesh, const cmgb_sdf_node* nodes, int n_nodes, int vtopk,
                            int etopk, double tol) {
  try {
    CollisionMesh m = static_cast<MeshBox*>(mesh)->mesh;
    auto* s = new SurfaceModel(build_surface(std::move(m), build_sdf(nodes, n_nodes), vtopk,
                                             etopk, tol));
    return s;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void cmgref_surface_destroy(void* s) { delete static_cast<SurfaceModel*>(s); }

int cmgref_surface_info(void* h, int32_t* out /* V, E, leaves, eff_v, eff_e, n_warn */) {
  auto* s = static_cast<SurfaceModel*>(h);
  out[0] = static_cast<int32_t>(s->mesh.vertices.size());
  out[1] = static_cast<int32_t>(s->mesh.edges.size());
  out[2] = static_cast<int32_t>(s->sdf.leaf_count());
  out[3] = s->effective_vertex_topk();
  out[4] = s->effective_edge_topk();
  out[5] = static_cast<int32_t>(s->build_warnings.size());
  return 0;
}

const char* cmgref_surface_warning(void* h, int i) {
  return static_cast<SurfaceModel*>(h)->build_warnings[i].c_str();
}

// SDF queries in the BODY frame: flavor 0 = value, 1 = value_and_gradient,
// 2 = value_and_normal_source. out: n x 4 (value, gx, gy, gz).
void cmgref_sdf_query(void* h, int flavor, const double* p, int64_t n, double* out) {
  auto* s = static_cast<SurfaceModel*>(h);
  for (int64_t i = 0; i < n; ++i) {
    const Vec3d q = v3(p + 3 * i);
    double* o = out + 4 * i;
    if (flavor == 0) {
      o[0] = s->sdf.value(q);
      o[1] = o[2] = o[3] = 0.0;
    } else {
      const SdfSample<double> r =
          flavor == 1 ? s->sdf.value_and_gradient(q) : s->sdf.value_and_normal_source(q);
      o[0] = r.value;
      o[1] = r.grad.x;
      o[2] = r.grad.y;
      o[3] = r.grad.z;
    }
  }
}

// Sphere tracing of world points against the posed SDF (sdf.hpp:318-326).
void cmgref_sphere_trace(void* h, const double* pose, const double* p, int64_t n, int iters,
                         double tau, double* out) {
  auto* s = static_cast<SurfaceModel*>(h);
  PosedSdf<double> posed{&s->sdf, se3_exp(pose6(pose))};
  for (int64_t i = 0; i < n; ++i) {
    const Vec3d r = sphere_trace_project(posed, v3(p + 3 * i), iters, tau);
    out[3 * i] = r.x;
    out[3 * i + 1] = r.y;
    out[3 * i + 2] = r.z;
  }
}

// ---- manifold ------------------------------------------------------------------
// layout out: n1, n2, m1, m2, n_contacts.
int cmgref_manifold(void* h1, void* h2, const double* pose1, const double* pose2,
                    const cmgb_config* c, double* contacts, int32_t* meta, double* ee,
                    int32_t* layout) {
  try {
    const auto m = generate_manifold(*static_cast<SurfaceModel*>(h1),
                                     *static_cast<SurfaceModel*>(h2), pose6(pose1), pose6(pose2),
                                     to_cfg(c));
    if (layout) {
      layout[0] = m.n1;
      layout[1] = m.n2;
      layout[2] = m.m1;
      layout[3] = m.m2;
      layout[4] = static_cast<int32_t>(m.contacts.size());
    }
    write_contacts(m, contacts, meta);
    write_ee(m.ee, ee);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Batch of envs with per-env poses (pose1_stride 0 = shared body-1 pose),
// parallel over `workers` std::threads like parallel_for (batch.cpp:27-41).
int cmgref_manifold_batch(void* h1, void* h2, const double* poses1, int pose1_stride,
                          const double* poses2, int pose2_stride, int64_t n,
                          const cmgb_config* c, int workers, double* contacts, int32_t* meta,
                          double* mean_dist) {
  try {
    const SurfaceModel& s1 = *static_cast<SurfaceModel*>(h1);
    const SurfaceModel& s2 = *static_cast<SurfaceModel*>(h2);
    const SmoothingConfig cfg = to_cfg(c);
    size_t per_env = 0;
    {
      const auto m0 = generate_manifold(s1, s2, pose6(poses1), pose6(poses2), cfg);
      per_env = m0.contacts.size();
    }
    auto body = [&](int64_t lo, int64_t hi) {
      for (int64_t i = lo; i < hi; ++i) {
        const auto m = generate_manifold(s1, s2, pose6(poses1 + 6 * i * pose1_stride),
                                         pose6(poses2 + 6 * i * pose2_stride), cfg);
        write_contacts(m, contacts ? contacts + 8 * per_env * i : nullptr,
                       meta ? meta + 4 * per_env * i : nullptr);
        if (mean_dist) mean_dist[i] = mean_contact_distance(m);
      }
    };
    workers = std::max(1, workers);
    if (workers == 1 || n < 64) {
      body(0, n);
    } else {
      std::vector<std::thread> pool;
      const int64_t chunk = (n + workers - 1) / workers;
      for (int w = 0; w < workers; ++w) {
        const int64_t lo = std::min<int64_t>(n, w * chunk);
        const int64_t hi = std::min<int64_t>(n, lo + chunk);
        if (lo < hi) pool.emplace_back(body, lo, hi);
      }
      for (auto& t : pool) t.join();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Forward-mode pose Jacobian of every contact field (Dual12, dual.hpp:249-262).
// tangents: n_contacts x 8 x 12; contacts: n_contacts x 8 (primal).
int cmgref_manifold_jvp(void* h1, void* h2, const double* pose1, const double* pose2,
                        const cmgb_config* c, double* contacts, double* tangents,
                        double* mean_dist_grad /* 13: value + 12 */) {
  try {
    const auto seeded = seed_pose_tangents(
        std::array<double, 6>{pose1[0], pose1[1], pose1[2], pose1[3], pose1[4], pose1[5]},
        std::array<double, 6>{pose2[0], pose2[1], pose2[2], pose2[3], pose2[4], pose2[5]});
    const auto m = generate_manifold(*static_cast<SurfaceModel*>(h1),
                                     *static_cast<SurfaceModel*>(h2), seeded.first,
                                     seeded.second, to_cfg(c));
    for (size_t i = 0; i < m.contacts.size(); ++i) {
      const auto& ct = m.contacts[i];
      const Dual12* f[8] = {&ct.point.x, &ct.point.y, &ct.point.z, &ct.dist,
                            &ct.normal.x, &ct.normal.y, &ct.normal.z, &ct.activity};
      for (int k = 0; k < 8; ++k) {
        if (contacts) contacts[8 * i + k] = f[k]->v;
        if (tangents)
          for (int d = 0; d < 12; ++d) tangents[(8 * i + k) * 12 + d] = f[k]->d[d];
      }
    }
    if (mean_dist_grad) {
      const Dual12 md = mean_contact_distance(m);
      mean_dist_grad[0] = md.v;
      for (int d = 0; d < 12; ++d) mean_dist_grad[1 + d] = md.d[d];
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- witness -----------------------------------------------------------------------
void cmgref_random_pairs(int64_t n, uint64_t seed, double* out) {
  const EeProblemSet p = make_random_ee_pairs(static_cast<size_t>(n), seed);
  std::memcpy(out, p.data.data(), sizeof(double) * 12 * n);
}

double cmgref_ee_batch(const double* pairs, int64_t n, const cmgb_config* c, int workers,
                       double* out) {
  EeProblemSet p{static_cast<size_t>(n), std::vector<double>(pairs, pairs + 12 * n)};
  std::vector<double> res;
  const double cs = run_ee_batch(p, to_cfg(c), workers, &res);
  if (out) std::memcpy(out, res.data(), sizeof(double) * res.size());
  return cs;
}

double cmgref_vf_batch(const double* pairs, int64_t n, const cmgb_config* c, int workers,
                       double* out) {
  VfProblemSet p{static_cast<size_t>(n), std::vector<double>(pairs, pairs + 12 * n)};
  std::vector<double> res;
  const double cs = run_vf_batch(p, to_cfg(c), workers, &res);
  if (out) std::memcpy(out, res.data(), sizeof(double) * res.size());
  return cs;
}

// Full E-E witness result: p1, p2, alpha1, alpha2, gamma_con (9 per pair).
void cmgref_ee_witness_full(const double* pairs, int64_t n, const cmgb_config* c, double* out) {
  const SmoothingConfig cfg = to_cfg(c);
  for (int64_t i = 0; i < n; ++i) {
    const double* p = pairs + 12 * i;
    const auto w = ee_witness<double>(v3(p), v3(p + 3), v3(p + 6), v3(p + 9), cfg);
    double* o = out + 9 * i;
    o[0] = w.p1.x;
    o[1] = w.p1.y;
    o[2] = w.p1.z;
    o[3] = w.p2.x;
    o[4] = w.p2.y;
    o[5] = w.p2.z;
    o[6] = w.alpha[0];
    o[7] = w.alpha[1];
    o[8] = w.gamma_con;
  }
}

// solve_box_qp_2 on raw QPs: in n x 5 (q11, q12, q22, c1, c2), out n x 3.
void cmgref_box_qp(const double* qp, int64_t n, const cmgb_config* c, double* out) {
  const SmoothingConfig cfg = to_cfg(c);
  for (int64_t i = 0; i < n; ++i) {
    BoxQp2<double> q{qp[5 * i], qp[5 * i + 1], qp[5 * i + 2], qp[5 * i + 3], qp[5 * i + 4]};
    const auto s = solve_box_qp_2(q, cfg);
    out[3 * i] = s.alpha[0];
    out[3 * i + 1] = s.alpha[1];
    out[3 * i + 2] = s.gamma_con;
  }
}

// ---- timing (the reference's own harness) ------------------------------------------
int cmgref_bench_manifold(void* h1, void* h2, const double* pose1, const double* pose2,
                          const cmgb_config* base, int64_t batch, const char* variant,
                          uint64_t seed, int reps, int workers, double* median_s,
                          double* std_s) {
  try {
    Scene scene;
    scene.smoothing = to_cfg(base);
    SceneBody b1, b2;
    b1.surface = *static_cast<SurfaceModel*>(h1);
    b2.surface = *static_cast<SurfaceModel*>(h2);
    b1.pose = pose6(pose1);
    b2.pose = pose6(pose2);
    scene.bodies.push_back(std::move(b1));
    scene.bodies.push_back(std::move(b2));
    const auto rec = bench_manifold(scene, {static_cast<size_t>(batch)}, {variant}, seed, reps,
                                    workers);
    *median_s = rec[0].timing.median_s;
    *std_s = rec[0].timing.std_s;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int cmgref_bench_witness(const char* kind, int64_t batch, const char* variant, uint64_t seed,
                         int reps, int workers, double* median_s, double* std_s) {
  try {
    const auto rec =
        bench_witness(kind, {static_cast<size_t>(batch)}, {variant}, seed, reps, workers);
    *median_s = rec[0].timing.median_s;
    *std_s = rec[0].timing.std_s;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- misc reference helpers ------------------------------------------------------------
void cmgref_se3_exp(const double* pose, double* R, double* t) {
  const Transformd tf = se3_exp(pose6(pose));
  for (int i = 0; i < 9; ++i) R[i] = tf.R.m[i];
  t[0] = tf.t.x;
  t[1] = tf.t.y;
  t[2] = tf.t.z;
}

void cmgref_so3_log(const double* R, double* w) {
  Mat3d m;
  for (int i = 0; i < 9; ++i) m.m[i] = R[i];
  const Vec3d r = so3_log(m);
  w[0] = r.x;
  w[1] = r.y;
  w[2] = r.z;
}

void cmgref_so3_exp(const double* w, double* R) {
  const Mat3d m = so3_exp_d(v3(w));
  for (int i = 0; i < 9; ++i) R[i] = m.m[i];
}

// soft_topk (smooth_ops.hpp:173-198): w out K x D.
int cmgref_soft_topk(const double* xs, int d, int k, double tau, double* w) {
  try {
    const auto sel = soft_topk(std::vector<double>(xs, xs + d), k, tau);
    std::memcpy(w, sel.w.data(), sizeof(double) * k * d);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int cmgref_config_validate(const cmgb_config* c) {
  try {
    to_cfg(c).validate();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// DemoSim (src/demosim.cpp:68-138) over a programmatic Scene (no JSON): runs
// `steps` steps of dt from the given state, recording after every step the
// poses / velocities [steps][n][6], deepest_penetration() and kinetic energy.
// Returns the number of steps that succeeded (step() == true).
int cmgref_demo_run(void* const* surfaces, int n, const int32_t* is_static, const double* mass,
                    const double* inertia, const double* poses, const double* vels, const cmgb_config* c,
                    const cmgb_demo_params* pp, double dt, int steps, double* poses_out, double* vels_out,
                    double* deepest_out, double* ke_out) {
  try {
    Scene scene;
    scene.smoothing = to_cfg(c);
    for (int i = 0; i < n; ++i) {
      SceneBody b;
      b.name = "b" + std::to_string(i);
      b.surface = *static_cast<SurfaceModel*>(surfaces[i]);
      for (int k = 0; k < 6; ++k) b.pose[k] = poses[6 * i + k];
      b.mass = mass[i];
      b.inertia_diag = Vec3d{inertia[3 * i], inertia[3 * i + 1], inertia[3 * i + 2]};
      b.is_static = is_static[i] != 0;
      scene.bodies.push_back(std::move(b));
    }
    PenaltyParams params;
    params.stiffness = pp->stiffness;
    params.damping = pp->damping;
    params.friction = pp->friction;
    params.friction_viscous = pp->friction_viscous;
    params.tau_force = pp->tau_force;
    params.gravity = Vec3d{pp->gravity[0], pp->gravity[1], pp->gravity[2]};
    DemoSim sim(scene, params);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < 6; ++k) sim.states()[i].velocity[k] = vels[6 * i + k];
    int done = 0;
    for (int s = 0; s < steps; ++s) {
      if (!sim.step(dt)) break;
      ++done;
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < 6; ++k) {
          poses_out[(s * n + i) * 6 + k] = sim.states()[i].pose[k];
          vels_out[(s * n + i) * 6 + k] = sim.states()[i].velocity[k];
        }
      if (deepest_out) deepest_out[s] = sim.deepest_penetration();
      if (ke_out) ke_out[s] = sim.kinetic_energy();
    }
    return done;
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

// PenaltyParams{} defaults (include/cmg/demosim.hpp:24-31).
void cmgref_demo_params_default(cmgb_demo_params* p) {
  const PenaltyParams d;
  p->stiffness = d.stiffness;
  p->damping = d.damping;
  p->friction = d.friction;
  p->friction_viscous = d.friction_viscous;
  p->tau_force = d.tau_force;
  p->gravity[0] = d.gravity.x;
  p->gravity[1] = d.gravity.y;
  p->gravity[2] = d.gravity.z;
}

// ---- sweep / scene / writers (src/sweep.cpp, src/scene.cpp, src/manifold_io.cpp) ----
// rotating_edge_sweep: out [n][7] = theta, p1, dp1/dtheta.
int cmgref_sweep(int variant, int n, double* out) {
  try {
    const auto v = variant == 0 ? SweepVariant::kNoSmoothing
                                : (variant == 1 ? SweepVariant::kRegularizedOnly : SweepVariant::kSmooth);
    const auto s = rotating_edge_sweep(v, n);
    for (int i = 0; i < n; ++i) {
      const double row[7] = {s[i].theta, s[i].p1.x, s[i].p1.y, s[i].p1.z,
                             s[i].dp1_dtheta.x, s[i].dp1_dtheta.y, s[i].dp1_dtheta.z};
      std::memcpy(out + 7 * i, row, sizeof(row));
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// write_sweep_csv of the three variants (the CLI's sweep-edges output).
int cmgref_sweep_csv(int n, char* buf, int64_t cap, int64_t* len) {
  try {
    std::ostringstream os;
    write_sweep_csv(os, rotating_edge_sweep(SweepVariant::kNoSmoothing, n),
                    rotating_edge_sweep(SweepVariant::kRegularizedOnly, n),
                    rotating_edge_sweep(SweepVariant::kSmooth, n));
    const std::string t = os.str();
    *len = (int64_t)t.size();
    if (buf && cap > (int64_t)t.size()) std::memcpy(buf, t.c_str(), t.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// parse_scene: a heap Scene, queried below.
void* cmgref_scene_parse(const char* json_text, const char* base_dir) {
  try {
    return new Scene(parse_scene(json_text, base_dir));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void cmgref_scene_destroy(void* s) { delete static_cast<Scene*>(s); }
int cmgref_scene_n_bodies(void* s) { return (int)static_cast<Scene*>(s)->bodies.size(); }
// body i: pose[6], mass, inertia[3], static, vertex/edge topk; surface handle (owned by the scene)
void* cmgref_scene_body(void* s, int i, double* pose, double* mass, double* inertia, int32_t* is_static,
                        int32_t* topk, char* name, int cap) {
  auto& b = static_cast<Scene*>(s)->bodies[i];
  for (int k = 0; k < 6; ++k) pose[k] = b.pose[k];
  *mass = b.mass;
  inertia[0] = b.inertia_diag.x;
  inertia[1] = b.inertia_diag.y;
  inertia[2] = b.inertia_diag.z;
  *is_static = b.is_static ? 1 : 0;
  topk[0] = b.surface.vertex_topk;
  topk[1] = b.surface.edge_topk;
  std::snprintf(name, cap, "%s", b.name.c_str());
  return &b.surface;
}
void cmgref_scene_smoothing(void* s, cmgb_config* out) {
  const SmoothingConfig& c = static_cast<Scene*>(s)->smoothing;
  out->lambda = c.lambda;
  out->tau_clip = c.tau_clip;
  out->tau_min = c.tau_min;
  out->tau_comp = c.tau_comp;
  out->tau_sign = c.tau_sign;
  out->tau_pen = c.tau_pen;
  out->tau_nn = c.tau_nn;
  out->tau_clash = c.tau_clash;
  out->tau_cont = c.tau_cont;
  out->tau_topk_verts = c.tau_topk_verts;
  out->tau_topk_edges = c.tau_topk_edges;
  out->tau_normal = c.tau_normal;
  out->tau_union = c.tau_union;
  out->hard_ops = c.hard_ops;
  out->sphere_trace = c.sphere_trace;
  out->sphere_trace_iters = c.sphere_trace_iters;
  out->containment_safeguard = c.containment_safeguard;
  out->mode = (int32_t)c.mode;
  out->reserved = 0;
}

// write_manifold_csv / manifold_to_json of one generate_manifold<double>.
int cmgref_manifold_text(void* h1, void* h2, const double* pose1, const double* pose2, const cmgb_config* c,
                         int as_json, char* buf, int64_t cap, int64_t* len) {
  try {
    const auto m = generate_manifold(*static_cast<SurfaceModel*>(h1), *static_cast<SurfaceModel*>(h2),
                                     pose6(pose1), pose6(pose2), to_cfg(c));
    std::string t;
    if (as_json) {
      t = manifold_to_json(m) + "\n";
    } else {
      std::ostringstream os;
      write_manifold_csv(os, m);
      t = os.str();
    }
    *len = (int64_t)t.size();
    if (buf && cap > (int64_t)t.size()) std::memcpy(buf, t.c_str(), t.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
