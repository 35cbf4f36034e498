/*
 * TEST INFRASTRUCTURE — CPU oracle (plain C, double precision) for the
 * batched contact-manifold path of arXiv 2602.20304. See cmg_oracle.h.
 *
 * Each function restates the reference algorithm and cites the file:line it
 * follows (paths relative to /root/reference/proj). Spatial gradients that the
 * reference obtains with a nested Dual<3> (sdf.hpp:183-190, 233-288) are
 * written out analytically here; the golden tests pin both routes to each
 * other. This file is the checker: the product (paper_2602_20304_b200/) never
 * links or calls it.
 */
#define _POSIX_C_SOURCE 200809L
#include "cmg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* small vector helpers (include/cmg/vec3.hpp:13-140)                         */
/* ------------------------------------------------------------------------- */
typedef struct { double x, y, z; } v3;

static v3 mk(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 scl(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 cross(v3 a, v3 b) {
  return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double nsq(v3 a) { return dot(a, a); }
static v3 ld3(const double* p) { return mk(p[0], p[1], p[2]); }
/* Mat3 row-major: R*v (vec3.hpp:88-92) and R^T v (vec3.hpp:125-130). */
static v3 mv(const double* R, v3 v) {
  return mk(R[0] * v.x + R[1] * v.y + R[2] * v.z, R[3] * v.x + R[4] * v.y + R[5] * v.z,
            R[6] * v.x + R[7] * v.y + R[8] * v.z);
}
static v3 mtv(const double* R, v3 v) {
  return mk(R[0] * v.x + R[3] * v.y + R[6] * v.z, R[1] * v.x + R[4] * v.y + R[7] * v.z,
            R[2] * v.x + R[5] * v.y + R[8] * v.z);
}
/* normalize_smooth: v / sqrt(tau + |v|^2) (vec3.hpp:56-62). */
static v3 normalize_smooth(v3 v, double tau) { return scl(v, 1.0 / sqrt(tau + nsq(v))); }

/* ------------------------------------------------------------------------- */
/* smooth operators (include/cmg/smooth_ops.hpp)                              */
/* ------------------------------------------------------------------------- */
/* stable_sigmoid (smooth_ops.hpp:22-35) */
static double stable_sigmoid(double x) {
  if (!(x < 0.0)) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}
/* sigma_greater (38-42) */
static double sigma_greater(double x, double a, double tau) { return stable_sigmoid((x - a) / tau); }
/* sigma_smaller (44-48) */
static double sigma_smaller(double x, double b, double tau) { return stable_sigmoid((b - x) / tau); }
/* within_s (51-54) */
static double within_s(double x, double lo, double hi, double tau) {
  return sigma_greater(x, lo, tau) * sigma_smaller(x, hi, tau);
}
/* sign_s (57-62) */
static double sign_s(double x, double tau) { return tanh(x / tau); }
/* softplus_s (66-81) */
static double softplus_s(double x, double tau) {
  const double s = x / tau;
  if (s > 0.0) return x + tau * log1p(exp(-s));
  return tau * log1p(exp(s));
}
/* clip_s (85-89) */
static double clip_s(double x, double lo, double hi, double tau) {
  return lo + softplus_s(x - lo, tau) - softplus_s(x - hi, tau);
}
/* argmin_s (126-144): softmax(-x/tau), min-shifted, first minimum. */
static void argmin_s(const double* xs, int n, double tau, double* out) {
  int mi = 0;
  for (int i = 1; i < n; ++i)
    if (xs[i] < xs[mi]) mi = i;
  const double m = xs[mi];
  double total = 0.0;
  for (int i = 0; i < n; ++i) {
    out[i] = exp((m - xs[i]) / tau);
    total += out[i];
  }
  const double inv = 1.0 / total;
  for (int i = 0; i < n; ++i) out[i] = out[i] * inv;
}
/* hard variants (202-218) */
static double clip_hard(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }
static double within_hard(double x, double lo, double hi) {
  return (x >= lo && x <= hi) ? 1.0 : 0.0;
}
static double sign_hard(double x) { return x < 0.0 ? -1.0 : (x > 0.0 ? 1.0 : 0.0); }
static void argmin_hard(const double* xs, int n, double* out) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (xs[i] < xs[best]) best = i;
  for (int i = 0; i < n; ++i) out[i] = 0.0;
  out[best] = 1.0;
}

static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x > y ? -1 : (x < y ? 1 : 0);
}

/* soft_topk (smooth_ops.hpp:173-198): row r = argmin_s(|sorted_desc_r - x|). */
int orc_soft_topk(const double* xs, int32_t d, int32_t k, double tau, double* w) {
  if (k < 1 || k > d) return 1;
  double* sorted = (double*)malloc(sizeof(double) * d);
  double* row = (double*)malloc(sizeof(double) * d);
  memcpy(sorted, xs, sizeof(double) * d);
  qsort(sorted, d, sizeof(double), cmp_desc);
  for (int r = 0; r < k; ++r) {
    for (int i = 0; i < d; ++i) row[i] = fabs(sorted[r] - xs[i]);
    argmin_s(row, d, tau, w + (size_t)r * d);
  }
  free(sorted);
  free(row);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* SE(3) (include/cmg/pose.hpp:37-91)                                         */
/* ------------------------------------------------------------------------- */
static void exp_coeffs(double th2, double* a, double* b, double* c) {
  if (th2 < 1e-8) { /* series branch, pose.hpp:47-51 */
    *a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    *b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    *c = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
  } else {
    const double th = sqrt(th2);
    *a = sin(th) / th;
    *b = (1.0 - cos(th)) / th2;
    *c = (1.0 - *a) / th2;
  }
}

/* se3_exp (pose.hpp:78-91): R = I + a W + b W^2, t = (I + b W + c W^2) rho. */
void orc_se3_exp(const double* xi, double* R, double* t) {
  const double wx = xi[3], wy = xi[4], wz = xi[5];
  const double th2 = wx * wx + wy * wy + wz * wz;
  double a, b, c;
  exp_coeffs(th2, &a, &b, &c);
  const double W[9] = {0, -wz, wy, wz, 0, -wx, -wy, wx, 0};
  double W2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = W[3 * i] * W[j];
      s += W[3 * i + 1] * W[3 + j];
      s += W[3 * i + 2] * W[6 + j];
      W2[3 * i + j] = s;
    }
  double V[9];
  for (int i = 0; i < 9; ++i) {
    const double id = (i % 4 == 0) ? 1.0 : 0.0;
    R[i] = (id + W[i] * a) + W2[i] * b;
    V[i] = (id + W[i] * b) + W2[i] * c;
  }
  const v3 r = mv(V, mk(xi[0], xi[1], xi[2]));
  t[0] = r.x;
  t[1] = r.y;
  t[2] = r.z;
}

/* ------------------------------------------------------------------------- */
/* SDF program (include/cmg/sdf.hpp)                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
  int op;
  int n_children;
  int children[64];
  double tau;
  /* SQ */
  double e1, e2, ax[3];
  double R[9], t[3]; /* body_from_prim (sdf.cpp:9) */
  /* CP / OPC */
  int count;
  double* normals;
  double* points;
  double* ls;
} onode;

struct orc_surface {
  int nv, ne;
  double* verts;
  int32_t* edges;
  onode* nodes;
  int n_nodes;
  int root;
  int vtopk, etopk;
  int leaves;
};

typedef struct {
  double v;
  v3 g;
} sample;

/* sq_inside_outside_canonical + sq_sdf_canonical (sdf.hpp:85-108) with the
 * analytic gradients of f and phi w.r.t. the canonical-frame point. */
static void sq_eval(const onode* q, v3 p, double* phi, v3* gphi, v3* gf) {
  const double xn = p.x / q->ax[0], yn = p.y / q->ax[1], zn = p.z / q->ax[2];
  const double x2 = xn * xn + 1e-30, y2 = yn * yn + 1e-30, z2 = zn * zn + 1e-30;
  const double p1 = 1.0 / q->e2, p2 = q->e2 / q->e1, p3 = 1.0 / q->e1, p4 = -q->e1 / 2.0;
  const double A = pow(x2, p1), B = pow(y2, p1);
  const double g = A + B;
  const double G = pow(g, p2);
  const double C = pow(z2, p3);
  const double f = G + C;
  /* d/d(p) through the normalisation p/axes; pow'(x) = p * pow(x, p - 1) (dual.hpp:224-232). */
  const double dA = p1 * pow(x2, p1 - 1.0) * (2.0 * xn) / q->ax[0];
  const double dB = p1 * pow(y2, p1 - 1.0) * (2.0 * yn) / q->ax[1];
  const double dG = p2 * pow(g, p2 - 1.0);
  const double dC = p3 * pow(z2, p3 - 1.0) * (2.0 * zn) / q->ax[2];
  const v3 df = mk(dG * dA, dG * dB, dC);
  const double r = sqrt(xn * xn + yn * yn + zn * zn + 1e-20);
  const double F = pow(f, p4);
  const double dFf = p4 * pow(f, p4 - 1.0);
  const double val = (1.0 - F) / r;
  const v3 dr = scl(mk(xn / q->ax[0], yn / q->ax[1], zn / q->ax[2]), 1.0 / r);
  if (phi) *phi = val;
  if (gphi) *gphi = scl(sub(scl(df, -dFf), scl(dr, val)), 1.0 / r);
  if (gf) *gf = df;
}

/* lse_max (smooth_ops.hpp:94-109) value + softmax weights. */
static double lse_max_w(const double* xs, int n, double tau, double* w) {
  int mi = 0;
  for (int i = 1; i < n; ++i)
    if (xs[i] > xs[mi]) mi = i;
  const double m = xs[mi];
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const double e = exp((xs[i] - m) / tau);
    if (w) w[i] = e;
    acc += e;
  }
  if (w)
    for (int i = 0; i < n; ++i) w[i] /= acc;
  return m + tau * log(acc);
}

/* flavor: 0 value, 1 true gradient, 2 normal source (sdf.hpp:204-288). */
static sample eval_node(const orc_surface* s, int idx, v3 p, int flavor) {
  const onode* nd = &s->nodes[idx];
  sample out = {0.0, {0, 0, 0}};
  switch (nd->op) {
    case CMGB_SDF_SUPERQUADRIC: {
      const v3 local = mtv(nd->R, sub(p, ld3(nd->t))); /* Transform::apply_inverse */
      double phi;
      v3 gphi, gf;
      sq_eval(nd, local, &phi, &gphi, &gf);
      out.v = phi;
      if (flavor == 1) out.g = mv(nd->R, gphi);
      if (flavor == 2) out.g = mv(nd->R, gf); /* SQ leaves contribute grad f (sdf.hpp:243-249) */
      break;
    }
    case CMGB_SDF_CONVEX_POLYHEDRON: { /* cp_sdf (sdf.hpp:110-117) */
      double d[256] = {0}, w[256];
      for (int i = 0; i < nd->count; ++i)
        d[i] = dot(ld3(nd->normals + 3 * i), sub(p, ld3(nd->points + 3 * i)));
      out.v = lse_max_w(d, nd->count, nd->tau, flavor ? w : NULL);
      if (flavor)
        for (int i = 0; i < nd->count; ++i)
          out.g = add(out.g, scl(ld3(nd->normals + 3 * i), w[i]));
      break;
    }
    case CMGB_SDF_ORIENTED_POINTCLOUD: { /* opc_sdf (sdf.hpp:119-132) */
      double num = 0.0, den = 1e-30;
      v3 dnum = mk(0, 0, 0), dden = mk(0, 0, 0);
      for (int i = 0; i < nd->count; ++i) {
        const v3 r = sub(p, ld3(nd->points + 3 * i));
        const v3 n = ld3(nd->normals + 3 * i);
        const double th = nd->ls[i];
        const double w = exp(-nsq(r) / (2.0 * th * th));
        const double nr = dot(n, r);
        num += w * nr;
        den += w;
        const v3 dw = scl(r, -w / (th * th));
        dnum = add(dnum, add(scl(dw, nr), scl(n, w)));
        dden = add(dden, dw);
      }
      out.v = num / den;
      if (flavor) out.g = scl(sub(dnum, scl(dden, out.v)), 1.0 / den);
      break;
    }
    case CMGB_SDF_UNION: { /* sdf.hpp:222-227, 260-277 */
      const int n = nd->n_children;
      double neg[64] = {0}, w[64];
      sample ch[64];
      for (int i = 0; i < n; ++i) {
        ch[i] = eval_node(s, nd->children[i], p, flavor);
        neg[i] = -ch[i].v;
      }
      out.v = -lse_max_w(neg, n, nd->tau, flavor ? w : NULL);
      if (flavor)
        for (int i = 0; i < n; ++i) out.g = add(out.g, scl(ch[i].g, w[i]));
      break;
    }
    case CMGB_SDF_SUBTRACTION: { /* sdf.hpp:228-230, 278-287 */
      const sample a = eval_node(s, nd->children[0], p, flavor);
      const sample b = eval_node(s, nd->children[1], p, flavor);
      const double args[2] = {a.v, -b.v};
      double w[2];
      out.v = lse_max_w(args, 2, nd->tau, flavor ? w : NULL);
      if (flavor) out.g = sub(scl(a.g, w[0]), scl(b.g, w[1]));
      break;
    }
  }
  return out;
}

static void surf_free(orc_surface* s) {
  if (!s) return;
  for (int i = 0; i < s->n_nodes; ++i) {
    free(s->nodes[i].normals);
    free(s->nodes[i].points);
    free(s->nodes[i].ls);
  }
  free(s->nodes);
  free(s->verts);
  free(s->edges);
  free(s);
}

static int count_leaves(const orc_surface* s, int idx) {
  const onode* nd = &s->nodes[idx];
  if (nd->op <= CMGB_SDF_ORIENTED_POINTCLOUD) return 1;
  int n = 0;
  for (int i = 0; i < nd->n_children; ++i) n += count_leaves(s, nd->children[i]);
  return n;
}

orc_surface* orc_surface_create(const double* vertices, int32_t n_vertices, const int32_t* edges,
                                int32_t n_edges, const cmgb_sdf_node* nodes, int32_t n_nodes,
                                int32_t vertex_topk, int32_t edge_topk) {
  orc_surface* s = (orc_surface*)calloc(1, sizeof(orc_surface));
  s->nv = n_vertices;
  s->ne = n_edges;
  s->verts = (double*)malloc(sizeof(double) * 3 * n_vertices);
  memcpy(s->verts, vertices, sizeof(double) * 3 * n_vertices);
  s->edges = (int32_t*)malloc(sizeof(int32_t) * 2 * n_edges);
  memcpy(s->edges, edges, sizeof(int32_t) * 2 * n_edges);
  s->nodes = (onode*)calloc(n_nodes, sizeof(onode));
  s->n_nodes = n_nodes;
  int stack[256], sp = 0;
  for (int i = 0; i < n_nodes; ++i) {
    const cmgb_sdf_node* in = &nodes[i];
    onode* nd = &s->nodes[i];
    nd->op = in->op;
    nd->tau = in->tau;
    nd->count = in->count;
    switch (in->op) {
      case CMGB_SDF_SUPERQUADRIC:
        nd->e1 = in->eps1;
        nd->e2 = in->eps2;
        memcpy(nd->ax, in->axes, sizeof(double) * 3);
        orc_se3_exp(in->pose, nd->R, nd->t);
        stack[sp++] = i;
        break;
      case CMGB_SDF_CONVEX_POLYHEDRON:
      case CMGB_SDF_ORIENTED_POINTCLOUD:
        nd->normals = (double*)malloc(sizeof(double) * 3 * in->count);
        nd->points = (double*)malloc(sizeof(double) * 3 * in->count);
        memcpy(nd->normals, in->normals, sizeof(double) * 3 * in->count);
        memcpy(nd->points, in->points, sizeof(double) * 3 * in->count);
        if (in->op == CMGB_SDF_ORIENTED_POINTCLOUD) {
          nd->ls = (double*)malloc(sizeof(double) * in->count);
          memcpy(nd->ls, in->lengthscales, sizeof(double) * in->count);
        }
        stack[sp++] = i;
        break;
      case CMGB_SDF_UNION:
        if (in->count < 1 || in->count > sp || in->count > 64) { surf_free(s); return NULL; }
        nd->n_children = in->count;
        for (int k = 0; k < in->count; ++k) nd->children[k] = stack[sp - in->count + k];
        sp -= in->count;
        stack[sp++] = i;
        break;
      case CMGB_SDF_SUBTRACTION:
        if (sp < 2) { surf_free(s); return NULL; }
        nd->n_children = 2;
        nd->children[0] = stack[sp - 2];
        nd->children[1] = stack[sp - 1];
        sp -= 2;
        stack[sp++] = i;
        break;
      default:
        surf_free(s);
        return NULL;
    }
  }
  if (sp != 1) { surf_free(s); return NULL; }
  s->root = stack[0];
  s->leaves = count_leaves(s, s->root);
  s->vtopk = vertex_topk;
  s->etopk = edge_topk;
  return s;
}

void orc_surface_destroy(orc_surface* s) { surf_free(s); }

/* effective_vertex_topk / effective_edge_topk (surface.hpp:24-32). */
static int eff_vtopk(const orc_surface* s) {
  return s->vtopk <= 0 ? s->nv : (s->vtopk < s->nv ? s->vtopk : s->nv);
}
static int eff_etopk(const orc_surface* s) {
  if (s->etopk <= 0) return s->leaves < s->ne ? s->leaves : s->ne;
  return s->etopk < s->ne ? s->etopk : s->ne;
}

void orc_surface_budgets(const orc_surface* s, int32_t* out3) {
  out3[0] = eff_vtopk(s);
  out3[1] = eff_etopk(s);
  out3[2] = s->leaves;
}

void orc_sdf_query(const orc_surface* s, int32_t flavor, const double* p, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const sample r = eval_node(s, s->root, ld3(p + 3 * i), flavor);
    out[4 * i] = r.v;
    out[4 * i + 1] = flavor ? r.g.x : 0.0;
    out[4 * i + 2] = flavor ? r.g.y : 0.0;
    out[4 * i + 3] = flavor ? r.g.z : 0.0;
  }
}

/* PosedSdf (sdf.hpp:294-312): world query pulled back, gradient pushed forward. */
typedef struct {
  const orc_surface* s;
  double R[9], t[3];
} posed;

static sample posed_eval(const posed* ps, v3 pw, int flavor) {
  const v3 pb = mtv(ps->R, sub(pw, ld3(ps->t)));
  sample r = eval_node(ps->s, ps->s->root, pb, flavor);
  if (flavor) r.g = mv(ps->R, r.g);
  return r;
}

/* sphere_trace_project (sdf.hpp:318-326). */
static v3 sphere_trace(const posed* ps, v3 p, int iters, double tau) {
  for (int k = 0; k < iters; ++k) {
    const sample s = posed_eval(ps, p, 1);
    p = sub(p, scl(normalize_smooth(s.g, tau), s.v));
  }
  return p;
}

void orc_sphere_trace(const orc_surface* s, const double* pose, const double* p, int64_t n,
                      int32_t iters, double tau, double* out) {
  posed ps;
  ps.s = s;
  orc_se3_exp(pose, ps.R, ps.t);
  for (int64_t i = 0; i < n; ++i) {
    const v3 r = sphere_trace(&ps, ld3(p + 3 * i), iters, tau);
    out[3 * i] = r.x;
    out[3 * i + 1] = r.y;
    out[3 * i + 2] = r.z;
  }
}

/* ------------------------------------------------------------------------- */
/* witness solvers (include/cmg/witness.hpp)                                  */
/* ------------------------------------------------------------------------- */
static double clip01(double x, const cmgb_config* c) { /* 45-52 */
  return c->hard_ops ? clip_hard(x, 0.0, 1.0) : clip_s(x, 0.0, 1.0, c->tau_clip);
}
static double within01(double x, const cmgb_config* c) { /* 54-61 */
  return c->hard_ops ? within_hard(x, 0.0, 1.0) : within_s(x, 0.0, 1.0, c->tau_comp);
}

/* solve_box_qp_2 (witness.hpp:74-121), plus the active-set label. */
static void box_qp(double q1, double q2, double q3, double c1, double c2, const cmgb_config* c,
                   double* a1, double* a2, double* gamma, int32_t* label) {
  const double q2_over_q1 = q2 / q1, q2_over_q3 = q2 / q3;
  const double c1_over_q1 = c1 / q1, c2_over_q3 = c2 / q3;
  const double a1u = (q2 * c2_over_q3 - c1) / (q1 - q2 * q2_over_q3);
  const double a2u = (q2 * c1_over_q1 - c2) / (q3 - q2 * q2_over_q1);
  const double a1_1_a2 = clip01(-(q2_over_q3 + c2_over_q3), c);
  const double a1_0_a2 = clip01(-c2_over_q3, c);
  const double a2_1_a1 = clip01(-(q2_over_q1 + c1_over_q1), c);
  const double a2_0_a1 = clip01(-c1_over_q1, c);
  const double costs[4] = {
      0.5 * (q1 + 2.0 * q2 * a1_1_a2 + q3 * a1_1_a2 * a1_1_a2) + c1 + c2 * a1_1_a2,
      0.5 * q3 * a1_0_a2 * a1_0_a2 + c2 * a1_0_a2,
      0.5 * (q1 * a2_1_a1 * a2_1_a1 + 2.0 * q2 * a2_1_a1 + q3) + c1 * a2_1_a1 + c2,
      0.5 * q1 * a2_0_a1 * a2_0_a1 + c1 * a2_0_a1,
  };
  const double cand[4][2] = {{1.0, a1_1_a2}, {0.0, a1_0_a2}, {a2_1_a1, 1.0}, {a2_0_a1, 0.0}};
  double w[4];
  if (c->hard_ops) argmin_hard(costs, 4, w);
  else argmin_s(costs, 4, c->tau_min, w);
  double k0 = 0.0, k1 = 0.0;
  for (int i = 0; i < 4; ++i) {
    k0 += cand[i][0] * w[i];
    k1 += cand[i][1] * w[i];
  }
  const double inside = within01(a1u, c) * within01(a2u, c);
  *gamma = inside;
  *a1 = a1u * inside + k0 * (1.0 - inside);
  *a2 = a2u * inside + k1 * (1.0 - inside);
  if (label) {
    int best = 0;
    for (int i = 1; i < 4; ++i)
      if (w[i] > w[best]) best = i;
    *label = best | ((inside >= 0.5) << 2);
  }
}

void orc_box_qp(const double* qp, int64_t n, const cmgb_config* cfg, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    const double* q = qp + 5 * i;
    box_qp(q[0], q[1], q[2], q[3], q[4], cfg, out + 3 * i, out + 3 * i + 1, out + 3 * i + 2, NULL);
  }
}

/* ee_witness (witness.hpp:137-158). */
static void ee_witness(v3 e1a, v3 e1b, v3 e2a, v3 e2b, const cmgb_config* c, v3* p1, v3* p2,
                       double* a1, double* a2, double* gamma, int32_t* label) {
  const v3 t1 = sub(e1b, e1a);
  const v3 t2n = sub(e2a, e2b);
  const v3 b = sub(e1a, e2a);
  const double q11 = dot(t1, t1) + c->lambda;
  const double q12 = dot(t1, t2n);
  const double q22 = dot(t2n, t2n) + c->lambda;
  const double c1 = dot(b, t1) - 0.5 * c->lambda;
  const double c2 = dot(b, t2n) - 0.5 * c->lambda;
  box_qp(q11, q12, q22, c1, c2, c, a1, a2, gamma, label);
  *p1 = add(e1a, scl(sub(e1b, e1a), *a1)); /* edge_point (130-133) */
  *p2 = add(e2a, scl(sub(e2b, e2a), *a2));
}

void orc_ee_witness(const double* pairs, int64_t n, const cmgb_config* cfg, double* out,
                    int32_t* labels) {
  for (int64_t i = 0; i < n; ++i) {
    const double* p = pairs + 12 * i;
    v3 p1, p2;
    double* o = out + 9 * i;
    ee_witness(ld3(p), ld3(p + 3), ld3(p + 6), ld3(p + 9), cfg, &p1, &p2, o + 6, o + 7, o + 8,
               labels ? labels + i : NULL);
    o[0] = p1.x; o[1] = p1.y; o[2] = p1.z;
    o[3] = p2.x; o[4] = p2.y; o[5] = p2.z;
  }
}

/* vf_witness (witness.hpp:163-227). */
static v3 vf_witness(v3 v, v3 t0, v3 t1, v3 t2, const cmgb_config* c, int32_t* label) {
  const v3 d10 = sub(t1, t0), d21 = sub(t2, t1), d20 = sub(t2, t0);
  const v3 dv0 = sub(v, t0), dv1 = sub(v, t1);
  const double guard = 1e-12; /* kEdgeNormalEps */
  const double len10 = sqrt(nsq(d10) + guard), len21 = sqrt(nsq(d21) + guard),
               len20 = sqrt(nsq(d20) + guard);
  /* u = d / len (Vec3 operator/, vec3.hpp:31) */
  const v3 U10 = mk(d10.x / len10, d10.y / len10, d10.z / len10);
  const v3 U21 = mk(d21.x / len21, d21.y / len21, d21.z / len21);
  const v3 U20 = mk(d20.x / len20, d20.y / len20, d20.z / len20);
#define CLIP_LEN(s, len) \
  (c->hard_ops ? clip_hard((s), 0.0, (len)) \
               : softplus_s((s), c->tau_clip) - softplus_s((s) - (len), c->tau_clip))
  const v3 on1 = add(t0, scl(U10, CLIP_LEN(dot(dv0, U10), len10)));
  const v3 on2 = add(t1, scl(U21, CLIP_LEN(dot(dv1, U21), len21)));
  const v3 on3 = add(t0, scl(U20, CLIP_LEN(dot(dv0, U20), len20)));
#undef CLIP_LEN
  const double costs[3] = {sqrt(nsq(sub(v, on1))), sqrt(nsq(sub(v, on2))), sqrt(nsq(sub(v, on3)))};
  double w[3];
  if (c->hard_ops) argmin_hard(costs, 3, w);
  else argmin_s(costs, 3, c->tau_min, w);
  const v3 cons = add(add(scl(on1, w[0]), scl(on2, w[1])), scl(on3, w[2]));
  const v3 n_raw = cross(d10, d20);
  const double n_norm = sqrt(nsq(n_raw) + guard);
  const v3 n = mk(n_raw.x / n_norm, n_raw.y / n_norm, n_raw.z / n_norm);
  const v3 dvp0 = sub(dv0, scl(n, dot(dv0, n)));
  const v3 plane = add(t0, dvp0);
  const double bv = dot(cross(d10, dvp0), n) / n_norm;
  const double bu = dot(cross(dvp0, d20), n) / n_norm;
  const double bw = 1.0 - bu - bv;
  const double inside = within01(bu, c) * within01(bv, c) * within01(bw, c);
  if (label) {
    int best = 0;
    for (int i = 1; i < 3; ++i)
      if (w[i] > w[best]) best = i;
    *label = best | ((inside >= 0.5) << 2);
  }
  return add(scl(plane, inside), scl(cons, 1.0 - inside));
}

void orc_vf_witness(const double* pairs, int64_t n, const cmgb_config* cfg, double* out,
                    int32_t* labels) {
  for (int64_t i = 0; i < n; ++i) {
    const double* p = pairs + 12 * i;
    const v3 r = vf_witness(ld3(p), ld3(p + 3), ld3(p + 6), ld3(p + 9), cfg,
                            labels ? labels + i : NULL);
    out[3 * i] = r.x;
    out[3 * i + 1] = r.y;
    out[3 * i + 2] = r.z;
  }
}

/* ------------------------------------------------------------------------- */
/* manifold pipeline (include/cmg/manifold.hpp)                               */
/* ------------------------------------------------------------------------- */
typedef struct {
  int k;
  v3* pos;      /* K */
  v3* b;        /* edges: second endpoint */
  int* source;  /* K */
} selected;

/* select_topk_vertices / select_topk_edges (manifold.hpp:128-181) +
 * hard_attribution (110-121). is_edge: payload = both endpoints. */
static void select_topk(const v3* verts, const int32_t* edges, int d, const double* pens, int k,
                        double tau, int is_edge, selected* out) {
  out->k = k;
  out->pos = (v3*)calloc(k, sizeof(v3));
  out->b = is_edge ? (v3*)calloc(k, sizeof(v3)) : NULL;
  out->source = (int*)calloc(k, sizeof(int));
  if (k == d) { /* K == D pass-through */
    for (int i = 0; i < d; ++i) {
      out->pos[i] = is_edge ? verts[edges[2 * i]] : verts[i];
      if (is_edge) out->b[i] = verts[edges[2 * i + 1]];
      out->source[i] = i;
    }
    return;
  }
  double* scores = (double*)malloc(sizeof(double) * d);
  double* w = (double*)malloc(sizeof(double) * (size_t)k * d);
  for (int i = 0; i < d; ++i) scores[i] = -pens[i];
  orc_soft_topk(scores, d, k, tau, w);
  for (int r = 0; r < k; ++r) {
    const double* row = w + (size_t)r * d;
    v3 a = mk(0, 0, 0), bb = mk(0, 0, 0);
    int best = 0;
    for (int i = 0; i < d; ++i) {
      if (is_edge) {
        a = add(a, scl(verts[edges[2 * i]], row[i]));
        bb = add(bb, scl(verts[edges[2 * i + 1]], row[i]));
      } else {
        a = add(a, scl(verts[i], row[i]));
      }
      if (i > 0 && row[i] > row[best]) best = i;
    }
    out->pos[r] = a;
    if (is_edge) out->b[r] = bb;
    out->source[r] = best;
  }
  free(scores);
  free(w);
}

static void sel_free(selected* s) {
  free(s->pos);
  free(s->b);
  free(s->source);
}

static void put_contact(double* c, int32_t* m, v3 p, double dist, v3 n, double act, int kind,
                        int side, int a, int b) {
  if (c) {
    c[0] = p.x; c[1] = p.y; c[2] = p.z; c[3] = dist;
    c[4] = n.x; c[5] = n.y; c[6] = n.z; c[7] = act;
  }
  if (m) { m[0] = kind; m[1] = side; m[2] = a; m[3] = b; }
}

/* vs_contacts (manifold.hpp:185-204). */
static void vs_contacts(const selected* sel, const posed* opp, const cmgb_config* c, int side,
                        double* contacts, int32_t* meta) {
  for (int i = 0; i < sel->k; ++i) {
    const sample s = posed_eval(opp, sel->pos[i], 2);
    put_contact(contacts ? contacts + 8 * i : NULL, meta ? meta + 4 * i : NULL, sel->pos[i], s.v,
                normalize_smooth(s.g, c->tau_normal), sigma_greater(-s.v, 0.0, c->tau_pen), 0,
                side, sel->source[i], -1);
  }
}

/* ee_contacts (manifold.hpp:212-332). */
static void ee_contacts(const selected* e1, const selected* e2, const posed* sdf1,
                        const posed* sdf2, const cmgb_config* c, double* contacts,
                        int32_t* meta, double* ee) {
  const int m1 = e1->k, m2 = e2->k, n = m1 * m2;
  double* mat = (double*)calloc((size_t)9 * n, sizeof(double));
  double *D = mat, *con = mat + n, *pen1 = mat + 2 * n, *pen2 = mat + 3 * n, *nn1 = mat + 4 * n,
         *nn2 = mat + 5 * n, *clash = mat + 6 * n, *act1 = mat + 7 * n, *act2 = mat + 8 * n;
  v3* wp1 = (v3*)malloc(sizeof(v3) * n);
  v3* wp2 = (v3*)malloc(sizeof(v3) * n);
  v3* nbar = (v3*)malloc(sizeof(v3) * n);
  double* s1 = (double*)malloc(sizeof(double) * n);
  double* s2 = (double*)malloc(sizeof(double) * n);
  double* cont = (double*)malloc(sizeof(double) * n);
  for (int k = 0; k < m1; ++k)
    for (int l = 0; l < m2; ++l) {
      const int i = k * m2 + l;
      v3 p1, p2;
      double a1, a2, g;
      ee_witness(e1->pos[k], e1->b[k], e2->pos[l], e2->b[l], c, &p1, &p2, &a1, &a2, &g, NULL);
      if (c->sphere_trace && c->sphere_trace_iters > 0) {
        p1 = sphere_trace(sdf1, p1, c->sphere_trace_iters, c->tau_normal);
        p2 = sphere_trace(sdf2, p2, c->sphere_trace_iters, c->tau_normal);
      }
      const v3 delta = sub(p1, p2);
      const double dg = sqrt(nsq(delta) + 1e-12);
      const v3 nu = mk(delta.x / dg, delta.y / dg, delta.z / dg);
      const sample own1 = posed_eval(sdf1, p1, 2);
      const sample own2 = posed_eval(sdf2, p2, 2);
      const v3 n1 = normalize_smooth(own1.g, c->tau_normal);
      const v3 n2 = normalize_smooth(own2.g, c->tau_normal);
      double g1, g2;
      if (c->hard_ops) {
        g1 = sign_hard(dot(n2, nu));
        g2 = sign_hard(dot(n1, nu));
      } else {
        g1 = sign_s(dot(n2, nu), c->tau_sign);
        g2 = sign_s(dot(n1, nu), c->tau_sign);
      }
      wp1[i] = p1;
      wp2[i] = p2;
      nbar[i] = nu;
      s1[i] = g1;
      s2[i] = g2;
      D[i] = dg;
      con[i] = g;
      pen1[i] = sigma_greater(-posed_eval(sdf2, p1, 0).v, 0.0, c->tau_pen);
      pen2[i] = sigma_greater(-posed_eval(sdf1, p2, 0).v, 0.0, c->tau_pen);
      clash[i] = sigma_greater(-dot(n1, n2), 0.0, c->tau_clash);
      cont[i] = 1.0;
      if (c->containment_safeguard)
        cont[i] = sigma_greater(-own1.v, 0.0, c->tau_cont) * sigma_greater(-own2.v, 0.0, c->tau_cont);
    }
  /* nearest-neighbour softmins: rows (side 1), columns (side 2) (289-301) */
  double buf[1024], col[1024];
  for (int k = 0; k < m1; ++k) {
    argmin_s(D + k * m2, m2, c->tau_nn, buf);
    for (int l = 0; l < m2; ++l) nn1[k * m2 + l] = buf[l];
  }
  for (int l = 0; l < m2; ++l) {
    for (int k = 0; k < m1; ++k) col[k] = D[k * m2 + l];
    argmin_s(col, m1, c->tau_nn, buf);
    for (int k = 0; k < m1; ++k) nn2[k * m2 + l] = buf[k];
  }
  for (int k = 0; k < m1; ++k)
    for (int l = 0; l < m2; ++l) {
      const int i = k * m2 + l;
      act1[i] = con[i] * pen1[i] * nn1[i] * clash[i] * cont[i];
      act2[i] = con[i] * pen2[i] * nn2[i] * clash[i] * cont[i];
      put_contact(contacts ? contacts + 16 * i : NULL, meta ? meta + 8 * i : NULL, wp1[i],
                  s1[i] * D[i], scl(nbar[i], s1[i]), act1[i], 1, 1, e1->source[k], e2->source[l]);
      put_contact(contacts ? contacts + 16 * i + 8 : NULL, meta ? meta + 8 * i + 4 : NULL, wp2[i],
                  s2[i] * D[i], scl(nbar[i], s2[i]), act2[i], 1, 2, e1->source[k], e2->source[l]);
    }
  if (ee) memcpy(ee, mat, sizeof(double) * 9 * n);
  free(mat); free(wp1); free(wp2); free(nbar); free(s1); free(s2); free(cont);
}

/* generate_manifold (manifold.hpp:336-377). */
int orc_manifold(const orc_surface* m1s, const orc_surface* m2s, const double* pose1,
                 const double* pose2, const cmgb_config* c, double* contacts, int32_t* meta,
                 double* ee, int32_t* layout) {
  posed ps1, ps2;
  ps1.s = m1s;
  ps2.s = m2s;
  orc_se3_exp(pose1, ps1.R, ps1.t);
  orc_se3_exp(pose2, ps2.R, ps2.t);
  v3* w1 = (v3*)malloc(sizeof(v3) * m1s->nv);
  v3* w2 = (v3*)malloc(sizeof(v3) * m2s->nv);
  for (int i = 0; i < m1s->nv; ++i) w1[i] = add(mv(ps1.R, ld3(m1s->verts + 3 * i)), ld3(ps1.t));
  for (int i = 0; i < m2s->nv; ++i) w2[i] = add(mv(ps2.R, ld3(m2s->verts + 3 * i)), ld3(ps2.t));
  double* pens1 = (double*)malloc(sizeof(double) * m1s->nv);
  double* pens2 = (double*)malloc(sizeof(double) * m2s->nv);
  for (int i = 0; i < m1s->nv; ++i) pens1[i] = posed_eval(&ps2, w1[i], 0).v;
  const int n1 = eff_vtopk(m1s);
  int n2 = 0, mm1 = 0, mm2 = 0;
  selected sv1;
  select_topk(w1, NULL, m1s->nv, pens1, n1, c->tau_topk_verts, 0, &sv1);
  vs_contacts(&sv1, &ps2, c, 1, contacts, meta);
  int off = n1;
  if (c->mode != CMGB_MODE_ONE_SIDED) {
    for (int i = 0; i < m2s->nv; ++i) pens2[i] = posed_eval(&ps1, w2[i], 0).v;
    n2 = eff_vtopk(m2s);
    selected sv2;
    select_topk(w2, NULL, m2s->nv, pens2, n2, c->tau_topk_verts, 0, &sv2);
    vs_contacts(&sv2, &ps1, c, 2, contacts ? contacts + 8 * off : NULL, meta ? meta + 4 * off : NULL);
    off += n2;
    sel_free(&sv2);
    if (c->mode == CMGB_MODE_FULL) {
      mm1 = eff_etopk(m1s);
      mm2 = eff_etopk(m2s);
      double* ep1 = (double*)malloc(sizeof(double) * m1s->ne);
      double* ep2 = (double*)malloc(sizeof(double) * m2s->ne);
      for (int i = 0; i < m1s->ne; ++i) /* edge_penetrations (86-94) */
        ep1[i] = (pens1[m1s->edges[2 * i]] + pens1[m1s->edges[2 * i + 1]]) * 0.5;
      for (int i = 0; i < m2s->ne; ++i)
        ep2[i] = (pens2[m2s->edges[2 * i]] + pens2[m2s->edges[2 * i + 1]]) * 0.5;
      selected se1, se2;
      select_topk(w1, m1s->edges, m1s->ne, ep1, mm1, c->tau_topk_edges, 1, &se1);
      select_topk(w2, m2s->edges, m2s->ne, ep2, mm2, c->tau_topk_edges, 1, &se2);
      ee_contacts(&se1, &se2, &ps1, &ps2, c, contacts ? contacts + 8 * off : NULL,
                  meta ? meta + 4 * off : NULL, ee);
      off += 2 * mm1 * mm2;
      sel_free(&se1);
      sel_free(&se2);
      free(ep1);
      free(ep2);
    }
  }
  sel_free(&sv1);
  if (layout) {
    layout[0] = n1; layout[1] = n2; layout[2] = mm1; layout[3] = mm2; layout[4] = off;
  }
  free(w1); free(w2); free(pens1); free(pens2);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* batch over envs (the oracle's own pthread split; src/batch.cpp:27-41 shape) */
/* ------------------------------------------------------------------------- */
typedef struct {
  const orc_surface *s1, *s2;
  const double *poses1, *poses2;
  int32_t st1, st2;
  const cmgb_config* cfg;
  int64_t lo, hi;
  int per_env, pairs;
  double* contacts;
  int32_t* meta;
  double* ee;
  double* mean;
} job;

static void* run_job(void* arg) {
  job* j = (job*)arg;
  double* tmp = j->mean && !j->contacts ? (double*)malloc(sizeof(double) * 8 * j->per_env) : NULL;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    double* c = j->contacts ? j->contacts + (size_t)8 * j->per_env * i : tmp;
    orc_manifold(j->s1, j->s2, j->poses1 + 6 * i * j->st1, j->poses2 + 6 * i * j->st2, j->cfg, c,
                 j->meta ? j->meta + (size_t)4 * j->per_env * i : NULL,
                 j->ee ? j->ee + (size_t)9 * j->pairs * i : NULL, NULL);
    if (j->mean) { /* mean_contact_distance (379-384) */
      double acc = 0.0;
      for (int q = 0; q < j->per_env; ++q) acc += c[8 * q + 3];
      j->mean[i] = acc / (double)j->per_env;
    }
  }
  free(tmp);
  return NULL;
}

int orc_manifold_batch(const orc_surface* s1, const orc_surface* s2, const double* poses1,
                       int32_t pose1_stride, const double* poses2, int32_t pose2_stride,
                       int64_t n_env, const cmgb_config* cfg, int32_t threads, double* contacts,
                       int32_t* meta, double* ee, double* mean_dist) {
  int32_t layout[5];
  orc_manifold(s1, s2, poses1, poses2, cfg, NULL, NULL, NULL, layout);
  const int per_env = layout[4];
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  job jobs[256];
  const int64_t chunk = (n_env + threads - 1) / threads;
  int launched = 0;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = (int64_t)t * chunk;
    const int64_t hi = lo + chunk < n_env ? lo + chunk : n_env;
    if (lo >= hi) break;
    job jb = {s1, s2, poses1, poses2, pose1_stride, pose2_stride, cfg, lo, hi, per_env,
              layout[2] * layout[3], contacts, meta, ee, mean_dist};
    jobs[t] = jb;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
    ++launched;
  }
  for (int t = 0; t < launched; ++t) pthread_join(th[t], NULL);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* std::mt19937_64 + uniform_real_distribution<double> (libstdc++), used by    */
/* make_random_*_pairs (batch.cpp:18-24, 45-51) and the pose jitter (196-203). */
/* ------------------------------------------------------------------------- */
void orc_mt19937_64_uniform(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  enum { NN = 312, MM = 156 };
  uint64_t mt[NN];
  mt[0] = seed;
  for (int i = 1; i < NN; ++i)
    mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  int idx = NN;
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  for (int64_t k = 0; k < n; ++k) {
    if (idx >= NN) {
      for (int i = 0; i < NN; ++i) {
        const uint64_t x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        mt[i] = mt[(i + MM) % NN] ^ xa;
      }
      idx = 0;
    }
    uint64_t y = mt[idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    double r = (double)y / 18446744073709551616.0; /* generate_canonical<double,53> */
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    out[k] = r * (hi - lo) + lo;
  }
}
