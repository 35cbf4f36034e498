// Forward-mode pose Jacobian of the batched contact manifold:
//   generate_manifold<Dual12> seeded by seed_pose_tangents (dual.hpp:249-263)
//   and mean_contact_distance (manifold.hpp:379-384), for every env.
//
// The reference carries 12 tangents through every scalar of the pipeline. Most
// of its arithmetic (the sphere trace, ~73%, plus the normal sources and the
// opposing-field values) is a function of a single 3-D body-frame point, so
// its 12-direction tangent factors through a 3x3 Jacobian: here those stages
// run ONCE per item in Dual<3> arithmetic seeded at the point (dual.cuh), and
// the 12 pose directions are then pushed through the small Jacobians by
// explicit chain-rule loops. The same holds for the witness QP, a function of
// the 5 numbers (Q, c) (witness.hpp:74-121): Dual<5>. Everything outside those
// bottlenecks (frames, slot payloads, pair quantities, NN softmins, activity)
// carries the 12 tangents directly (Dual<12> records in shared memory,
// per-direction loops in registers).
//
// Work mapping (one CTA owns `units_per_block` consecutive envs; items of all
// its envs spread over the CTA's threads phase by phase, as manifold.cu):
//   A  frames: se3_exp in Dual<6> per pose (pose.hpp:78-91)
//   B  top-K scores: opposing field value + gradient (double), 12-direction chain
//   C  rank sort on primals, stable on ties (smooth_ops.hpp:180-185)
//   D  slots: soft top-K rows / pass-through, one item per (slot, direction)
//   E  E-E pairs (QP Dual<5>, two sides' trace + normal Dual<3>, opposing
//      value gradient) and V-S items (normal source Dual<3>); then the 12
//      directions through the Jacobians; point / dist / normal rows out
//   F  NN softmin statistics (argmin_s shift carries its tangent)
//   G  activity product + its tangents
//   H  mean contact distance + gradient (fixed order)
// Semantics that touch tangents are the reference's: branches on primals,
// fabs subgradient 0 at the kink (dual.hpp:236-246), soft top-K sort stable on
// ties (libstdc++ insertion sort for D <= 16), argmin / LSE shifts carry their
// tangents. hard_ops is rejected by the host (smooth_ops.hpp:199).
//
// Outputs: contacts (primal, FP32), tangents [n_env][C][8][12] FP32, mean_dist
// and its 12 tangents.
#include <cuda_runtime.h>

#include "../common.h"
#include "launch_util.cuh"
#include "../device/dmath.cuh"
#include "../device/dual.cuh"
#include "../device/sdf.cuh"
#include "../device/witness.cuh"

namespace cmgb {

namespace {

#ifndef CMGB_JVP_THREADS
#define CMGB_JVP_THREADS 128
#endif
#ifndef CMGB_JVP_MINB
#define CMGB_JVP_MINB 2
#endif
#ifndef CMGB_JVP_SMEM_KB
#define CMGB_JVP_SMEM_KB 110
#endif
constexpr int kJvpThreads = CMGB_JVP_THREADS;
constexpr int kJvpMinBlocks = CMGB_JVP_MINB;

using D3 = Dual<3>;

// Shared-memory tangent record: FP64 primal, 12 FP32 pose tangents (the
// tangent outputs are FP32; every combination of tangents, differences
// included, is formed in FP64 registers).
struct T12 {
  double v;
  float d[12];
};

struct Frame {
  T12 R[9];
  T12 t[3];
};

// ---- primal / tangent views of frames and Dual<12> vectors ---------------------
__device__ __forceinline__ double3 val3(const T12* q) { return d3(q[0].v, q[1].v, q[2].v); }
__device__ __forceinline__ double3 tan3(const T12* q, int j) { return d3(q[0].d[j], q[1].d[j], q[2].d[j]); }
__device__ __forceinline__ double3 fR(const Frame& F, double3 v) {  // R v
  return d3(F.R[0].v * v.x + F.R[1].v * v.y + F.R[2].v * v.z, F.R[3].v * v.x + F.R[4].v * v.y + F.R[5].v * v.z,
            F.R[6].v * v.x + F.R[7].v * v.y + F.R[8].v * v.z);
}
__device__ __forceinline__ double3 fRt(const Frame& F, double3 v) {  // R^T v
  return d3(F.R[0].v * v.x + F.R[3].v * v.y + F.R[6].v * v.z, F.R[1].v * v.x + F.R[4].v * v.y + F.R[7].v * v.z,
            F.R[2].v * v.x + F.R[5].v * v.y + F.R[8].v * v.z);
}
__device__ __forceinline__ double3 fdR(const Frame& F, double3 v, int j) {  // (dR/dj) v
  return d3(F.R[0].d[j] * v.x + F.R[1].d[j] * v.y + F.R[2].d[j] * v.z,
            F.R[3].d[j] * v.x + F.R[4].d[j] * v.y + F.R[5].d[j] * v.z,
            F.R[6].d[j] * v.x + F.R[7].d[j] * v.y + F.R[8].d[j] * v.z);
}
__device__ __forceinline__ double3 fdRt(const Frame& F, double3 v, int j) {  // (dR/dj)^T v
  return d3(F.R[0].d[j] * v.x + F.R[3].d[j] * v.y + F.R[6].d[j] * v.z,
            F.R[1].d[j] * v.x + F.R[4].d[j] * v.y + F.R[7].d[j] * v.z,
            F.R[2].d[j] * v.x + F.R[5].d[j] * v.y + F.R[8].d[j] * v.z);
}
__device__ __forceinline__ double3 ft(const Frame& F) { return val3(F.t); }
__device__ __forceinline__ double3 fdt(const Frame& F, int j) { return tan3(F.t, j); }
// M v for a row-major 3x3 held in registers
__device__ __forceinline__ double3 mv3(const double (&M)[9], double3 v) {
  return d3(M[0] * v.x + M[1] * v.y + M[2] * v.z, M[3] * v.x + M[4] * v.y + M[5] * v.z,
            M[6] * v.x + M[7] * v.y + M[8] * v.z);
}
__device__ __forceinline__ void put3(T12* q, double3 v) {
  q[0].v = v.x;
  q[1].v = v.y;
  q[2].v = v.z;
}
__device__ __forceinline__ void put3d(T12* q, double3 v, int j) {
  q[0].d[j] = v.x;
  q[1].d[j] = v.y;
  q[2].d[j] = v.z;
}
__device__ __forceinline__ double3 dvert(const double* v, int i) {
  return d3(__ldg(v + 3 * i), __ldg(v + 3 * i + 1), __ldg(v + 3 * i + 2));
}

// A 3-vector of Dual<3> seeded with the identity at p (d p_r / d p_c = delta).
__device__ __forceinline__ V3<D3> seed3(double3 p) {
  V3<D3> q;
  q.x = D3(p.x);
  q.y = D3(p.y);
  q.z = D3(p.z);
  q.x.d[0] = 1.0;
  q.y.d[1] = 1.0;
  q.z.d[2] = 1.0;
  return q;
}
__device__ __forceinline__ double3 prim3(const V3<D3>& q) { return d3(q.x.v, q.y.v, q.z.v); }
__device__ __forceinline__ void jac3(const V3<D3>& q, double (&J)[9]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    J[c] = q.x.d[c];
    J[3 + c] = q.y.d[c];
    J[6 + c] = q.z.d[c];
  }
}

template <class T>
__device__ __forceinline__ V3<T> normalize_smooth_t(const V3<T>& v, double tau) {
  return dscale(v, rsqrt_d(tau + ddot(v, v)));
}

// Tangent output of one contact field: t[(row * 8 + k) * 12 + j].
__device__ __forceinline__ void put_t(const JvpParams& p, int64_t row, int k, int j, double x) {
  p.tangents[(row * 8 + k) * 12 + j] = (float)x;
}

// One side of an E-E pair, direction-independent part (manifold.hpp:245-256,
// 279-280): the trace, own normal and own value as Dual<3> functions of the
// body-frame witness pb0, then the opposing field's value and gradient at the
// world point (double). J5 = d pb5 / d pb0, Jn = d n_body / d pb0.
struct SideJac {
  double J5[9], Jn[9];
  double3 pb5, nb, pw, rel;  // rel = pw - t_other
  double3 gv;            // grad of the opposing phi at its body point
  double3 gown;          // d phi_own / d pb0 (containment)
  double vo, phi_own;
};

// Witness QP of a pair as a function of (Q11, Q12, Q22, c1, c2): primal
// alpha / gamma and their 3x5 Jacobian (witness.hpp:74-121).
struct QpRec {
  double a1, a2, gam;
  double J[15];
};

static_assert(sizeof(T12) == 56 && sizeof(SideJac) == 38 * 8 && sizeof(QpRec) == 18 * 8,
              "record sizes are mirrored by plan_jvp (host/api.cpp)");

struct EnvUnit {
  unsigned char* base;
  const JvpParams* p;
  int64_t env;
  __device__ Frame& frame(int s) const { return reinterpret_cast<Frame*>(base + p->o_frames)[s]; }
  __device__ T12* scores() const { return reinterpret_cast<T12*>(base + p->o_scores); }
  __device__ int* order() const { return reinterpret_cast<int*>(base + p->o_sorted); }
  __device__ T12* vslot(int i) const { return reinterpret_cast<T12*>(base + p->o_vslots) + 3 * i; }
  __device__ T12* eslot(int i) const { return reinterpret_cast<T12*>(base + p->o_eslots) + 12 * i; }
  __device__ int* prov() const { return reinterpret_cast<int*>(base + p->o_prov); }
  // per pair: dg, A1 = con pen1 clash cont, A2, dist1 + dist2
  __device__ T12* pair(int i) const { return reinterpret_cast<T12*>(base + p->o_pairs) + 4 * i; }
  __device__ SideJac& sj(int i, int s) const { return reinterpret_cast<SideJac*>(base + p->o_sj)[2 * i + s]; }
  __device__ QpRec& qrec(int i) const { return reinterpret_cast<QpRec*>(base + p->o_qp)[i]; }
  __device__ T12* vsdist() const { return reinterpret_cast<T12*>(base + p->o_vsdist); }
  __device__ T12* nnstat() const { return reinterpret_cast<T12*>(base + p->o_nnstat); }
};

template <int KS, int KO>
__device__ __forceinline__ void side_jac(const DevSdf& own, const DevSdf& oth, const Frame& Fs, const Frame& Fo,
                                         double3 pb0, const DevCfg& c, SideJac& r) {
  V3<D3> p = seed3(pb0);
#pragma unroll 1
  for (int k = 0; k < c.trace_iters; ++k) {
    const SdfOutT<D3> s = sdf_eval<kGrad, KS, D3>(own, p);
    p = p - dscale(normalize_smooth_t<D3>(s.g, c.tau_normal), s.v);
  }
  const SdfOutT<D3> o = c.containment ? sdf_eval<kNormalSource, KS, D3>(own, p)
                                      : sdf_eval<kNormalOnly, KS, D3>(own, p);
  const V3<D3> nb = normalize_smooth_t<D3>(o.g, c.tau_normal);
  r.pb5 = prim3(p);
  jac3(p, r.J5);
  r.nb = prim3(nb);
  jac3(nb, r.Jn);
  r.phi_own = o.v.v;
  r.gown = d3(o.v.d[0], o.v.d[1], o.v.d[2]);
  r.pw = fR(Fs, r.pb5) + ft(Fs);
  r.rel = r.pw - ft(Fo);
  const SdfOut v = sdf_eval<kGrad, KO>(oth, fRt(Fo, r.rel));
  r.vo = v.v;
  r.gv = v.g;
}

// Direction j of one side: world point / normal / opposing value / own value
// tangents from the body-frame witness tangent dpb0.
__device__ __forceinline__ void side_tan(const SideJac& r, const Frame& Fs, const Frame& Fo, double3 dpb0, int j,
                                         double3& dpw, double3& dn, double& dvo, double& dphi) {
  const double3 dpb5 = mv3(r.J5, dpb0);
  const double3 dnb = mv3(r.Jn, dpb0);
  dpw = fdR(Fs, r.pb5, j) + fR(Fs, dpb5) + fdt(Fs, j);
  dn = fdR(Fs, r.nb, j) + fR(Fs, dnb);
  const double3 dq = fdRt(Fo, r.rel, j) + fRt(Fo, dpw - fdt(Fo, j));
  dvo = ddot(r.gv, dq);
  dphi = ddot(r.gown, dpb0);
}

template <int K1, int K2>
__global__ void __launch_bounds__(kJvpThreads, kJvpMinBlocks) manifold_jvp_kernel(const __grid_constant__ JvpParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int upb = p.units_per_block;
  const int64_t u0 = (int64_t)blockIdx.x * upb;
  const ManifoldParams& m = p.m;
  const int n_here = (int)(m.n_env - u0 < upb ? m.n_env - u0 : upb);
  const int tid = threadIdx.x, nth = blockDim.x;
  const DevCfg& c = m.cfg;
  const DevSide& S1 = m.side[0];
  const DevSide& S2 = m.side[1];
  const int n1 = m.n1, n2 = m.n2, m1 = m.m1, m2 = m.m2, P = m1 * m2;
  const bool full = m1 > 0 && m2 > 0;
  const int C = m.n_contacts;
  auto unit = [&](int k) { return EnvUnit{smem + (size_t)k * p.bytes, &p, u0 + k}; };

  // ---- A: frames, se3_exp in Dual<6> seeded at the pose (dual.hpp:252-262) ----
  for (int it = tid; it < 2 * n_here; it += nth) {
    const EnvUnit u = unit(it >> 1);
    const int s = it & 1;
    const double* pose = s == 0 ? m.poses1 + m.pose_stride1 * u.env : m.poses2 + m.pose_stride2 * u.env;
    Dual<6> xi[6], R[9], t[3];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      xi[k] = Dual<6>(__ldg(pose + k));
      xi[k].d[k] = 1.0;
    }
    se3_exp_d(xi, R, t);
    Frame& F = u.frame(s);
    auto widen = [&](T12& o, const Dual<6>& x) {
      o.v = x.v;
#pragma unroll
      for (int j = 0; j < 12; ++j) o.d[j] = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) o.d[6 * s + j] = x.d[j];
    };
#pragma unroll
    for (int i = 0; i < 9; ++i) widen(F.R[i], R[i]);
#pragma unroll
    for (int i = 0; i < 3; ++i) widen(F.t[i], t[i]);
  }
  __syncthreads();

  const int off1 = S1.nv, off2 = S1.nv + S2.nv, off3 = off2 + S1.ne, off4 = off3 + S2.ne;
  const bool topk_any = S1.topk_v | S2.topk_v | S1.topk_e | S2.topk_e;
  if (topk_any) {
    // ---- B: vertex scores -phi_opp(vertex) (vertex_penetrations, 77-84) ----------
    for (int it = tid; it < n_here * off2; it += nth) {
      const int k = it / off2, i = it - k * off2;
      const EnvUnit u = unit(k);
      const int s = i < S1.nv ? 0 : 1;
      const int vi = s == 0 ? i : i - S1.nv;
      const Frame& Fs = u.frame(s);
      const Frame& Fo = u.frame(1 - s);
      const double3 v = dvert(s == 0 ? S1.verts : S2.verts, vi);
      const double3 rel = fR(Fs, v) + ft(Fs) - ft(Fo);
      const double3 q = fRt(Fo, rel);
      const SdfOut o = s == 0 ? sdf_eval<kGrad, K2>(S2.sdf, q) : sdf_eval<kGrad, K1>(S1.sdf, q);
      T12& sc = u.scores()[i];
      sc.v = -o.v;
#pragma unroll 1
      for (int j = 0; j < 12; ++j) {
        const double3 dpw = fdR(Fs, v, j) + fdt(Fs, j);
        const double3 dq = fdRt(Fo, rel, j) + fRt(Fo, dpw - fdt(Fo, j));
        sc.d[j] = -ddot(o.g, dq);
      }
    }
    __syncthreads();
    // edge scores: -(mean of endpoint penetrations) (edge_penetrations, 86-94)
    const int ne_all = S1.ne + S2.ne;
    for (int it = tid; it < n_here * ne_all * 13; it += nth) {
      const int k = it / (ne_all * 13), r = it - k * ne_all * 13;
      const int i = r / 13, j = r - (r / 13) * 13;  // j = 12: primal
      const EnvUnit u = unit(k);
      const int s = i < S1.ne ? 0 : 1;
      const int ei = s == 0 ? i : i - S1.ne;
      const int32_t* E = s == 0 ? S1.edges : S2.edges;
      const int voff = s == 0 ? 0 : S1.nv;
      T12* sc = u.scores();
      const T12& A = sc[voff + __ldg(E + 2 * ei)];
      const T12& B = sc[voff + __ldg(E + 2 * ei + 1)];
      if (j == 12) sc[off2 + i].v = -((-A.v + -B.v) * 0.5);
      else sc[off2 + i].d[j] = -((-A.d[j] + -B.d[j]) * 0.5);
    }
    __syncthreads();
    // ---- C: descending rank sort on primals, stable on ties -------------------
    for (int it = tid; it < n_here * off4; it += nth) {
      const int k = it / off4, i = it - k * off4;
      const EnvUnit u = unit(k);
      const int set = i < off1 ? 0 : i < off2 ? 1 : i < off3 ? 2 : 3;
      const bool active = set == 0 ? S1.topk_v : set == 1 ? S2.topk_v : set == 2 ? S1.topk_e : S2.topk_e;
      if (!active) continue;
      const int lo = set == 0 ? 0 : set == 1 ? off1 : set == 2 ? off2 : off3;
      const int hi = set == 0 ? off1 : set == 1 ? off2 : set == 2 ? off3 : off4;
      const T12* sc = u.scores();
      const double x = sc[i].v;
      int rank = 0;
      for (int j = lo; j < hi; ++j) {
        const double y = sc[j].v;
        rank += (y > x) || (y == x && j < i);
      }
      u.order()[lo + rank] = i;
    }
    __syncthreads();
  }

  // ---- D: selected slots, one item per (slot, direction | primal) -------------
  {
    const int nsl = n1 + n2 + m1 + m2;
    for (int it = tid; it < n_here * nsl * 13; it += nth) {
      const int k = it / (nsl * 13), rr = it - k * nsl * 13;
      const int r0 = rr / 13, j = rr - (rr / 13) * 13;  // j = 12: primal
      const EnvUnit u = unit(k);
      const bool is_edge = r0 >= n1 + n2;
      const int s = is_edge ? (r0 - n1 - n2 < m1 ? 0 : 1) : (r0 < n1 ? 0 : 1);
      const int r = is_edge ? (s == 0 ? r0 - n1 - n2 : r0 - n1 - n2 - m1) : (s == 0 ? r0 : r0 - n1);
      const DevSide& S = s == 0 ? S1 : S2;
      const bool sel = is_edge ? S.topk_e : S.topk_v;
      double3 a, b = d3(0, 0, 0), da = d3(0, 0, 0), db = d3(0, 0, 0);
      int prov = r;
      if (!sel) {  // K == D pass-through (manifold.hpp:135-140, 158-167): constant body points
        if (is_edge) {
          a = dvert(S.verts, __ldg(S.edges + 2 * r));
          b = dvert(S.verts, __ldg(S.edges + 2 * r + 1));
        } else {
          a = dvert(S.verts, r);
        }
      } else {  // soft top-K row r (smooth_ops.hpp:186-196; manifold.hpp:141-148, 168-180)
        const int set = (is_edge ? 2 : 0) + s;
        const int lo = set == 0 ? 0 : set == 1 ? off1 : set == 2 ? off2 : off3;
        const int hi = set == 0 ? off1 : set == 1 ? off2 : set == 2 ? off3 : off4;
        const T12* x = u.scores() + lo;
        const int D = hi - lo;
        const T12& sr = u.scores()[u.order()[lo + r]];
        const double inv_tau = is_edge ? c.inv_tau_topk_e : c.inv_tau_topk_v;
        const double srd = j < 12 ? sr.d[j] : 0.0;
        // argmin_s shift: the first minimal distance, with its tangent (smooth_ops.hpp:130-136)
        int imin = 0;
        double dmin = fabs(sr.v - x[0].v);
        for (int i = 1; i < D; ++i) {
          const double di = fabs(sr.v - x[i].v);
          if (di < dmin) { dmin = di; imin = i; }
        }
        auto sgn = [](double z) { return z < 0.0 ? -1.0 : (z > 0.0 ? 1.0 : 0.0); };
        const double dm = j < 12 ? sgn(sr.v - x[imin].v) * (srd - x[imin].d[j]) : 0.0;
        // weights w_i = e_i / tot, e_i = exp((m - |s_r - x_i|) / tau); one pass:
        //   a = S_v / tot,  da = (S_uv - (T / tot) S_v) / tot,  T = sum e_i u_i
        double tot = 0.0, T = 0.0;
        double3 Sa = d3(0, 0, 0), Sb = Sa, Sua = Sa, Sub = Sa;
        prov = -1;
        for (int i = 0; i < D; ++i) {
          const double z = sr.v - x[i].v;
          const double dist = fabs(z);
          if (prov < 0 && dist == 0.0) prov = i;
          const double e = exp_d((dmin - dist) * inv_tau);
          const double uu = j < 12 ? (dm - sgn(z) * (srd - x[i].d[j])) * inv_tau : 0.0;
          tot += e;
          T = fma(e, uu, T);
          const double eu = e * uu;
          double3 va, vb = d3(0, 0, 0);
          if (is_edge) {
            va = dvert(S.verts, __ldg(S.edges + 2 * i));
            vb = dvert(S.verts, __ldg(S.edges + 2 * i + 1));
          } else {
            va = dvert(S.verts, i);
          }
          Sa = Sa + va * e;
          Sua = Sua + va * eu;
          if (is_edge) {
            Sb = Sb + vb * e;
            Sub = Sub + vb * eu;
          }
        }
        const double inv = rcp_d(tot), Tn = T * inv;
        a = Sa * inv;
        b = Sb * inv;
        da = (Sua - Sa * Tn) * inv;
        db = (Sub - Sb * Tn) * inv;
      }
      const Frame& F = u.frame(s);
      if (j == 12) {
        u.prov()[r0] = prov;
        if (is_edge) {
          T12* q = u.eslot(r0 - n1 - n2);
          put3(q, fR(F, a) + ft(F));
          put3(q + 3, fR(F, b) + ft(F));
          put3(q + 6, a);
          put3(q + 9, b);
        } else {
          put3(u.vslot(r0), fR(F, a) + ft(F));
        }
      } else {
        const double3 daw = fdR(F, a, j) + fR(F, da) + fdt(F, j);
        if (is_edge) {
          T12* q = u.eslot(r0 - n1 - n2);
          put3d(q, daw, j);
          put3d(q + 3, fdR(F, b, j) + fR(F, db) + fdt(F, j), j);
          put3d(q + 6, da, j);
          put3d(q + 9, db, j);
        } else {
          put3d(u.vslot(r0), daw, j);
        }
      }
    }
  }
  __syncthreads();

  // ---- E1: one item per pair SIDE (side-major order: warps are side-uniform,
  // so the two SDF kinds never diverge inside a warp) -------------------------
  // Side 0 also carries the witness QP in Dual<5> (its Jacobian is the pair's);
  // side 1 needs only its primal alpha (bit-identical primal arithmetic).
  const int NP = full ? n_here * P : 0;
  for (int it = tid; it < 2 * NP; it += nth) {
    const int s = it >= NP ? 1 : 0;
    const int pi = it - s * NP;
    const int ku = pi / P, i = pi - ku * P;
    const EnvUnit u = unit(ku);
    const int k = i / m2, l = i - (i / m2) * m2;
    const T12* s1 = u.eslot(k);
    const T12* s2 = u.eslot(m1 + l);
    // ee_witness (witness.hpp:137-158) on the world edges
    const double3 t1 = val3(s1 + 3) - val3(s1), t2n = val3(s2) - val3(s2 + 3), bv = val3(s1) - val3(s2);
    const double q1 = ddot(t1, t1) + c.lambda, q2 = ddot(t1, t2n), q3 = ddot(t2n, t2n) + c.lambda;
    const double c1 = ddot(bv, t1) - 0.5 * c.lambda, c2 = ddot(bv, t2n) - 0.5 * c.lambda;
    double al;
    if (s == 0) {
      Dual<5> in[5] = {Dual<5>(q1), Dual<5>(q2), Dual<5>(q3), Dual<5>(c1), Dual<5>(c2)};
#pragma unroll
      for (int q = 0; q < 5; ++q) in[q].d[q] = 1.0;
      const QpSolT<Dual<5>> w = solve_box_qp_2<Dual<5>>(in[0], in[1], in[2], in[3], in[4], c);
      QpRec& qr = u.qrec(i);
      qr.a1 = w.a1.v;
      qr.a2 = w.a2.v;
      qr.gam = w.gamma.v;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        qr.J[q] = w.a1.d[q];
        qr.J[5 + q] = w.a2.d[q];
        qr.J[10 + q] = w.gamma.d[q];
      }
      al = w.a1.v;
    } else {
      al = solve_box_qp_2<double>(q1, q2, q3, c1, c2, c).a2;
    }
    // edge_point (witness.hpp:130-133) on the body-frame endpoints of this side
    const T12* se = s == 0 ? s1 : s2;
    const double3 pb0 = val3(se + 6) + (val3(se + 9) - val3(se + 6)) * al;
    if constexpr (K1 == K2) {
      side_jac<K1, K1>(m.side[s].sdf, m.side[1 - s].sdf, u.frame(s), u.frame(1 - s), pb0, c, u.sj(i, s));
    } else {
      if (s == 0) side_jac<K1, K2>(S1.sdf, S2.sdf, u.frame(0), u.frame(1), pb0, c, u.sj(i, 0));
      else side_jac<K2, K1>(S2.sdf, S1.sdf, u.frame(1), u.frame(0), pb0, c, u.sj(i, 1));
    }
  }
  __syncthreads();

  // ---- E2: V-S items, then one item per (pair, half of the 12 directions) ------
  {
    const int nvs = n1 + n2, NV = n_here * nvs;
    for (int it = tid; it < NV + 2 * NP; it += nth) {
      if (it < NV) {
        const int k = it / nvs, r = it - k * nvs;
        const EnvUnit u = unit(k);
        const bool first = r < n1;
        const Frame& Fo = u.frame(first ? 1 : 0);
        const T12* q = u.vslot(r);
        const double3 pw = val3(q);
        const double3 rel = pw - ft(Fo);
        // vs_contacts (manifold.hpp:185-204): normal source of the opposing field,
        // Dual<3> in its body point
        const V3<D3> xb = seed3(fRt(Fo, rel));
        const SdfOutT<D3> sv = first ? sdf_eval<kNormalSource, K2, D3>(S2.sdf, xb)
                                     : sdf_eval<kNormalSource, K1, D3>(S1.sdf, xb);
        const V3<D3> nbd = normalize_smooth_t<D3>(sv.g, c.tau_normal);
        double Jn[9];
        jac3(nbd, Jn);
        const double3 nb = prim3(nbd);
        const double3 gv = d3(sv.v.d[0], sv.v.d[1], sv.v.d[2]);
        double act, cact;
        sigmoid_pair_d(-sv.v.v * c.inv_tau_pen, &act, &cact);
        const double3 n = fR(Fo, nb);
        const int64_t row = u.env * C + r;
        float* dst = m.contacts + row * 8;
        dst[0] = (float)pw.x; dst[1] = (float)pw.y; dst[2] = (float)pw.z; dst[3] = (float)sv.v.v;
        dst[4] = (float)n.x; dst[5] = (float)n.y; dst[6] = (float)n.z; dst[7] = (float)act;
        if (m.src) {
          m.src[row * 2] = u.prov()[r];
          m.src[row * 2 + 1] = -1;
        }
        T12& vd = u.vsdist()[r];
        vd.v = sv.v.v;
        const double sact = -act * cact * c.inv_tau_pen;
#pragma unroll 1
        for (int j = 0; j < 12; ++j) {
          const double3 dpw = tan3(q, j);
          const double3 dx = fdRt(Fo, rel, j) + fRt(Fo, dpw - fdt(Fo, j));
          const double dv = ddot(gv, dx);
          const double3 dn = fdR(Fo, nb, j) + fR(Fo, mv3(Jn, dx));
          vd.d[j] = dv;
          put_t(p, row, 0, j, dpw.x);
          put_t(p, row, 1, j, dpw.y);
          put_t(p, row, 2, j, dpw.z);
          put_t(p, row, 3, j, dv);
          put_t(p, row, 4, j, dn.x);
          put_t(p, row, 5, j, dn.y);
          put_t(p, row, 6, j, dn.z);
          put_t(p, row, 7, j, sact * dv);
        }
        continue;
      }
      const int qi = it - NV, h = qi & 1, pi = qi >> 1;
      const int ku = pi / P, i = pi - ku * P;
      const EnvUnit u = unit(ku);
      const int k = i / m2, l = i - (i / m2) * m2;
      const T12* s1 = u.eslot(k);
      const T12* s2 = u.eslot(m1 + l);
      const Frame& F1 = u.frame(0);
      const Frame& F2 = u.frame(1);
      const QpRec& qr = u.qrec(i);
      const SideJac& r1 = u.sj(i, 0);
      const SideJac& r2 = u.sj(i, 1);
      const double al1 = qr.a1, al2 = qr.a2, gam = qr.gam;
      const double3 t1 = val3(s1 + 3) - val3(s1), t2n = val3(s2) - val3(s2 + 3), bv = val3(s1) - val3(s2);
      const double3 e1 = val3(s1 + 9) - val3(s1 + 6), e2 = val3(s2 + 9) - val3(s2 + 6);
      // E3: pair quantities (manifold.hpp:248-266, 279-285), FP64
      const double3 p1w = r1.pw, p2w = r2.pw;
      const double3 nw1 = fR(F1, r1.nb), nw2 = fR(F2, r2.nb);
      const double3 de = p1w - p2w;
      const double dg = sqrt(ddot(de, de) + 1e-12);  // kEdgeNormalEps
      const double idg = rcp_d(dg);
      const double3 nbar = de * idg;
      const double g1 = tanh(ddot(nw2, nbar) * c.inv_tau_sign);
      const double g2 = tanh(ddot(nw1, nbar) * c.inv_tau_sign);
      double pen1, cpen1, pen2, cpen2, cl, ccl, ct1 = 1.0, cct1 = 0.0, ct2 = 1.0, cct2 = 0.0;
      sigmoid_pair_d(-r1.vo * c.inv_tau_pen, &pen1, &cpen1);
      sigmoid_pair_d(-r2.vo * c.inv_tau_pen, &pen2, &cpen2);
      sigmoid_pair_d(-ddot(nw1, nw2) * c.inv_tau_clash, &cl, &ccl);
      if (c.containment) {
        sigmoid_pair_d(-r1.phi_own * c.inv_tau_cont, &ct1, &cct1);
        sigmoid_pair_d(-r2.phi_own * c.inv_tau_cont, &ct2, &cct2);
      }
      const double cont = ct1 * ct2;
      const double base = gam * cl * cont;
      const int64_t row = u.env * C + n1 + n2 + 2 * i;
      T12* rec = u.pair(i);
      if (h == 0) {
        float* dst = m.contacts + row * 8;
        const double3 o1 = nbar * g1, o2 = nbar * g2;
        dst[0] = (float)p1w.x; dst[1] = (float)p1w.y; dst[2] = (float)p1w.z; dst[3] = (float)(g1 * dg);
        dst[4] = (float)o1.x; dst[5] = (float)o1.y; dst[6] = (float)o1.z;
        dst[8] = (float)p2w.x; dst[9] = (float)p2w.y; dst[10] = (float)p2w.z; dst[11] = (float)(g2 * dg);
        dst[12] = (float)o2.x; dst[13] = (float)o2.y; dst[14] = (float)o2.z;
        if (m.src) {
          int* sp = m.src + row * 2;
          const int sa = u.prov()[n1 + n2 + k], sb = u.prov()[n1 + n2 + m1 + l];
          sp[0] = sa; sp[1] = sb; sp[2] = sa; sp[3] = sb;
        }
        rec[0].v = dg;
        rec[1].v = base * pen1;
        rec[2].v = base * pen2;
        rec[3].v = g1 * dg + g2 * dg;
      }
      const double k1 = (1.0 - g1 * g1) * c.inv_tau_sign, k2 = (1.0 - g2 * g2) * c.inv_tau_sign;
#pragma unroll 1
      for (int j = 6 * h; j < 6 * h + 6; ++j) {
        // QP inputs -> alpha, gamma tangents
        const double3 dt1 = tan3(s1 + 3, j) - tan3(s1, j), dt2n = tan3(s2, j) - tan3(s2 + 3, j);
        const double3 dbv = tan3(s1, j) - tan3(s2, j);
        const double dq[5] = {2.0 * ddot(t1, dt1), ddot(dt1, t2n) + ddot(t1, dt2n), 2.0 * ddot(t2n, dt2n),
                              ddot(dbv, t1) + ddot(bv, dt1), ddot(dbv, t2n) + ddot(bv, dt2n)};
        double da1 = 0.0, da2 = 0.0, dgam = 0.0;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          da1 = fma(qr.J[q], dq[q], da1);
          da2 = fma(qr.J[5 + q], dq[q], da2);
          dgam = fma(qr.J[10 + q], dq[q], dgam);
        }
        const double3 dpb1 = tan3(s1 + 6, j) + (tan3(s1 + 9, j) - tan3(s1 + 6, j)) * al1 + e1 * da1;
        const double3 dpb2 = tan3(s2 + 6, j) + (tan3(s2 + 9, j) - tan3(s2 + 6, j)) * al2 + e2 * da2;
        double3 dp1, dn1, dp2, dn2;
        double dvo1, dph1, dvo2, dph2;
        side_tan(r1, F1, F2, dpb1, j, dp1, dn1, dvo1, dph1);
        side_tan(r2, F2, F1, dpb2, j, dp2, dn2, dvo2, dph2);
        const double3 dde = dp1 - dp2;
        const double ddg = ddot(nbar, dde);
        const double3 dnbar = (dde - nbar * ddg) * idg;
        const double dg1 = k1 * (ddot(dn2, nbar) + ddot(nw2, dnbar));
        const double dg2 = k2 * (ddot(dn1, nbar) + ddot(nw1, dnbar));
        const double dpen1 = -pen1 * cpen1 * c.inv_tau_pen * dvo1;
        const double dpen2 = -pen2 * cpen2 * c.inv_tau_pen * dvo2;
        const double dcl = -cl * ccl * c.inv_tau_clash * (ddot(dn1, nw2) + ddot(nw1, dn2));
        const double dcont = c.containment ? -c.inv_tau_cont * (ct1 * cct1 * dph1 * ct2 + ct1 * ct2 * cct2 * dph2) : 0.0;
        const double dbase = (dgam * cl + gam * dcl) * cont + gam * cl * dcont;
        const double dd1 = dg1 * dg + g1 * ddg, dd2 = dg2 * dg + g2 * ddg;
        rec[0].d[j] = ddg;
        rec[1].d[j] = dbase * pen1 + base * dpen1;
        rec[2].d[j] = dbase * pen2 + base * dpen2;
        rec[3].d[j] = dd1 + dd2;
        const double3 dm1 = nbar * dg1 + dnbar * g1, dm2 = nbar * dg2 + dnbar * g2;
        put_t(p, row, 0, j, dp1.x);
        put_t(p, row, 1, j, dp1.y);
        put_t(p, row, 2, j, dp1.z);
        put_t(p, row, 3, j, dd1);
        put_t(p, row, 4, j, dm1.x);
        put_t(p, row, 5, j, dm1.y);
        put_t(p, row, 6, j, dm1.z);
        put_t(p, row + 1, 0, j, dp2.x);
        put_t(p, row + 1, 1, j, dp2.y);
        put_t(p, row + 1, 2, j, dp2.z);
        put_t(p, row + 1, 3, j, dd2);
        put_t(p, row + 1, 4, j, dm2.x);
        put_t(p, row + 1, 5, j, dm2.y);
        put_t(p, row + 1, 6, j, dm2.z);
      }
    }
  }
  __syncthreads();

  if (full) {
    // ---- F: NN softmin statistics, shift = first minimum (argmin_s 126-144) ----
    const int nrc = m1 + m2;
    for (int it = tid; it < n_here * nrc * 13; it += nth) {
      const int ku = it / (nrc * 13), rr = it - ku * nrc * 13;
      const int r = rr / 13, j = rr - (rr / 13) * 13;  // j = 12: primal
      const EnvUnit u = unit(ku);
      const bool row = r < m1;
      const int n = row ? m2 : m1;
      auto dgv = [&](int q) -> const T12& { return u.pair(row ? r * m2 + q : q * m2 + (r - m1))[0]; };
      int jm = 0;
      for (int q = 1; q < n; ++q)
        if (dgv(q).v < dgv(jm).v) jm = q;
      const double mn = dgv(jm).v;
      const double dmn = j < 12 ? dgv(jm).d[j] : 0.0;
      double tot = 0.0, dtot = 0.0;
      for (int q = 0; q < n; ++q) {
        const T12& x = dgv(q);
        const double e = exp_d((mn - x.v) * c.inv_tau_nn);
        tot += e;
        if (j < 12) dtot = fma(e, (dmn - x.d[j]) * c.inv_tau_nn, dtot);
      }
      const double inv = rcp_d(tot);
      T12* ns = u.nnstat() + 2 * r;
      if (j == 12) {
        ns[0].v = mn;
        ns[1].v = inv;
      } else {
        ns[0].d[j] = dmn;
        ns[1].d[j] = -inv * inv * dtot;
      }
    }
    __syncthreads();
    // ---- G: activity = con pen_b nn_b clash cont (manifold.hpp:303-330) -------
    for (int it = tid; it < n_here * P; it += nth) {
      const int ku = it / P, i = it - ku * P;
      const EnvUnit u = unit(ku);
      const int k = i / m2, l = i - (i / m2) * m2;
      const T12* rec = u.pair(i);
      const T12* na = u.nnstat() + 2 * k;
      const T12* nb = u.nnstat() + 2 * (m1 + l);
      const double dg = rec[0].v;
      const double e1 = exp_d((na[0].v - dg) * c.inv_tau_nn), e2 = exp_d((nb[0].v - dg) * c.inv_tau_nn);
      const double nn1 = e1 * na[1].v, nn2 = e2 * nb[1].v;
      const int64_t row = u.env * C + n1 + n2 + 2 * i;
      m.contacts[row * 8 + 7] = (float)(rec[1].v * nn1);
      m.contacts[row * 8 + 15] = (float)(rec[2].v * nn2);
#pragma unroll 1
      for (int j = 0; j < 12; ++j) {
        const double dnn1 = fma(e1 * (na[0].d[j] - rec[0].d[j]) * c.inv_tau_nn, na[1].v, e1 * na[1].d[j]);
        const double dnn2 = fma(e2 * (nb[0].d[j] - rec[0].d[j]) * c.inv_tau_nn, nb[1].v, e2 * nb[1].d[j]);
        put_t(p, row, 7, j, rec[1].d[j] * nn1 + rec[1].v * dnn1);
        put_t(p, row + 1, 7, j, rec[2].d[j] * nn2 + rec[2].v * dnn2);
      }
    }
  }
  __syncthreads();

  // ---- H: mean contact distance (manifold.hpp:379-384), fixed order ---------
  if (m.mean_dist || p.mean_grad || p.mean_f64 || p.mean_grad_f64) {
    for (int it = tid; it < n_here * 13; it += nth) {
      const int k = it / 13, j = it - k * 13;  // j = 12: primal
      const EnvUnit u = unit(k);
      double acc = 0.0;
      for (int r = 0; r < n1 + n2; ++r) acc += j < 12 ? u.vsdist()[r].d[j] : u.vsdist()[r].v;
      for (int i = 0; i < P && full; ++i) acc += j < 12 ? u.pair(i)[3].d[j] : u.pair(i)[3].v;
      const double mean = acc * (1.0 / (double)C);
      if (j == 12) {
        if (m.mean_dist) m.mean_dist[u.env] = (float)mean;
        if (p.mean_f64) p.mean_f64[u.env] = mean;
      } else {
        if (p.mean_grad) p.mean_grad[u.env * 12 + j] = (float)mean;
        if (p.mean_grad_f64) p.mean_grad_f64[u.env * 12 + j] = mean;
      }
    }
  }
}

template <int K1, int K2>
int launch_jvp_kind(const JvpParams& p, int threads, cudaStream_t s) {
  static PerDeviceOnce configured;
  configured([] {  // per device: the attribute does not carry across devices
    cudaFuncSetAttribute(manifold_jvp_kernel<K1, K2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  const int64_t grid = (p.m.n_env + p.units_per_block - 1) / p.units_per_block;
  manifold_jvp_kernel<K1, K2><<<(unsigned)grid, threads, (size_t)p.bytes * p.units_per_block, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// SQ kinds share the runtime-exponent path (kSqE01 -> kSingleSq), box_planes
// the general CP leaf: one instantiation per shape class keeps the library small.
constexpr int jvp_kind(int k) { return k == kSqE01 ? kSingleSq : (k == kBoxCp ? kSingleCp : k); }

template <int K1>
int launch_jvp_k2(const JvpParams& p, int threads, cudaStream_t s) {
  switch (jvp_kind(p.m.side[1].sdf.kind)) {
    case kSingleSq: return launch_jvp_kind<K1, kSingleSq>(p, threads, s);
    case kSingleCp: return launch_jvp_kind<K1, kSingleCp>(p, threads, s);
    default: return launch_jvp_kind<K1, kGeneric>(p, threads, s);
  }
}

}  // namespace

int jvp_directions() { return 12; }
int jvp_max_threads() { return kJvpThreads; }
int jvp_smem_cap() { return CMGB_JVP_SMEM_KB * 1024; }

int launch_manifold_jvp(const JvpParams& p, int block_threads, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int threads = block_threads > 0 && block_threads <= kJvpThreads ? block_threads : kJvpThreads;
  switch (jvp_kind(p.m.side[0].sdf.kind)) {
    case kSingleSq: return launch_jvp_k2<kSingleSq>(p, threads, s);
    case kSingleCp: return launch_jvp_k2<kSingleCp>(p, threads, s);
    default: return launch_jvp_k2<kGeneric>(p, threads, s);
  }
}

}  // namespace cmgb
