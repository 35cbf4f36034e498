// Forward-mode pose Jacobian of the batched contact manifold:
//   generate_manifold<Dual12> seeded by seed_pose_tangents (dual.hpp:249-263)
//   and mean_contact_distance (manifold.hpp:379-384), for every env.
//
// The reference runs the whole pipeline once in Dual<12> arithmetic. Here one
// CTA owns one (env, direction group): it evaluates the same pipeline as
// manifold.cu in Dual<ND> arithmetic (dual.cuh; ND tangent directions of the
// 12), so 12 / ND CTAs cover an env. The primal is recomputed per group -- on
// the B200 that is cheaper than a 13-double scalar, which would not fit in
// registers. Every routine is the templated FP64 code of the value kernel
// (sdf.cuh, witness.cuh, dmath.cuh) with T = Dual<ND>; the FP32 indicator
// shortcuts of the value kernel (tanhf / expf sigmoids, NN weights) are FP64
// here because their tangents carry 1/tau amplification.
//
// Semantics that touch tangents (all as in the reference):
//   - soft top-K: hard sort on primals; ties between equal scores keep the
//     stable (index) order, which is what libstdc++'s std::sort does for the
//     D <= 16 candidate sets of the tested meshes (smooth_ops.hpp:180-185);
//   - argmin / LSE shift elements carry their tangents (smooth_ops.hpp:95-144);
//   - fabs has subgradient 0 at the kink (dual.hpp:236-246);
//   - the spatial gradient inside the sphere trace / normals is the analytic
//     gradient expression differentiated again (the reference nests
//     Dual<3, Dual12>, sdf.hpp:183-190).
// hard_ops is rejected by the host (the reference's hard mode is double-only,
// smooth_ops.hpp:199).
//
// Outputs: contacts (primal, FP32, group 0), tangents [n_env][C][8][12] FP32,
// mean_dist (group 0) and its 12 tangents.
#include <cuda_runtime.h>

#include "../common.h"
#include "launch_util.cuh"
#include "../device/dmath.cuh"
#include "../device/dual.cuh"
#include "../device/sdf.cuh"
#include "../device/witness.cuh"

namespace cmgb {

namespace {

// Tangent directions per thread (12 / ND groups), CTA size and CTAs per SM;
// overridable at build time for tuning (tools/jvp_variants.sh).
#ifndef CMGB_JVP_ND
#define CMGB_JVP_ND 2
#endif
#ifndef CMGB_JVP_THREADS
#define CMGB_JVP_THREADS 128
#endif
#ifndef CMGB_JVP_MINB
#define CMGB_JVP_MINB 4
#endif
#ifndef CMGB_JVP_SMEM_KB
#define CMGB_JVP_SMEM_KB 56
#endif
constexpr int kJvpND = CMGB_JVP_ND;
constexpr int kJvpThreads = CMGB_JVP_THREADS;
constexpr int kJvpMinBlocks = CMGB_JVP_MINB;
static_assert(12 % kJvpND == 0, "ND must divide the 12 pose directions");

template <class T>
struct Frame {
  T R[9];
  T t[3];
};

template <class T>
__device__ __forceinline__ vec3<T> to_world_t(const Frame<T>& f, const vec3<T>& pb) {
  return mul_R(f.R, pb) + mk3<T>(f.t[0], f.t[1], f.t[2]);
}
template <class T>
__device__ __forceinline__ vec3<T> to_body_t(const Frame<T>& f, const vec3<T>& pw) {
  return mul_Rt(f.R, pw - mk3<T>(f.t[0], f.t[1], f.t[2]));
}
template <class T>
__device__ __forceinline__ vec3<T> normalize_smooth_t(const vec3<T>& v, double tau) {
  return dscale(v, rsqrt_d(tau + ddot(v, v)));
}
template <class T>
__device__ __forceinline__ vec3<T> dvert(const double* v, int i) {
  return mk3<T>(__ldg(v + 3 * i), __ldg(v + 3 * i + 1), __ldg(v + 3 * i + 2));
}

template <int ND>
struct Unit {
  using T = Dual<ND>;
  unsigned char* base;
  const JvpParams* p;
  int64_t env;
  int group;
  __device__ Frame<T>& frame(int s) const { return reinterpret_cast<Frame<T>*>(base + p->o_frames)[s]; }
  __device__ T* scores() const { return reinterpret_cast<T*>(base + p->o_scores); }
  __device__ T* sorted() const { return reinterpret_cast<T*>(base + p->o_sorted); }
  __device__ T* vslot(int i) const { return reinterpret_cast<T*>(base + p->o_vslots) + 3 * i; }
  __device__ T* eslot(int i) const { return reinterpret_cast<T*>(base + p->o_eslots) + 12 * i; }
  __device__ int* prov() const { return reinterpret_cast<int*>(base + p->o_prov); }
  __device__ T* pair(int i) const { return reinterpret_cast<T*>(base + p->o_pairs) + (kPairRec / 2) * i; }
  __device__ T* vsdist() const { return reinterpret_cast<T*>(base + p->o_vsdist); }
  __device__ T* nnstat() const { return reinterpret_cast<T*>(base + p->o_nnstat); }
};

// Output of one scalar of contact row `row`, field k: primal (group 0) and the
// group's ND tangent entries.
template <int ND>
__device__ __forceinline__ void put(const JvpParams& p, int group, int64_t row, int k, const Dual<ND>& x) {
  if (group == 0) p.m.contacts[row * 8 + k] = (float)x.v;
  float* t = p.tangents + (row * 8 + k) * 12 + group * ND;
#pragma unroll
  for (int j = 0; j < ND; ++j) t[j] = (float)x.d[j];
}

template <int ND>
__device__ __forceinline__ void put_contact(const JvpParams& p, int group, int64_t row,
                                            const vec3<Dual<ND>>& pt, const Dual<ND>& dist,
                                            const vec3<Dual<ND>>& n, const Dual<ND>& act) {
  put(p, group, row, 0, pt.x);
  put(p, group, row, 1, pt.y);
  put(p, group, row, 2, pt.z);
  put(p, group, row, 3, dist);
  put(p, group, row, 4, n.x);
  put(p, group, row, 5, n.y);
  put(p, group, row, 6, n.z);
  put(p, group, row, 7, act);
}

template <int K, class T>
__device__ __forceinline__ vec3<T> trace_t(const DevSdf& sdf, vec3<T> p, const DevCfg& c) {
#pragma unroll 1
  for (int k = 0; k < c.trace_iters; ++k) {
    const SdfOutT<T> s = sdf_eval<kGrad, K, T>(sdf, p);
    p = p - dscale(normalize_smooth_t<T>(s.g, c.tau_normal), s.v);
  }
  return p;
}

// One side of an E-E pair (manifold.hpp:245-256, 279-280); record layout as
// in manifold.cu (side s at 8 s: world point, own normal, phi_other, phi_own).
template <int KS, int KO, int ND>
__device__ __forceinline__ void side_t(const JvpParams& p, const Unit<ND>& u, int s, Dual<ND>* r) {
  using T = Dual<ND>;
  const DevCfg& c = p.m.cfg;
  const DevSdf& own = p.m.side[s].sdf;
  const DevSdf& oth = p.m.side[1 - s].sdf;
  vec3<T> pb = mk3<T>(r[0], r[1], r[2]);
  if (c.trace_iters > 0) pb = trace_t<KS, T>(own, pb, c);
  const SdfOutT<T> o = sdf_eval<kNormalSource, KS, T>(own, pb);
  const Frame<T>& F = u.frame(s);
  const vec3<T> n = mul_R(F.R, normalize_smooth_t<T>(o.g, c.tau_normal));
  const vec3<T> pw = to_world_t(F, pb);
  const T v_oth = sdf_eval<kValue, KO, T>(oth, to_body_t(u.frame(1 - s), pw)).v;
  r[0] = pw.x; r[1] = pw.y; r[2] = pw.z;
  r[3] = n.x; r[4] = n.y; r[5] = n.z;
  r[6] = v_oth;
  r[7] = o.v;
}

// A CTA owns `units_per_block` consecutive units; unit U = (env U / groups,
// direction group U % groups). Work items of all its units are spread over
// the CTA's threads, phase by phase (as manifold.cu does with envs).
template <int K1, int K2, int ND>
__global__ void __launch_bounds__(kJvpThreads, kJvpMinBlocks) manifold_jvp_kernel(const __grid_constant__ JvpParams p) {
  using T = Dual<ND>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int upb = p.units_per_block;
  const int64_t u0 = (int64_t)blockIdx.x * upb;
  const int64_t n_units = p.m.n_env * p.groups;
  const int n_here = (int)(n_units - u0 < upb ? n_units - u0 : upb);
  const int tid = threadIdx.x, nth = blockDim.x;
  const ManifoldParams& m = p.m;
  const DevCfg& c = m.cfg;
  const DevSide& S1 = m.side[0];
  const DevSide& S2 = m.side[1];
  const int n1 = m.n1, n2 = m.n2, m1 = m.m1, m2 = m.m2, P = m1 * m2;
  const bool full = m1 > 0 && m2 > 0;
  const int C = m.n_contacts;
  auto unit = [&](int k) {
    const int64_t U = u0 + k;
    return Unit<ND>{smem + (size_t)k * p.bytes, &p, U / p.groups, (int)(U % p.groups)};
  };

  // ---- A: poses seeded with the unit's tangent directions, se3_exp ---------
  // Direction d = group * ND + j tracks pose1[d] (d < 6) or pose2[d - 6].
  for (int it = tid; it < 2 * n_here; it += nth) {
    const Unit<ND> u = unit(it >> 1);
    const int s = it & 1;
    const double* pose = s == 0 ? m.poses1 + m.pose_stride1 * u.env : m.poses2 + m.pose_stride2 * u.env;
    T xi[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      xi[k] = T(__ldg(pose + k));
#pragma unroll
      for (int j = 0; j < ND; ++j) xi[k].d[j] = (u.group * ND + j == 6 * s + k) ? 1.0 : 0.0;
    }
    Frame<T>& F = u.frame(s);
    se3_exp_d(xi, F.R, F.t);
  }
  __syncthreads();

  const int off1 = S1.nv, off2 = S1.nv + S2.nv, off3 = off2 + S1.ne, off4 = off3 + S2.ne;
  const bool topk_any = S1.topk_v | S2.topk_v | S1.topk_e | S2.topk_e;
  if (topk_any) {
    // ---- B: scores (-penetration) of every vertex, then edges -------------
    for (int it = tid; it < n_here * off2; it += nth) {
      const int k = it / off2, i = it - k * off2;
      const Unit<ND> u = unit(k);
      const int s = i < S1.nv ? 0 : 1;
      const int vi = s == 0 ? i : i - S1.nv;
      const vec3<T> pw = to_world_t(u.frame(s), dvert<T>(s == 0 ? S1.verts : S2.verts, vi));
      const vec3<T> pb = to_body_t(u.frame(1 - s), pw);
      const T pen = s == 0 ? sdf_eval<kValue, K2, T>(S2.sdf, pb).v : sdf_eval<kValue, K1, T>(S1.sdf, pb).v;
      u.scores()[i] = -pen;
    }
    __syncthreads();
    const int ne_all = S1.ne + S2.ne;
    for (int it = tid; it < n_here * ne_all; it += nth) {
      const int k = it / ne_all, i = it - k * ne_all;
      const Unit<ND> u = unit(k);
      const int s = i < S1.ne ? 0 : 1;
      const int ei = s == 0 ? i : i - S1.ne;
      const int32_t* E = s == 0 ? S1.edges : S2.edges;
      const int voff = s == 0 ? 0 : S1.nv;
      T* sc = u.scores();
      const T pa = -sc[voff + __ldg(E + 2 * ei)], pb = -sc[voff + __ldg(E + 2 * ei + 1)];
      sc[off2 + i] = -((pa + pb) * 0.5);
    }
    __syncthreads();
    // ---- C: descending rank sort on primals, stable on ties -------------
    for (int it = tid; it < n_here * off4; it += nth) {
      const int k = it / off4, i = it - k * off4;
      const Unit<ND> u = unit(k);
      const int set = i < off1 ? 0 : i < off2 ? 1 : i < off3 ? 2 : 3;
      const bool active = set == 0 ? S1.topk_v : set == 1 ? S2.topk_v : set == 2 ? S1.topk_e : S2.topk_e;
      if (!active) continue;
      const int lo = set == 0 ? 0 : set == 1 ? off1 : set == 2 ? off2 : off3;
      const int hi = set == 0 ? off1 : set == 1 ? off2 : set == 2 ? off3 : off4;
      const T* sc = u.scores();
      const double x = sc[i].v;
      int rank = 0;
      for (int j = lo; j < hi; ++j) {
        const double y = sc[j].v;
        rank += (y > x) || (y == x && j < i);
      }
      u.sorted()[lo + rank] = sc[i];
    }
    __syncthreads();
  }

  // ---- D: selected slots (pass-through or soft top-K rows) ---------------
  {
    const int nsl = n1 + n2 + m1 + m2;
    for (int it = tid; it < n_here * nsl; it += nth) {
      const int k = it / nsl, r0 = it - k * nsl;
      const Unit<ND> u = unit(k);
      const bool is_edge = r0 >= n1 + n2;
      const int s = is_edge ? (r0 - n1 - n2 < m1 ? 0 : 1) : (r0 < n1 ? 0 : 1);
      const int r = is_edge ? (s == 0 ? r0 - n1 - n2 : r0 - n1 - n2 - m1) : (s == 0 ? r0 : r0 - n1);
      const DevSide& S = s == 0 ? S1 : S2;
      const bool sel = is_edge ? S.topk_e : S.topk_v;
      vec3<T> a = mk3<T>(0.0, 0.0, 0.0), b = a;
      int prov = r;
      if (!sel) {
        if (is_edge) {
          a = dvert<T>(S.verts, __ldg(S.edges + 2 * r));
          b = dvert<T>(S.verts, __ldg(S.edges + 2 * r + 1));
        } else {
          a = dvert<T>(S.verts, r);
        }
      } else {  // soft top-K row r: softmax(-|sorted_r - x| / tau) (smooth_ops.hpp:186-196)
        const int set = (is_edge ? 2 : 0) + s;
        const int lo = set == 0 ? 0 : set == 1 ? off1 : set == 2 ? off2 : off3;
        const int hi = set == 0 ? off1 : set == 1 ? off2 : set == 2 ? off3 : off4;
        const T* x = u.scores() + lo;
        const int D = hi - lo;
        const T sr = u.sorted()[lo + r];
        const double inv_tau = is_edge ? c.inv_tau_topk_e : c.inv_tau_topk_v;
        // argmin_s shift: the first minimal distance (value 0 at the row's own
        // element), carried as a full scalar (smooth_ops.hpp:130-136)
        int imin = 0;
        double dmin = fabs(sr.v - x[0].v);
        for (int i = 1; i < D; ++i) {
          const double di = fabs(sr.v - x[i].v);
          if (di < dmin) { dmin = di; imin = i; }
        }
        const T mshift = fabs(sr - x[imin]);
        T tot = 0.0;
        prov = -1;
        for (int i = 0; i < D; ++i) {
          const T dist = fabs(sr - x[i]);
          tot += exp((mshift - dist) * inv_tau);
          if (prov < 0 && dist.v == 0.0) prov = i;
        }
        const T inv = 1.0 / tot;
        for (int i = 0; i < D; ++i) {
          const T wi = exp((mshift - fabs(sr - x[i])) * inv_tau) * inv;
          if (is_edge) {
            a = a + dvert<T>(S.verts, __ldg(S.edges + 2 * i)) * wi;
            b = b + dvert<T>(S.verts, __ldg(S.edges + 2 * i + 1)) * wi;
          } else {
            a = a + dvert<T>(S.verts, i) * wi;
          }
        }
      }
      u.prov()[r0] = prov;
      const Frame<T>& F = u.frame(s);
      if (is_edge) {
        T* q = u.eslot(r0 - n1 - n2);
        const vec3<T> aw = to_world_t(F, a), bw = to_world_t(F, b);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
        q[3] = bw.x; q[4] = bw.y; q[5] = bw.z;
        q[6] = a.x; q[7] = a.y; q[8] = a.z;
        q[9] = b.x; q[10] = b.y; q[11] = b.z;
      } else {
        T* q = u.vslot(r0);
        const vec3<T> aw = to_world_t(F, a);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
      }
    }
  }
  __syncthreads();

  // ---- E: V-S contacts (vs_contacts, manifold.hpp:185-204), E-E pairs -----
  // V-S items start on the thread after the last pair item, so the two kinds
  // run side by side instead of V-S then pairs on the same threads.
  {
    const int nvs = n1 + n2;
    const int vs0 = full ? (n_here * P) % nth : 0;
    for (int it = tid >= vs0 ? tid - vs0 : tid - vs0 + nth; it < n_here * nvs; it += nth) {
      const int k = it / nvs, r = it - k * nvs;
      const Unit<ND> u = unit(k);
      const bool first = r < n1;
      const DevSdf& opp = first ? S2.sdf : S1.sdf;
      const Frame<T>& Fo = u.frame(first ? 1 : 0);
      const T* q = u.vslot(r);
      const vec3<T> pw = mk3<T>(q[0], q[1], q[2]);
      const SdfOutT<T> s = first ? sdf_eval<kNormalSource, K2, T>(opp, to_body_t(Fo, pw))
                                 : sdf_eval<kNormalSource, K1, T>(opp, to_body_t(Fo, pw));
      const vec3<T> n = mul_R(Fo.R, normalize_smooth_t<T>(s.g, c.tau_normal));
      const T act = sigmoid_d(-s.v * c.inv_tau_pen);
      u.vsdist()[r] = s.v;
      const int64_t row = u.env * C + r;
      put_contact<ND>(p, u.group, row, pw, s.v, n, act);
      if (u.group == 0 && m.src) {
        m.src[row * 2] = u.prov()[r];
        m.src[row * 2 + 1] = -1;
      }
    }
  }
  if (full) {
    for (int it = tid; it < n_here * P; it += nth) {
      const int ku = it / P, i = it - ku * P;
      const Unit<ND> u = unit(ku);
      const int k = i / m2, l = i - (i / m2) * m2;
      T* r = u.pair(i);
      // E1: witness QP (ee_witness, witness.hpp:137-158), body-frame points
      {
        const T* s1 = u.eslot(k);
        const T* s2 = u.eslot(m1 + l);
        const QpSolT<T> w = ee_qp<T>(mk3<T>(s1[0], s1[1], s1[2]), mk3<T>(s1[3], s1[4], s1[5]),
                                     mk3<T>(s2[0], s2[1], s2[2]), mk3<T>(s2[3], s2[4], s2[5]), c);
        r[0] = s1[6] + (s1[9] - s1[6]) * w.a1;
        r[1] = s1[7] + (s1[10] - s1[7]) * w.a1;
        r[2] = s1[8] + (s1[11] - s1[8]) * w.a1;
        r[8] = s2[6] + (s2[9] - s2[6]) * w.a2;
        r[9] = s2[7] + (s2[10] - s2[7]) * w.a2;
        r[10] = s2[8] + (s2[11] - s2[8]) * w.a2;
        r[16] = w.gamma;
      }
      // E2: both sides
      if constexpr (K1 == K2) {  // one code copy for both sides (I-cache)
#pragma unroll 1
        for (int s = 0; s < 2; ++s) side_t<K1, K1, ND>(p, u, s, r + 8 * s);
      } else {
        side_t<K1, K2, ND>(p, u, 0, r);
        side_t<K2, K1, ND>(p, u, 1, r + 8);
      }
      // E3: pair quantities (manifold.hpp:248-266, 279-285)
      const vec3<T> de = mk3<T>(r[0] - r[8], r[1] - r[9], r[2] - r[10]);
      const T dg = sqrt(ddot(de, de) + 1e-12);
      const vec3<T> nb = dscale(de, rcp_d(dg));
      const vec3<T> n1v = mk3<T>(r[3], r[4], r[5]), n2v = mk3<T>(r[11], r[12], r[13]);
      const T g1 = tanh(ddot(n2v, nb) * c.inv_tau_sign);
      const T g2 = tanh(ddot(n1v, nb) * c.inv_tau_sign);
      const T pen1 = sigmoid_d(-r[6] * c.inv_tau_pen);
      const T pen2 = sigmoid_d(-r[14] * c.inv_tau_pen);
      const T clash = sigmoid_d(-ddot(n1v, n2v) * c.inv_tau_clash);
      const T cont = c.containment ? sigmoid_d(-r[7] * c.inv_tau_cont) * sigmoid_d(-r[15] * c.inv_tau_cont)
                                   : T(1.0);
      r[3] = dg;
      r[4] = g1;
      r[5] = g2;
      r[11] = nb.x; r[12] = nb.y; r[13] = nb.z;
      r[6] = pen1;
      r[14] = pen2;
      r[7] = cont;
      r[15] = clash;
    }
  }
  __syncthreads();

  if (full) {
    // ---- F: NN softmin statistics, shift = first minimum (argmin_s) --------
    const int nrc = m1 + m2;
    for (int it = tid; it < n_here * nrc; it += nth) {
      const int ku = it / nrc, r = it - ku * nrc;
      const Unit<ND> u = unit(ku);
      const bool row = r < m1;
      const int n = row ? m2 : m1;
      auto idx = [&](int j) { return row ? r * m2 + j : j * m2 + (r - m1); };
      int jm = 0;
      for (int j = 1; j < n; ++j)
        if (u.pair(idx(j))[3].v < u.pair(idx(jm))[3].v) jm = j;
      const T mn = u.pair(idx(jm))[3];
      T tot = 0.0;
      for (int j = 0; j < n; ++j) tot += exp_d((mn - u.pair(idx(j))[3]) * c.inv_tau_nn);
      u.nnstat()[2 * r] = mn;
      u.nnstat()[2 * r + 1] = rcp_d(tot);
    }
    __syncthreads();
    // ---- G: activity product + fixed-layout E-E rows (303-330) ---------------
    for (int it = tid; it < n_here * P; it += nth) {
      const int ku = it / P, i = it - ku * P;
      const Unit<ND> u = unit(ku);
      const int k = i / m2, l = i - (i / m2) * m2;
      const T* rec = u.pair(i);
      const T* ns = u.nnstat();
      const T dg = rec[3];
      const T nn1 = exp_d((ns[2 * k] - dg) * c.inv_tau_nn) * ns[2 * k + 1];
      const T nn2 = exp_d((ns[2 * (m1 + l)] - dg) * c.inv_tau_nn) * ns[2 * (m1 + l) + 1];
      const T act1 = rec[16] * rec[6] * nn1 * rec[15] * rec[7];
      const T act2 = rec[16] * rec[14] * nn2 * rec[15] * rec[7];
      const T g1 = rec[4], g2 = rec[5];
      const vec3<T> nb = mk3<T>(rec[11], rec[12], rec[13]);
      const int64_t row = u.env * C + n1 + n2 + 2 * i;
      put_contact<ND>(p, u.group, row, mk3<T>(rec[0], rec[1], rec[2]), g1 * dg, dscale(nb, g1), act1);
      put_contact<ND>(p, u.group, row + 1, mk3<T>(rec[8], rec[9], rec[10]), g2 * dg, dscale(nb, g2), act2);
      if (u.group == 0 && m.src) {
        int* sp = m.src + row * 2;
        const int sa = u.prov()[n1 + n2 + k], sb = u.prov()[n1 + n2 + m1 + l];
        sp[0] = sa; sp[1] = sb; sp[2] = sa; sp[3] = sb;
      }
    }
  }
  __syncthreads();

  // ---- H: mean contact distance (manifold.hpp:379-384), fixed order ---------
  if (m.mean_dist || p.mean_grad || p.mean_f64 || p.mean_grad_f64) {
    for (int k = tid; k < n_here; k += nth) {
      const Unit<ND> u = unit(k);
      T acc = 0.0;
      for (int r = 0; r < n1 + n2; ++r) acc += u.vsdist()[r];
      for (int i = 0; i < P && full; ++i) {
        const T* rec = u.pair(i);
        acc += rec[4] * rec[3];
        acc += rec[5] * rec[3];
      }
      const T mean = acc * (1.0 / (double)C);
      if (u.group == 0 && m.mean_dist) m.mean_dist[u.env] = (float)mean.v;
      if (p.mean_grad)
#pragma unroll
        for (int j = 0; j < ND; ++j) p.mean_grad[u.env * 12 + u.group * ND + j] = (float)mean.d[j];
      if (u.group == 0 && p.mean_f64) p.mean_f64[u.env] = mean.v;
      if (p.mean_grad_f64)
#pragma unroll
        for (int j = 0; j < ND; ++j) p.mean_grad_f64[u.env * 12 + u.group * ND + j] = mean.d[j];
    }
  }
}

template <int K1, int K2>
int launch_jvp_kind(const JvpParams& p, int threads, cudaStream_t s) {
  static PerDeviceOnce configured;
  configured([] {  // per device: the attribute does not carry across devices
    cudaFuncSetAttribute(manifold_jvp_kernel<K1, K2, kJvpND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
  });
  const int64_t units = p.m.n_env * p.groups;
  const int64_t grid = (units + p.units_per_block - 1) / p.units_per_block;
  manifold_jvp_kernel<K1, K2, kJvpND><<<(unsigned)grid, threads, (size_t)p.bytes * p.units_per_block, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// SQ kinds share the runtime-exponent path (kSqE01 -> kSingleSq): the JVP is
// not the throughput path, one instantiation per shape class keeps the
// library small.
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

int jvp_directions() { return kJvpND; }
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
