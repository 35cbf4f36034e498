// Fused batched contact-manifold kernel templates (K1-K5 of SURVEY.md §2),
// instantiated by manifold.cu (the base SDF kinds) and manifold_ct.cu (the
// other compile-time-exponent superquadric kinds):
//   generate_manifold<T> (include/cmg/manifold.hpp:336-377) for every env of
//   a batch, + mean_contact_distance (379-384), in ONE launch.
//
// Mapping: a CTA owns `envs_per_block` consecutive envs (all envs share the
// same two surfaces, so every branch on geometry / config is warp-uniform;
// the SDF kind of each side is a template parameter). Phases, separated by
// __syncthreads():
//   A  pose -> (R, t)                         se3_exp            pose.hpp:78-91
//   B  opposing-SDF vertex scores (top-K)     vertex/edge_penetrations 77-94
//   C  rank sort of scores (top-K)            soft_topk sort     smooth_ops.hpp:180-185
//   D  selected vertex / edge slots           select_topk_*      manifold.hpp:128-181
//   E  E-E pair stage                         ee_contacts 237-287
//   F  row / column NN softmin statistics     ee_contacts 289-301
//      + V-S contacts on the idle warps       vs_contacts 185-204
//   G  activity product + fixed-layout store  ee_contacts 303-330
//   H  per-env mean contact distance          mean_contact_distance 379-384
// Per-env state lives in shared memory (SmemLayout); the only HBM traffic is
// the poses in (96 B/env), mesh/SDF reads (L1/L2-resident) and the contacts
// out (C x 32 B/env).
#pragma once

#include <cuda_runtime.h>

#include "../common.h"
#include "launch_util.cuh"
#include "../device/dmath.cuh"
#include "../device/sdf.cuh"
#include "../device/witness.cuh"

namespace cmgb {

namespace {

// Developer instrumentation (-DCMGB_PHASE_CLOCKS): SM clocks per phase,
// summed over CTAs by thread 0 at each barrier (tools/phase_clocks.py).
#ifdef CMGB_PHASE_CLOCKS
__device__ unsigned long long g_mf_phase[16];
#define MF_PHASE_START() long long t_prev_ = clock64()
#define MF_PHASE_MARK(k)                                                    \
  do {                                                                      \
    __syncthreads();                                                        \
    if (threadIdx.x == 0) {                                                 \
      const long long t_ = clock64();                                       \
      atomicAdd(&g_mf_phase[k], (unsigned long long)(t_ - t_prev_));       \
      t_prev_ = t_;                                                         \
    }                                                                       \
  } while (0)
#define MF_PHASE_MARK_DBG(k) MF_PHASE_MARK(k)
#else
#define MF_PHASE_START() (void)0
#define MF_PHASE_MARK(k) __syncthreads()
#define MF_PHASE_MARK_DBG(k) (void)0  // no barrier in production builds
#endif

// CTA shape per SDF kind pair (measured):
//   box-box (both sides the same compile-time-exponent superquadric kind, e.g.
//     eps = 0.1): 9 warps (2 envs x 144 E-E pairs), 4 CTAs/SM (<= 56
//     registers), V-S contacts on the warps the NN phase leaves idle (F);
//   everything else: 10 warps, 3 CTAs/SM (<= 64 registers), V-S contacts in
//     the pair phase (E) after the pair items (config D forward +4%).
__host__ __device__ constexpr bool box_box(int k1, int k2) { return k1 == k2 && ct_sq(k1); }
#ifndef CMGB_CAPSULE_BLOCKS
#define CMGB_CAPSULE_BLOCKS 3  // measured: 2 CTAs x 96 registers still spill and run 10% slower
#endif
constexpr int kCapsuleBlocks = CMGB_CAPSULE_BLOCKS;  // resident CTAs/SM of the capsule instantiations
__host__ __device__ constexpr int max_threads(int k1, int k2) { return box_box(k1, k2) ? 288 : 320; }
__host__ __device__ constexpr int min_blocks(int k1, int k2) {
  return box_box(k1, k2) ? 4 : (k1 == kCapsule || k2 == kCapsule ? kCapsuleBlocks : 3);
}
__host__ __device__ constexpr bool vs_in_pair_phase(int k1, int k2) { return !box_box(k1, k2); }

// Pair record (doubles; kPairRec = 38 floats = 19 doubles = 152 B), rewritten
// in place by the E-E sub-phases:
//   side s at 8 s: [0-2] witness point (body frame -> traced -> world),
//                  [3-5] own normal (world), [6] phi_other(p), [7] phi_own(p)
//   [16] con (gamma of the QP)
// after E3: [3] dbar, [4] sign1, [5] sign2, [11-13] nbar, [6] pen1, [14] pen2,
//           [7] cont, [15] clash, [0-2] / [8-10] world witness points
struct EnvView {
  unsigned char* base;
  const SmemLayout* L;
  double* prec;  // this env's pair records: shared memory, or the global workspace
  __device__ double* R(int s) const { return reinterpret_cast<double*>(base + L->frames) + 12 * s; }
  __device__ double* t(int s) const { return R(s) + 9; }
  __device__ double* vslot(int i) const { return reinterpret_cast<double*>(base + L->vslots) + 3 * i; }
  // 12 doubles per edge slot + 1 pad: odd stride, so the lanes of a warp reading
  // different slots hit distinct shared-memory banks
  __device__ double* eslot(int i) const { return reinterpret_cast<double*>(base + L->eslots) + 13 * i; }
  __device__ int* prov() const { return reinterpret_cast<int*>(base + L->prov); }
  __device__ double* scores() const { return reinterpret_cast<double*>(base + L->scores); }
  __device__ int* sorted() const { return reinterpret_cast<int*>(base + L->sorted); }
  __device__ double* tkw() const { return reinterpret_cast<double*>(base + L->tkw); }
  __device__ double* pair(int i) const { return prec + (kPairRec / 2) * i; }
  __device__ float* vsdist() const { return reinterpret_cast<float*>(base + L->vsdist); }
  __device__ double* nnstat() const { return reinterpret_cast<double*>(base + L->nnstat); }
  __device__ double* hpart() const { return reinterpret_cast<double*>(base + L->hpart); }
  __device__ uint32_t* amask() const { return reinterpret_cast<uint32_t*>(base + L->amask); }
  __device__ double& dbar(int i) const { return pair(i)[3]; }
};

// q = n / d, r = n % d with the host-precomputed multiplier.
__device__ __forceinline__ int fdiv(int n, const FastDiv& f) {
  return (int)(((uint64_t)(uint32_t)n * f.mul) >> 32);
}
__device__ __forceinline__ void fdivmod(int n, const FastDiv& f, int& q, int& r) {
  q = fdiv(n, f);
  r = n - q * (int)f.d;
}

__device__ __forceinline__ double3 ld_vert(const double* v, int i) {
  return d3(__ldg(v + 3 * i), __ldg(v + 3 * i + 1), __ldg(v + 3 * i + 2));
}

__device__ __forceinline__ double3 to_world(const double* R, const double* t, double3 pb) {
  return mul_R(R, pb) + d3(t[0], t[1], t[2]);
}
__device__ __forceinline__ double3 to_body(const double* R, const double* t, double3 pw) {
  return mul_Rt(R, pw - d3(t[0], t[1], t[2]));
}

// Score-set index helpers: sets 0 = V1, 1 = V2, 2 = E1, 3 = E2.
struct Sets {
  int off[5];
  __device__ Sets(const ManifoldParams& p) {
    off[0] = 0;
    off[1] = p.side[0].nv;
    off[2] = off[1] + p.side[1].nv;
    off[3] = off[2] + p.side[0].ne;
    off[4] = off[3] + p.side[1].ne;
  }
};

__device__ __forceinline__ void store_contact(float* dst, float px, float py, float pz, float d,
                                              float nx, float ny, float nz, float a) {
  float4* o = reinterpret_cast<float4*>(dst);
  o[0] = make_float4(px, py, pz, d);
  o[1] = make_float4(nx, ny, nz, a);
}

// normalize_smooth (vec3.hpp:56-62) in FP64.
__device__ __forceinline__ double3 normalize_smooth(double3 v, double tau) {
  return dscale(v, rsqrt_d(tau + ddot(v, v)));
}

// V-S contact for a selected vertex (world) against the opposing posed SDF
// (vs_contacts, manifold.hpp:185-204).
// Returns the stored (FP32) activity.
template <int KO>
__device__ __forceinline__ float vs_contact(const DevSdf& opp, const double* Ro, const double* to,
                                            double3 pw, const DevCfg& c, float* out_dist,
                                            float* dst) {
  const SdfOut s = sdf_eval<kNormalSource, KO>(opp, to_body(Ro, to, pw));
  const float3 n = to_f3v(mul_R(Ro, normalize_smooth(s.g, c.tau_normal)));
  const double act = sigmoid_d(-s.v * c.inv_tau_pen);  // sigma_greater(-phi, 0, tau_pen)
  *out_dist = (float)s.v;
  store_contact(dst, (float)pw.x, (float)pw.y, (float)pw.z, (float)s.v, n.x, n.y, n.z, (float)act);
  return (float)act;
}

// sphere_trace_project (sdf.hpp:318-326) in the body frame, FP64.
// One step p -= normalize_smooth(grad phi) phi, as p - g (phi / sqrt(tau + |g|^2)):
// one product for the scale, three FMAs for the update.
template <int K>
__device__ __forceinline__ double3 trace_step(const DevSdf& sdf, double3 p, double tau_normal) {
  const SdfOut s = sdf_eval<kGrad, K>(sdf, p);
  const double sc = rsqrt_d(tau_normal + ddot(s.g, s.g)) * s.v;
  return d3(fma(-s.g.x, sc, p.x), fma(-s.g.y, sc, p.y), fma(-s.g.z, sc, p.z));
}

// The same projection for a lone compile-time superquadric, run in the
// primitive's normalised coordinates u = R^T (p - t) / axes (the field's own
// variables; the update is rotation-equivariant, so tracing in the primitive
// frame is the same iteration). With w = 1 / |u|^2 and the gradient written as
// grad phi = |u|^-1 diag(1/axes) H, H_i = u_i (k c A'_i - (1 - f^p4) w):
//   phi grad / sqrt(tau + |grad|^2) = diag(1/axes) H (1 - f^p4) w / sqrt(tau + w |diag(1/axes) H|^2),
// so one reciprocal replaces the radius rsqrt, the 1/|u| scalings of phi and
// of the gradient drop out, and u needs no per-step rescaling (a quarter fewer
// FP64 operations per step than trace_step); mapped back once at the end.
template <int K>
__device__ __forceinline__ double3 trace_sq(const DevSq& q, double3 p, const DevCfg& c) {
  constexpr SqExpTuple E = sq_exps(K);
  if (q.has_frame) p = mul_Rt(q.R, p - d3(q.t[0], q.t[1], q.t[2]));
  double ux = p.x * q.inv_ax[0], uy = p.y * q.inv_ax[1], uz = p.z * q.inv_ax[2];
  const double a2x = q.inv_ax[0] * q.inv_ax[0], a2y = q.inv_ax[1] * q.inv_ax[1], a2z = q.inv_ax[2] * q.inv_ax[2];
#pragma unroll 1
  for (int it = 0; it < c.trace_iters; ++it) {
    const double x2 = fma(ux, ux, kMC.floor30), y2 = fma(uy, uy, kMC.floor30), z2 = fma(uz, uz, kMC.floor30);
    double A, Am1, B, Bm1, G, Gm1, Cz, Czm1;
    // (compile-time exponents, or -- kSingleSq -- the descriptor's: integer
    // chains where exact, else pow_rt)
    pow_pair_t<E.n1>(x2, E.n1 ? E.n1 : q.n1, q.p1, A, Am1);
    pow_pair_t<E.n1>(y2, E.n1 ? E.n1 : q.n1, q.p1, B, Bm1);
    pow_pair_t<E.n2>(A + B, E.n2 ? E.n2 : q.n2, q.p2, G, Gm1);
    pow_pair_t<E.n3>(z2, E.n3 ? E.n3 : q.n3, q.p3, Cz, Czm1);
    const double f = G + Cz;
    const double w = rcp_d(fma(ux, ux, fma(uy, uy, fma(uz, uz, kMC.floor20))));
    double F, inv_f;
    const double omF = one_minus_pow<E.n4>(f, q.p4, E.n4 ? E.n4 : q.n4, &F, &inv_f);
    const double k = -q.p4 * F * inv_f;
    const double kxy = k * (q.c_xy * Gm1), kz = k * q.c_z;
    const double hw = omF * w;
    const double Hx = ux * fma(kxy, Am1, -hw), Hy = uy * fma(kxy, Bm1, -hw), Hz = uz * fma(kz, Czm1, -hw);
    const double Px = a2x * Hx, Py = a2y * Hy, Pz = a2z * Hz;
    const double sc = hw * rsqrt_d(fma(w, fma(Px, Hx, fma(Py, Hy, Pz * Hz)), c.tau_normal));
    ux = fma(-Px, sc, ux);
    uy = fma(-Py, sc, uy);
    uz = fma(-Pz, sc, uz);
  }
  p = d3(ux * q.ax[0], uy * q.ax[1], uz * q.ax[2]);
  if (q.has_frame) p = mul_R(q.R, p) + d3(q.t[0], q.t[1], q.t[2]);
  return p;
}

template <int K>
__device__ __forceinline__ double3 trace(const DevSdf& sdf, double3 p, const DevCfg& c) {
  if constexpr (ct_sq(K) || K == kSingleSq) {  // a lone superquadric leaf: the normalised-coordinate trace
    return trace_sq<K>(sdf.nodes[0].sq, p, c);
  } else {
#pragma unroll 1
    for (int k = 0; k < c.trace_iters; ++k) p = trace_step<K>(sdf, p, c.tau_normal);
    return p;
  }
}

// E1: witness QP of pair (k, l) (ee_witness, witness.hpp:137-158; edges in the
// world frame), witness points written in their own body frames.
template <int kH = -1>
__device__ __forceinline__ void ee_stage_qp(const ManifoldParams& p, const EnvView& ev, int k, int l,
                                            double* rec) {
  const double* s1 = ev.eslot(k);
  const double* s2 = ev.eslot(p.m1 + l);
  const QpSol w = ee_qp<double, double, false, kH>(d3(s1[0], s1[1], s1[2]), d3(s1[3], s1[4], s1[5]), d3(s2[0], s2[1], s2[2]),
                        d3(s2[3], s2[4], s2[5]), p.cfg);
  // edge_point (witness.hpp:130-133) on the body-frame endpoints
  rec[0] = s1[6] + (s1[9] - s1[6]) * w.a1;
  rec[1] = s1[7] + (s1[10] - s1[7]) * w.a1;
  rec[2] = s1[8] + (s1[11] - s1[8]) * w.a1;
  rec[8] = s2[6] + (s2[9] - s2[6]) * w.a2;
  rec[9] = s2[7] + (s2[10] - s2[7]) * w.a2;
  rec[10] = s2[8] + (s2[11] - s2[8]) * w.a2;
  rec[16] = w.gamma;
}

// E2: one side of a pair: sphere-trace the witness on its own surface
// (manifold.hpp:245-247), own normal source (253-256), world point, and the
// opposing surface's value for the penetration indicator (279-280).
template <int KS, int KO>
__device__ __forceinline__ void ee_stage_side(const ManifoldParams& p, const EnvView& ev, int s,
                                              double* r) {
  const DevCfg& c = p.cfg;
  const DevSdf& own = p.side[s].sdf;
  const DevSdf& oth = p.side[1 - s].sdf;
  double3 pb = d3(r[0], r[1], r[2]);
  if (c.trace_iters > 0) pb = trace<KS>(own, pb, c);
  const SdfOut o = c.containment ? sdf_eval<kNormalSource, KS>(own, pb) : sdf_eval<kNormalOnly, KS>(own, pb);
  const double* R = ev.R(s);
  const double3 n = mul_R(R, normalize_smooth(o.g, c.tau_normal));
  const double3 pw = to_world(R, ev.t(s), pb);
  const double v_oth = sdf_eval<kValue, KO>(oth, to_body(ev.R(1 - s), ev.t(1 - s), pw)).v;
  r[0] = pw.x; r[1] = pw.y; r[2] = pw.z;
  r[3] = n.x; r[4] = n.y; r[5] = n.z;
  r[6] = v_oth;
  r[7] = o.v;
}

// exp(x) for the NN softmin weights (x <= 0, FP64-exact argument rounded
// once): SFU ex2 (2^-22 relative; the weights only scale FP32 activities).
__device__ __forceinline__ float nn_weight(double x) { return ex2f((float)x * 1.44269504088896341f); }

// sigma(x) in FP32 with the accurate expf (arguments are FP64-exact; the
// indicators only scale the activity, tolerance 1e-5 relative).
__device__ __forceinline__ float sigmoid_acc(double xd) {
  const float x = (float)xd;
  const float e = expf(-fabsf(x));
  const float inv = __frcp_rn(1.0f + e);  // correctly rounded, without the division's slow-path checks
  return x >= 0.0f ? inv : e * inv;
}

// E3: pair quantities (manifold.hpp:248-266, 279-285): separation, unsigned
// normal, soft signs, penetration / clash / containment indicators.
__device__ __forceinline__ void ee_stage_pair(const DevCfg& c, double* r) {
  const double3 p1w = d3(r[0], r[1], r[2]), p2w = d3(r[8], r[9], r[10]);
  const double3 n1 = d3(r[3], r[4], r[5]), n2 = d3(r[11], r[12], r[13]);
  const double3 de = p1w - p2w;
  // |de|_guarded and de / |de| from one refined reciprocal square root (1.3e-12
  // relative, far below the FP32 outputs' resolution) instead of sqrt + reciprocal
  const double dd = ddot(de, de) + 1e-12;  // kEdgeNormalEps
  const double rs = rsqrt_d(dd);
  const double dg = dd * rs;
  const double3 nb = dscale(de, rs);
  const double d2 = ddot(n2, nb), d1 = ddot(n1, nb);
  double g1, g2;
  if (c.hard_ops) {  // sign_hard (smooth_ops.hpp:208)
    g1 = d2 < 0.0 ? -1.0 : (d2 > 0.0 ? 1.0 : 0.0);
    g2 = d1 < 0.0 ? -1.0 : (d1 > 0.0 ? 1.0 : 0.0);
  } else {  // sign_s = tanh(x / tau_sign) (smooth_ops.hpp:57-62), FP64-exact argument
    g1 = (double)tanhf((float)(d2 * c.inv_tau_sign));
    g2 = (double)tanhf((float)(d1 * c.inv_tau_sign));
  }
  const double pen1 = sigmoid_acc(-r[6] * c.inv_tau_pen);
  const double pen2 = sigmoid_acc(-r[14] * c.inv_tau_pen);
  const double clash = sigmoid_acc(-ddot(n1, n2) * c.inv_tau_clash);
  const double cont = c.containment ? (double)sigmoid_acc(-r[7] * c.inv_tau_cont) *
                                          (double)sigmoid_acc(-r[15] * c.inv_tau_cont)
                                    : 1.0;
  r[3] = dg;
  r[4] = g1;
  r[5] = g2;
  r[11] = nb.x; r[12] = nb.y; r[13] = nb.z;
  r[6] = pen1;
  r[14] = pen2;
  r[7] = cont;
  r[15] = clash;
}

// Pose -> frame (R, t) for every distinct pose (se3_exp, pose.hpp:78-91), one
// thread each, ahead of the manifold kernel: keeps the FP64 sincos latency
// chain off the manifold CTAs' critical path (they would otherwise idle at
// the first barrier while 4 threads evaluate it).
__global__ void __launch_bounds__(256) frames_kernel(const double* __restrict__ poses1, int64_t stride1, int64_t n1,
                                                     double* __restrict__ frames1, const double* __restrict__ poses2,
                                                     int64_t stride2, int64_t n2, double* __restrict__ frames2) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n1 + n2) return;
  const bool second = i >= n1;  // both bodies' poses in one launch
  if (second) i -= n1;
  const double* poses = second ? poses2 : poses1;
  const int64_t stride = second ? stride2 : stride1;
  double xi[6], R[9], t[3];
#pragma unroll
  for (int k = 0; k < 6; ++k) xi[k] = __ldg(poses + stride * i + k);
  se3_exp_d(xi, R, t);
  double* f = (second ? frames2 : frames1) + 12 * i;
#pragma unroll
  for (int k = 0; k < 9; ++k) f[k] = R[k];
  f[9] = t[0];
  f[10] = t[1];
  f[11] = t[2];
}

// The K largest of a set's D <= 32 R scores in order, ties to the lowest index
// (the soft top-K's sort, smooth_ops.hpp:180-185), by one warp: per round,
// each lane's best remaining order-preserving 64-bit key, then warp reductions
// over (high word, low word, lowest index); out[r] = set-local index of rank r.
template <int R>
__device__ __forceinline__ void extract_topk(const double* sc, int D, int K, int* out, int lane) {
  uint64_t key[R];  // 0 = taken / absent
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int j = lane + 32 * k;
    const uint64_t u = j < D ? (uint64_t)__double_as_longlong(sc[j]) : 0ull;
    key[k] = j >= D ? 0ull : ((int64_t)u < 0 ? ~u : (u | 0x8000000000000000ull));
  }
  for (int r = 0; r < K; ++r) {
    uint64_t b = key[0];
    int bj = lane;
#pragma unroll
    for (int k = 1; k < R; ++k)
      if (key[k] > b) {  // strict: the lowest index among equal keys
        b = key[k];
        bj = lane + 32 * k;
      }
    const unsigned bh = (unsigned)(b >> 32), bl = (unsigned)b;
    const unsigned mh = __reduce_max_sync(0xffffffffu, bh);
    const unsigned ml = __reduce_max_sync(0xffffffffu, bh == mh ? bl : 0u);
    const int wj = __reduce_min_sync(0xffffffffu, (bh == mh && bl == ml) ? bj : 0x7fffffff);
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (lane + 32 * k == wj) key[k] = 0ull;
    if (lane == 0) out[r] = wj;
  }
}

// kGP: pair records in the global workspace (p.pairs_gmem; large pass-through
// pair sets, one generic instantiation) instead of shared memory. kVsX: the
// V-S contacts come from vs_kernel (box-box, pass-through vertex sets; p.vs_ext).
template <int K1, int K2, bool kGP = false, bool kVsX = false>
__global__ void __launch_bounds__(max_threads(K1, K2), min_blocks(K1, K2))
    manifold_kernel(const __grid_constant__ ManifoldParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int epb = p.envs_per_block;
  const int64_t env0 = (int64_t)blockIdx.x * epb;
  const int n_here = (int)(p.n_env - env0 < epb ? p.n_env - env0 : epb);
  const int tid = threadIdx.x, nth = blockDim.x;
  MF_PHASE_START();
  const DevCfg& c = p.cfg;
  const DevSide& S1 = p.side[0];
  const DevSide& S2 = p.side[1];
  const int n1 = p.n1, n2 = p.n2, m1 = p.m1, m2 = p.m2, P = m1 * m2;
  const bool full = m1 > 0 && m2 > 0;
  auto env = [&](int e) {
    unsigned char* b = smem + (size_t)e * p.smem.bytes;
    if constexpr (kGP) return EnvView{b, &p.smem, p.pairs_gmem + (env0 + e) * p.pair_stride};
    else return EnvView{b, &p.smem, reinterpret_cast<double*>(b + p.smem.pairs)};
  };

  // ---- A: frames (precomputed by frames_kernel) -> shared memory ----------
  for (int i = tid; i < 24 * n_here; i += nth) {
    const int e = i / 24, s = (i % 24) / 12, k = i % 12;
    const double* f = s == 0 ? p.frames1 + 12 * (env0 + e) * p.stride1
                             : p.frames2 + 12 * (env0 + e) * p.stride2;
    env(e).R(s)[k] = __ldg(f + k);
  }

  // activity masks of the compaction extra: zero, or (kVsX) the V-S bits vs_kernel left in word 0
  if (p.act_mask)
    for (int i = tid; i < p.mask_words * n_here; i += nth) {
      const int e = i / p.mask_words, w = i - e * p.mask_words;
      env(e).amask()[w] = (kVsX && w == 0) ? p.act_mask[(env0 + e) * p.mask_words] : 0u;
    }

  const bool topk_any = S1.topk_v | S2.topk_v | S1.topk_e | S2.topk_e;
  const int nsl = n1 + n2 + m1 + m2;
  // ---- D for pass-through slots (K == D, manifold.hpp:135-140, 158-167), in
  // the same phase as A: each slot reads its env's frame straight from global
  // memory and its body-frame payload from the pre-expanded edge endpoints (no
  // dependent index load), so the frame copy and the slot transforms overlap
  // their memory latencies behind one barrier.
  if (!topk_any) {
    for (int it = tid; it < n_here * nsl; it += nth) {
      int e, r0;
      fdivmod(it, p.div_nslots, e, r0);
      const EnvView ev = env(e);
      const bool is_edge = r0 >= n1 + n2;
      const int s = is_edge ? (r0 - n1 - n2 < m1 ? 0 : 1) : (r0 < n1 ? 0 : 1);
      const int r = is_edge ? (s == 0 ? r0 - n1 - n2 : r0 - n1 - n2 - m1) : (s == 0 ? r0 : r0 - n1);
      const DevSide& S = s == 0 ? S1 : S2;
      const double* f = s == 0 ? p.frames1 + 12 * (env0 + e) * p.stride1 : p.frames2 + 12 * (env0 + e) * p.stride2;
      ev.prov()[r0] = r;
      if (is_edge) {
        const double* eb = S.edge_body + 6 * r;
        const double3 a = d3(__ldg(eb), __ldg(eb + 1), __ldg(eb + 2));
        const double3 b = d3(__ldg(eb + 3), __ldg(eb + 4), __ldg(eb + 5));
        double* q = ev.eslot(r0 - n1 - n2);
        const double3 aw = to_world(f, f + 9, a), bw = to_world(f, f + 9, b);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
        q[3] = bw.x; q[4] = bw.y; q[5] = bw.z;
        q[6] = a.x; q[7] = a.y; q[8] = a.z;
        q[9] = b.x; q[10] = b.y; q[11] = b.z;
      } else {
        const double3 a = ld_vert(S.verts, r);
        double* q = ev.vslot(r0);
        const double3 aw = to_world(f, f + 9, a);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
      }
    }
  }
  MF_PHASE_MARK(0);

  const Sets sets(p);
  if (topk_any) {
    // ---- B: vertex penetration scores (opposing posed SDF value) ----------
    const int nv_all = S1.nv + S2.nv;
    for (int it = tid; it < n_here * nv_all; it += nth) {
      int e, i;
      fdivmod(it, p.div_nv_all, e, i);
      const int s = i < S1.nv ? 0 : 1;
      const int vi = s == 0 ? i : i - S1.nv;
      const EnvView ev = env(e);
      const double3 pw = to_world(ev.R(s), ev.t(s), ld_vert(s == 0 ? S1.verts : S2.verts, vi));
      const double3 pb = to_body(ev.R(1 - s), ev.t(1 - s), pw);
      const double pen = s == 0 ? sdf_eval<kValue, K2>(S2.sdf, pb).v : sdf_eval<kValue, K1>(S1.sdf, pb).v;
      ev.scores()[i] = -pen;  // scores = negated penetrations (manifold.hpp:142-143)
    }
    MF_PHASE_MARK(1);
    // edge scores: -(mean of endpoint penetrations) (edge_penetrations, 86-94)
    const int ne_all = S1.ne + S2.ne;
    for (int it = tid; it < n_here * ne_all; it += nth) {
      int e, i;
      fdivmod(it, p.div_ne_all, e, i);
      const int s = i < S1.ne ? 0 : 1;
      const int ei = s == 0 ? i : i - S1.ne;
      const int32_t* E = s == 0 ? S1.edges : S2.edges;
      const int va = __ldg(E + 2 * ei), vb = __ldg(E + 2 * ei + 1);
      double* sc = env(e).scores();
      const int voff = s == 0 ? 0 : S1.nv;
      const double pa = -sc[voff + va], pb = -sc[voff + vb];
      sc[sets.off[2] + i] = -((pa + pb) * 0.5);
    }
    MF_PHASE_MARK(2);
    // ---- C: descending order of the scores of each set, ties by index (the
    // reference's sort, smooth_ops.hpp:180-185, only matters through its
    // values). The soft top-K rows read only ranks < K: sorted[lo + r] holds
    // the set-local index of the score of rank r. Two schemes:
    //  * large sets (K x 104 < D^2, D <= 128): one warp extracts the K largest
    //    in order -- per round, each lane's best remaining key, then warp
    //    reductions over (key high word, key low word, lowest index);
    //  * the others: rank_i = #{j: x_j > x_i or (x_j == x_i and j < i)}, one
    //    lane per score (the lanes of a warp read the same x_j: broadcasts).
    const int total = sets.off[4];
    auto set_active = [&](int set) {
      return set == 0 ? S1.topk_v : set == 1 ? S2.topk_v : set == 2 ? S1.topk_e : S2.topk_e;
    };
    auto set_K = [&](int set) { return set == 0 ? S1.n_sel : set == 1 ? S2.n_sel : set == 2 ? S1.m_sel : S2.m_sel; };
    auto extracted = [&](int set) {
      const int D = sets.off[set + 1] - sets.off[set];
      return set_active(set) && D <= 128 && set_K(set) * 104 < D * D;
    };
    {
      const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
      for (int task = warp; task < n_here * 4; task += nwarps) {  // warp-uniform
        const int e = task >> 2, set = task & 3;
        if (!extracted(set)) continue;
        const EnvView ev = env(e);
        const int lo = sets.off[set], D = sets.off[set + 1] - lo, K = set_K(set);
        const double* sc = ev.scores() + lo;
        int* out = ev.sorted() + lo;
        switch ((D + 31) >> 5) {  // key registers per lane: the set's size, not the 128 maximum
          case 1: extract_topk<1>(sc, D, K, out, lane); break;
          case 2: extract_topk<2>(sc, D, K, out, lane); break;
          case 3: extract_topk<3>(sc, D, K, out, lane); break;
          default: extract_topk<4>(sc, D, K, out, lane); break;
        }
      }
    }
    for (int it = tid; it < n_here * total; it += nth) {
      int e, i;
      fdivmod(it, p.div_scores, e, i);
      const int set = i < sets.off[1] ? 0 : i < sets.off[2] ? 1 : i < sets.off[3] ? 2 : 3;
      if (!set_active(set) || extracted(set)) continue;
      const int K = set_K(set);
      const EnvView ev = env(e);
      const double* sc = ev.scores();
      const double x = sc[i];
      const int lo = sets.off[set], hi = sets.off[set + 1];
      int rank = 0;
#pragma unroll 4
      for (int j = lo; j < hi; ++j) {
        const double y = sc[j];
        rank += y > x || (y == x && j < i);
      }
      if (rank < K) ev.sorted()[lo + rank] = i - lo;
    }
    MF_PHASE_MARK(3);
    // ---- C2: soft top-K weight factors. With the set's top score c and
    // P_i = exp((x_i - c) / tau), a row's weights exp(-|s_r - x_i| / tau) are
    // P_i / P_r (x_i <= s_r) or P_r / P_i (x_i > s_r): one exponential per
    // element instead of one per (row, element). Rows whose (c - s_r) / tau
    // leaves the range where every quotient is finite evaluate their
    // exponentials directly (D).
    for (int it = tid; it < n_here * total; it += nth) {
      int e, i;
      fdivmod(it, p.div_scores, e, i);
      const int set = i < sets.off[1] ? 0 : i < sets.off[2] ? 1 : i < sets.off[3] ? 2 : 3;
      const bool active = set == 0 ? S1.topk_v : set == 1 ? S2.topk_v : set == 2 ? S1.topk_e : S2.topk_e;
      if (!active) continue;
      const EnvView ev = env(e);
      const double* sc = ev.scores();
      const int lo = sets.off[set];
      const double top = sc[lo + min(max(ev.sorted()[lo], 0), sets.off[set + 1] - lo - 1)];
      ev.tkw()[i] = exp_d((sc[i] - top) * (set < 2 ? c.inv_tau_topk_v : c.inv_tau_topk_e));
    }
    MF_PHASE_MARK(9);
    MF_PHASE_MARK(3);
  }

  // ---- D: selected slots with soft top-K active (pass-through sets of the
  // same launch are handled here too; without top-K, D ran with A) ----------
  if (topk_any) {
    // With soft top-K active, each slot is a group of 4 adjacent lanes that
    // splits the row's candidates (shuffle-reduced): the rows are long serial
    // loops (D up to ~100) that otherwise keep the whole CTA at the barrier.
    constexpr int lshift = 2;  // measured: 2 lanes per row +6%, 8 lanes +9% time (config C)
    constexpr int lanes = 1 << lshift;
    for (int it = tid; it < (n_here * nsl) << lshift; it += nth) {
      const int ql = it & (lanes - 1);
      int e, r0;
      fdivmod(it >> lshift, p.div_nslots, e, r0);
      const EnvView ev = env(e);
      const bool is_edge = r0 >= n1 + n2;
      const int s = is_edge ? (r0 - n1 - n2 < m1 ? 0 : 1) : (r0 < n1 ? 0 : 1);
      const int r = is_edge ? (s == 0 ? r0 - n1 - n2 : r0 - n1 - n2 - m1) : (s == 0 ? r0 : r0 - n1);
      const DevSide& S = s == 0 ? S1 : S2;
      const double* R = ev.R(s);
      const double* t = ev.t(s);
      const bool sel = is_edge ? S.topk_e : S.topk_v;
      double3 a = d3(0, 0, 0), b = d3(0, 0, 0);
      int prov = r;
      if (!sel) {  // K == D pass-through (manifold.hpp:135-140, 158-167)
        if (is_edge) {
          const double* eb = S.edge_body + 6 * r;
          a = d3(__ldg(eb), __ldg(eb + 1), __ldg(eb + 2));
          b = d3(__ldg(eb + 3), __ldg(eb + 4), __ldg(eb + 5));
        } else {
          a = ld_vert(S.verts, r);
        }
      } else {  // soft top-K row r (smooth_ops.hpp:191-196, manifold.hpp:141-148, 168-180)
        const int set = (is_edge ? 2 : 0) + s;
        const int lo = sets.off[set];
        const double* x = ev.scores() + lo;
        const double* q = ev.tkw() + lo;
        const int* order = ev.sorted() + lo;
        const int D = sets.off[set + 1] - lo;
        auto ord = [&](int k) { return min(max(order[k], 0), D - 1); };  // in range even for NaN scores
        const int ir = ord(r);
        const double sr = x[ir];
        const double Pr = q[ir];
        const double inv_tau = is_edge ? c.inv_tau_topk_e : c.inv_tau_topk_v;
        // One pass: unnormalised weights w_i = exp(-|s_r - x_i| / tau) accumulate
        // the total and the payload, normalised once at the end. The row's own
        // element has w = 1, so the total is >= 1 and a term below e^-50 moves
        // neither it nor the payload at FP64 resolution: those are skipped.
        double tot = 0.0;
        const double* __restrict__ pay = is_edge ? S.edge_body : S.verts;  // body-frame payload rows
        auto rows = [&](auto edge) {
          constexpr bool kE = decltype(edge)::value;
          auto add = [&](int i, double w) {
            tot += w;
            const double* pp = pay + (kE ? 6 : 3) * i;
            a = a + d3(__ldg(pp), __ldg(pp + 1), __ldg(pp + 2)) * w;
            if constexpr (kE) b = b + d3(__ldg(pp + 3), __ldg(pp + 4), __ldg(pp + 5)) * w;
          };
          if (Pr >= 1e-260) {  // (c - s_r) / tau <= 598: quotients of the C2 factors
            const double iPr = rcp_d(Pr);
            for (int i = ql; i < D; i += lanes) {
              const double Pi = q[i];
              const double w = Pi <= Pr ? Pi * iPr : Pr * rcp_d(Pi);  // Pi >= Pr >= 1e-260 in the second arm
              if (w < 1.9287498479639178e-22) continue;  // e^-50
              add(i, w);
            }
          } else {
            for (int i = ql; i < D; i += lanes) {
              const double arg = -fabs(sr - x[i]) * inv_tau;
              if (arg < -50.0) continue;
              add(i, exp_d(arg));
            }
          }
        };
        if (is_edge) rows(std::true_type{});
        else rows(std::false_type{});
        {  // reduce over the slot's lane group (fixed order)
          const unsigned gm = ((1u << lanes) - 1u) << ((tid & 31) & ~(lanes - 1));
#pragma unroll
          for (int o = 1; o < lanes; o <<= 1) {
            tot += __shfl_xor_sync(gm, tot, o);
            a.x += __shfl_xor_sync(gm, a.x, o);
            a.y += __shfl_xor_sync(gm, a.y, o);
            a.z += __shfl_xor_sync(gm, a.z, o);
            b.x += __shfl_xor_sync(gm, b.x, o);
            b.y += __shfl_xor_sync(gm, b.y, o);
            b.z += __shfl_xor_sync(gm, b.z, o);
          }
        }
        // provenance = first argmax of the row's weights (hard_attribution,
        // 110-121) = the lowest index holding s_r; equal scores take
        // consecutive ranks in index order, so it is the first rank of s_r's run
        int rr = r;
        while (rr > 0 && x[ord(rr - 1)] == sr) --rr;
        prov = sr == sr ? ord(rr) : -1;
        const double inv = rcp_d(tot);  // tot >= 1
        a = a * inv;
        b = b * inv;
      }
      if (ql != 0) continue;  // lane 0 of the group stores the slot
      ev.prov()[r0] = prov;
      if (is_edge) {
        double* q = ev.eslot(r0 - n1 - n2);
        const double3 aw = to_world(R, t, a), bw = to_world(R, t, b);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
        q[3] = bw.x; q[4] = bw.y; q[5] = bw.z;
        q[6] = a.x; q[7] = a.y; q[8] = a.z;
        q[9] = b.x; q[10] = b.y; q[11] = b.z;
      } else {
        double* q = ev.vslot(r0);
        const double3 aw = to_world(R, t, a);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
      }
    }
    MF_PHASE_MARK(4);
  }

  // ---- E: E-E pair stage + V-S contacts --------------------------------------
  // E1-E3 per pair, one thread owning the pair end to end (no barriers in
  // between; state passes through the pair's shared-memory record so each
  // stage's registers are released): QP -> trace/normal/opposing value of
  // side 1 and side 2 -> pair quantities. On the 10-warp CTA shape the V-S
  // contacts (vs_contacts, manifold.hpp:185-204; they read only phase-D state)
  // follow the pair items, beside them.
  const int C = p.n_contacts;
  const int nvs = n1 + n2;
  constexpr bool kVsE = vs_in_pair_phase(K1, K2);
  auto pair_item = [&](int it) {
    int e, i, k, l;
    fdivmod(it, p.div_pairs, e, i);
    fdivmod(i, p.div_m2, k, l);
    const EnvView ev = env(e);
    double* r = ev.pair(i);
    ee_stage_qp(p, ev, k, l, r);  // (a soft / hard split of this call spills at 56 registers)
    // both sides inline (measured: a shared code copy looping over the side
    // reads the side's SDF parameters with per-thread constant loads; +2%)
    ee_stage_side<K1, K2>(p, ev, 0, r);
    ee_stage_side<K2, K1>(p, ev, 1, r + 8);
    ee_stage_pair(c, r);
  };
  if constexpr (!kVsE) {
    if (full)
      for (int it = tid; it < n_here * P; it += nth) pair_item(it);
  } else {
    const int nE = full ? n_here * P : 0, nV = n_here * nvs;
    auto vs_item = [&](int v) {
      int e, r;
      fdivmod(v, p.div_nvs, e, r);
      const EnvView ev = env(e);
      const double* q = ev.vslot(r);
      float* dst = p.contacts + ((env0 + e) * C + r) * 8;
      const float act = r < n1 ? vs_contact<K2>(S2.sdf, ev.R(1), ev.t(1), d3(q[0], q[1], q[2]), c, ev.vsdist() + r, dst)
                               : vs_contact<K1>(S1.sdf, ev.R(0), ev.t(0), d3(q[0], q[1], q[2]), c, ev.vsdist() + r, dst);
      if (p.act_mask && act > p.act_thr) atomicOr(ev.amask() + (r >> 5), 1u << (r & 31));
      if (p.src) {
        int* sp = p.src + ((env0 + e) * C + r) * 2;
        sp[0] = ev.prov()[r];
        sp[1] = -1;
      }
    };
    // Fewer pairs than threads: the V-S items (~1/6 of a pair each) go to the
    // threads without a pair, up to 4 each, so the phase lasts one pair item
    // (config C: 256 pairs + 128 V-S items on 320 threads); else round robin.
    // (one call site each: the item bodies are large)
    const int spare = nth - nE;
    const bool spare_mode = nE > 0 && spare > 0 && nV <= 4 * spare;
    const int step = !spare_mode ? nth : tid < nE ? nE + nV : spare;
    for (int it = tid; it < nE + nV; it += step) {
      if (it < nE) pair_item(it);
      else vs_item(it - nE);
    }
  }
  MF_PHASE_MARK(5);

  {
    // ---- F: NN softmin statistics: rows (side 1) and columns (side 2) -------
    // and, on the 9-warp shape, the V-S contacts on the warps the NN items
    // leave idle (dense warps: a V-S item is ~1/6 of a pair).
    for (int i = tid; i < 10 * n_here; i += nth) env(i / 10).hpart()[i % 10] = 0.0;  // G's partials
    // 2 adjacent lanes per row / column split its elements (shuffle-reduced in
    // a fixed order; measured: 4 lanes +0.6%, 1 lane -0.2% but serial for long rows)
    constexpr int kNL = 2;
    const int nrc = m1 + m2;
    const int nF = full ? kNL * n_here * nrc : 0;
    for (int it = tid; it < nF; it += nth) {
      const int ql = it & (kNL - 1);
      int e, r;
      fdivmod(it / kNL, p.div_nrc, e, r);
      const EnvView ev = env(e);
      const bool row = r < m1;
      const int n = row ? m2 : m1;
      const unsigned gm = ((1u << kNL) - 1u) << ((tid & 31) & ~(kNL - 1));
      double m = INFINITY;
      for (int j = ql; j < n; j += kNL) {  // minimum shift (argmin_s, smooth_ops.hpp:130-136)
        const int i = row ? r * m2 + j : j * m2 + (r - m1);
        const double d = ev.dbar(i);
        m = d < m ? d : m;
      }
#pragma unroll
      for (int o = 1; o < kNL; o <<= 1) {
        const double mo = __shfl_xor_sync(gm, m, o);
        m = mo < m ? mo : m;
      }
      double tot = 0.0;
      for (int j = ql; j < n; j += kNL) {
        const int i = row ? r * m2 + j : j * m2 + (r - m1);
        tot += (double)nn_weight((m - ev.dbar(i)) * c.inv_tau_nn);
      }
#pragma unroll
      for (int o = 1; o < kNL; o <<= 1) tot += __shfl_xor_sync(gm, tot, o);
      if (ql == 0) {
        ev.nnstat()[3 * r] = m;  // stride 3 (odd): conflict-free reads in G
        ev.nnstat()[3 * r + 1] = rcp_d(tot);  // tot >= 1
      }
    }
    if constexpr (!kVsE && !kVsX) {
      const int vs0 = ((nF + 31) & ~31) % nth;  // first thread of the first warp after the NN items
      for (int it = tid >= vs0 ? tid - vs0 : tid - vs0 + nth; it < n_here * nvs; it += nth) {
        int e, r;
        fdivmod(it, p.div_nvs, e, r);
        const EnvView ev = env(e);
        const double* q = ev.vslot(r);
        float* dst = p.contacts + ((env0 + e) * C + r) * 8;
        const float act = r < n1 ? vs_contact<K2>(S2.sdf, ev.R(1), ev.t(1), d3(q[0], q[1], q[2]), c, ev.vsdist() + r, dst)
                                 : vs_contact<K1>(S1.sdf, ev.R(0), ev.t(0), d3(q[0], q[1], q[2]), c, ev.vsdist() + r, dst);
        if (p.act_mask && act > p.act_thr) atomicOr(ev.amask() + (r >> 5), 1u << (r & 31));
        if (p.src) {
          int* sp = p.src + ((env0 + e) * C + r) * 2;
          sp[0] = ev.prov()[r];
          sp[1] = -1;
        }
      }
    }
  }
  MF_PHASE_MARK(6);

  if (full) {
    // ---- G: activity product + fixed-layout E-E output (303-330) -----------
    // Warp-uniform trip count (lanes past the end idle), so each warp also
    // reduces its pairs' E-E distances per env (segmented shuffle reduction,
    // fixed order) into one partial per (env, warp) for H.
    const int warp = tid >> 5, lane = tid & 31;
    const int total = n_here * P;
    for (int base = warp << 5; base < total; base += nth) {
      const int it = base + lane;
      const bool on = it < total;
      int e = 0, i = 0;
      double contrib = 0.0;
      if (on) {
        int k, l;
        fdivmod(it, p.div_pairs, e, i);
        fdivmod(i, p.div_m2, k, l);
        const EnvView ev = env(e);
        const double* rec = ev.pair(i);
        const double* ns = ev.nnstat();
        const double dg = rec[3];
        const double nn1 = (double)nn_weight((ns[3 * k] - dg) * c.inv_tau_nn) * ns[3 * k + 1];
        const double nn2 = (double)nn_weight((ns[3 * (m1 + l)] - dg) * c.inv_tau_nn) * ns[3 * (m1 + l) + 1];
        const double pen1 = rec[6], pen2 = rec[14], con = rec[16], clash = rec[15], cont = rec[7];
        const float act1 = (float)(con * pen1 * nn1 * clash * cont);
        const float act2 = (float)(con * pen2 * nn2 * clash * cont);
        const double g1 = rec[4], g2 = rec[5];
        const float d1 = (float)(g1 * dg), d2 = (float)(g2 * dg);
        contrib = (double)d1 + (double)d2;
        const int64_t row = (env0 + e) * C + n1 + n2 + 2 * i;
        float* dst = p.contacts + row * 8;
        // contacts (manifold.hpp:303-330): dist = sign * dbar, normal = sign * nbar
        store_contact(dst, (float)rec[0], (float)rec[1], (float)rec[2], d1, (float)(rec[11] * g1),
                      (float)(rec[12] * g1), (float)(rec[13] * g1), act1);
        store_contact(dst + 8, (float)rec[8], (float)rec[9], (float)rec[10], d2, (float)(rec[11] * g2),
                      (float)(rec[12] * g2), (float)(rec[13] * g2), act2);
        if (p.act_mask) {
          const int c0 = n1 + n2 + 2 * i;  // contact index of side 1; side 2 follows
          if (act1 > p.act_thr) atomicOr(ev.amask() + (c0 >> 5), 1u << (c0 & 31));
          if (act2 > p.act_thr) atomicOr(ev.amask() + ((c0 + 1) >> 5), 1u << ((c0 + 1) & 31));
        }
        if (p.src) {
          int* sp = p.src + row * 2;
          const int sa = ev.prov()[n1 + n2 + k], sb = ev.prov()[n1 + n2 + m1 + l];
          sp[0] = sa; sp[1] = sb; sp[2] = sa; sp[3] = sb;
        }
        if (p.ee) {  // EeIndicatorMatrices (manifold.hpp:41-52)
          float* E = p.ee + (env0 + e) * 9 * P;
          E[i] = (float)dg;
          E[P + i] = (float)con;
          E[2 * P + i] = (float)pen1;
          E[3 * P + i] = (float)pen2;
          E[4 * P + i] = (float)nn1;
          E[5 * P + i] = (float)nn2;
          E[6 * P + i] = (float)clash;
          E[7 * P + i] = act1;
          E[8 * P + i] = act2;
        }
      }
      if (p.mean_dist) {
        // segmented sum over the warp's lanes of the same env (contiguous runs)
        const int seg = on ? e : -1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double vo = __shfl_down_sync(0xffffffffu, contrib, o);
          const int so = __shfl_down_sync(0xffffffffu, seg, o);
          if (lane + o < 32 && so == seg) contrib += vo;
        }
        const int sprev = __shfl_up_sync(0xffffffffu, seg, 1);
        if (on && (lane == 0 || sprev != seg)) env(e).hpart()[warp] += contrib;  // this warp's run of env e
        __syncwarp();
      }
    }
  }
  MF_PHASE_MARK(7);

  // ---- H: mean contact distance (manifold.hpp:379-384): one warp per env sums
  // the V-S distances and the G partials, fixed order; and the env's activity
  // mask + count for the compaction extra ------------------------------------
  if (p.act_mask) {
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
    for (int e = warp; e < n_here; e += nwarps) {
      const EnvView ev = env(e);
      int cnt = 0;
      for (int w = lane; w < p.mask_words; w += 32) {
        const uint32_t m = ev.amask()[w];
        p.act_mask[(env0 + e) * p.mask_words + w] = m;
        cnt += __popc(m);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      if (lane == 0) p.act_count[env0 + e] = cnt;
    }
  }
  if (p.mean_dist) {
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
    for (int e = warp; e < n_here; e += nwarps) {
      const EnvView ev = env(e);
      double acc = 0.0;
      if constexpr (kVsX) {  // vs_kernel left the V-S share (its fixed-order sum) in mean_dist
        if (lane == 0) acc = (double)p.mean_dist[env0 + e];
      } else {
        for (int r = lane; r < n1 + n2; r += 32) acc += (double)ev.vsdist()[r];
      }
      if (full && lane < nwarps) acc += ev.hpart()[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.mean_dist[env0 + e] = (float)(acc / (double)C);
    }
  }
  MF_PHASE_MARK_DBG(8);
}

// V-S contacts of pass-through vertex sets as their own launch (box-box): G
// lanes per env (a power of two >= n1 + n2), frames from the workspace, the
// env's V-S distance sum (fixed shuffle order) left in mean_dist for the
// manifold kernel's H phase. Keeps the ~1/6-pair V-S items off the manifold
// CTAs, whose F phase then holds only the short NN statistics.
template <int K1, int K2>
__global__ void __launch_bounds__(256) vs_kernel(const __grid_constant__ ManifoldParams p, int G) {
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t e = gt / G;
  const int r = (int)(gt - e * G);
  const int n1 = p.n1, nvs = p.n1 + p.n2, C = p.n_contacts;
  const bool act = e < p.n_env && r < nvs;
  double d = 0.0;
  float act_v = 0.0f;
  if (act) {
    const int s = r < n1 ? 0 : 1;
    const int vi = s == 0 ? r : r - n1;
    const double* f1 = p.frames1 + 12 * e * p.stride1;
    const double* f2 = p.frames2 + 12 * e * p.stride2;
    const double* fs = s == 0 ? f1 : f2;
    const double* fo = s == 0 ? f2 : f1;
    const double3 pw = to_world(fs, fs + 9, ld_vert(p.side[s].verts, vi));
    float dist;
    float* dst = p.contacts + (e * C + r) * 8;
    if (s == 0) act_v = vs_contact<K2>(p.side[1].sdf, fo, fo + 9, pw, p.cfg, &dist, dst);
    else act_v = vs_contact<K1>(p.side[0].sdf, fo, fo + 9, pw, p.cfg, &dist, dst);
    if (p.src) {
      int* sp = p.src + (e * C + r) * 2;
      sp[0] = vi;
      sp[1] = -1;
    }
    d = (double)dist;
  }
  for (int o = G >> 1; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  if (act && r == 0 && p.mean_dist) p.mean_dist[e] = (float)d;
  if (p.act_mask) {  // the env's V-S bits (nvs <= 32: word 0), completed by the manifold kernel
    const unsigned b = __ballot_sync(0xffffffffu, act && act_v > p.act_thr);
    const int g0 = (threadIdx.x & 31) & ~(G - 1);
    if (act && r == 0) p.act_mask[e * p.mask_words] = G == 32 ? b : (b >> g0) & ((1u << G) - 1u);
  }
}

[[maybe_unused]] int launch_frames(const double* poses1, int64_t stride1, int64_t n1, double* frames1, const double* poses2,
                  int64_t stride2, int64_t n2, double* frames2, cudaStream_t s) {
  if (n1 + n2 <= 0) return 0;
  note_launch();
  frames_kernel<<<(unsigned)((n1 + n2 + 255) / 256), 256, 0, s>>>(poses1, stride1, n1, frames1, poses2, stride2, n2,
                                                                  frames2);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <int K1, int K2, bool kGP = false, bool kVsX = false>
int launch_kind(const ManifoldParams& p, int threads, int grid, size_t smem, cudaStream_t s);

// Both sides the same compile-time superquadric kind K with pass-through
// vertex sets (box-box): V-S contacts in their own launch (vs_kernel), then the
// kVsX manifold instantiation. Returns -1 when the case does not apply.
template <int K>
int launch_same_kind(const ManifoldParams& p, int threads, int grid, size_t smem, cudaStream_t s) {
  const int nvs = p.n1 + p.n2;
  if (box_box(K, K) && !p.side[0].topk_v && !p.side[1].topk_v && nvs > 0 && nvs <= 32) {
    ManifoldParams q = p;
    q.vs_ext = 1;
    int G = 1;
    while (G < nvs) G <<= 1;
    const int64_t lanes = p.n_env * G;
    note_launch();
    vs_kernel<K, K><<<(unsigned)((lanes + 255) / 256), 256, 0, s>>>(q, G);
    if (cudaGetLastError() != cudaSuccess) return 1;
    return launch_kind<K, K, false, true>(q, threads, grid, smem, s);
  }
  return launch_kind<K, K>(p, threads, grid, smem, s);
}

template <int K1, int K2, bool kGP, bool kVsX>
int launch_kind(const ManifoldParams& p, int threads, int grid, size_t smem, cudaStream_t s) {
  static PerDeviceOnce configured;
  configured([] {  // per device: the attribute does not carry across devices
    allow_max_dynamic_smem(manifold_kernel<K1, K2, kGP, kVsX>);
  });
  note_launch();
  manifold_kernel<K1, K2, kGP, kVsX><<<grid, threads, smem, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace

}  // namespace cmgb
