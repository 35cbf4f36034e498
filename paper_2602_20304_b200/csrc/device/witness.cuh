// Branch-free analytical active-set witness solvers (witness.hpp:74-227).
//
// The E-E witness feeds the signed normal n = sign_s(n_b . de/|de|) de/|de|,
// whose sensitivity to a tangential witness error is (1/|de|)(1 + 1/tau_sign):
// matching the reference's FP64 outputs to 1e-5 at |de| ~ 1e-3 needs ~1e-10
// witness accuracy, so the QP, its soft operators and the blend are FP64 on
// the B200's half-rate DFMA pipe. The soft and hard modes are selected by a
// warp-uniform flag.
#pragma once

#include "../common.h"
#include "dmath.cuh"
#include "dual.cuh"

namespace cmgb {

// Scalars: T is the value type of the QP (double, or Dual<N> for the pose
// Jacobian kernel); I is the arithmetic type of the soft indicators (sigmoid /
// softplus / softmin weights) -- T itself on the manifold path (the witness
// feeds the amplified E-E normal, see above), float for the K6 witness
// batches, whose outputs are the witness points themselves: there an indicator
// error of 1e-7 moves alpha by <= tau_clip * 1e-7 (clip) or 1e-7 |cand - cand'|
// (weights / blend), far inside 1e-6 + 1e-5 |p|. Indicator
// ARGUMENTS are always formed in T (FP64) and rounded once.

// exp(-|x - 1| / tau) from a = exp(-|x| / tau) and C = exp(-1 / tau):
// |x| and |x - 1| differ by exactly 1, so b = a C (x < 0), C / a (0 <= x <= 1),
// a / C (x > 1) -- one exponential per softplus / sigmoid pair. The partner
// identities hold as functions of x, so Dual tangents are exact too.
template <class I>
__device__ __forceinline__ I partner_exp(const I& x, const I& a, double C, double inv_C,
                                         double inv_tau, int pair) {
  if (!pair) return exp_d(-fabs(x - I(1.0)) * I(inv_tau));
  if constexpr (std::is_same_v<I, float>) {
    // branch-free (the lanes of a warp hold unrelated pairs): one reciprocal
    // always, then selects
    const float r = rcp_d(a);
    const float lo = a * (float)C, mid = (float)C * r, hi = a * (float)inv_C;
    return pv(x) < 0.0f ? lo : (pv(x) <= 1.0f ? mid : hi);
  } else {
    return pv(x) < 0.0 ? a * I(C) : (pv(x) <= 1.0 ? I(C) * rcp_d(a) : a * I(inv_C));
  }
}

template <class I, class T>
__device__ __forceinline__ I to_ind(const T& x) {
  if constexpr (std::is_same_v<I, float>) return (float)pv(x);
  else return x;
}

// max(x, 0) as one compare + selects for double (fmax's NaN handling costs
// five instructions; the two agree for every non-NaN x and give 0 for NaN).
template <class T>
__device__ __forceinline__ T pos0(const T& x) {
  if constexpr (std::is_same_v<T, double>) return x > 0.0 ? x : 0.0;
  else return fmax(x, T(0.0));
}

// Compile-time operator mode of the witness solvers: kH < 0 reads the
// config's hard_ops flag at run time, 0 / 1 fix soft / hard (the K6 kernels
// dispatch on the flag once, so the other mode's code is not issued).
template <int kH>
__device__ __forceinline__ bool hard_mode(const DevCfg& c) {
  if constexpr (kH < 0) return c.hard_ops != 0;
  else return kH == 1;
}

// clip01 (witness.hpp:45-52): clip_s(x, 0, 1, tau) = softplus(x) - softplus(x - 1)
// (smooth_ops.hpp:66-89) = [max(x,0) - max(x-1,0)] + tau log1p((a - b) / (1 + b)),
// a = exp(-|x|/tau), b = exp(-|x-1|/tau); hard: clamp.
template <class T, class I = T, int kH = -1>
__device__ __forceinline__ T clip01(const T& x, const DevCfg& c) {
  if constexpr (is_dual<T>::value) {
    if (!hard_mode<kH>(c)) {  // Dual: the double formula + its analytic derivative
      const double xv = x.v;  // d clip / dx = sigma(x/tau) - sigma((x-1)/tau)
      const double a = exp_d(-fabs(xv) * c.inv_tau_clip);
      const double b = partner_exp(xv, a, c.clip_C, c.inv_clip_C, c.inv_tau_clip, c.pair_exp);
      const double ia = rcp_d(1.0 + a), ib = rcp_d(1.0 + b);
      const double corr = c.tau_clip * log_d((1.0 + a) * ib);
      const double s1 = xv >= 0.0 ? ia : a * ia, s2 = xv >= 1.0 ? ib : b * ib;
      return T::chain((fmax(xv, 0.0) - fmax(xv - 1.0, 0.0)) + corr, s1 - s2, x);
    }
  }
  if (hard_mode<kH>(c)) return fmin(fmax(x, T(0.0)), T(1.0));
  const I xi = to_ind<I>(x);
  const I a = exp_d(-fabs(xi) * I(c.inv_tau_clip));
  const I b = partner_exp(xi, a, c.clip_C, c.inv_clip_C, c.inv_tau_clip, c.pair_exp);
  // tau (log1p(a) - log1p(b)) = tau log((1 + a) / (1 + b)); the quotient is
  // formed in I (FP64 on the manifold path: absolute error ~1e-16, scaled by tau)
  const I corr = I(c.tau_clip) * log_d((I(1.0) + a) * rcp_d(I(1.0) + b));
  return (pos0(x) - pos0(x - 1.0)) + T(corr);
}

// within01 (witness.hpp:54-61): gamma = sigma(x/tau) sigma((1-x)/tau) and its
// complement 1 - gamma = (1 - s1) + s1 (1 - s2), both relatively accurate;
// hard mode: [0 <= x <= 1] exactly (within_hard, smooth_ops.hpp:204-206).
template <class T, class I = T>
__device__ __forceinline__ void within01(const T& x, double inv_tau, double C, double inv_C, int pair,
                                         int hard, I* g, I* omg) {
  if (hard) {
    const bool in = pv(x) >= 0.0 && pv(x) <= 1.0;
    *g = in ? 1.0 : 0.0;
    *omg = in ? 0.0 : 1.0;
    return;
  }
  if constexpr (is_dual<T>::value && std::is_same_v<T, I>) {
    // Dual: the double formula + d gamma / dx = gamma (c1 - c2) / tau
    const double xv = x.v;
    const double e1 = exp_d(-fabs(xv) * inv_tau), e2 = partner_exp(xv, e1, C, inv_C, inv_tau, pair);
    const double i1 = rcp_d(1.0 + e1), i2 = rcp_d(1.0 + e2);
    const double s1 = xv >= 0.0 ? i1 : e1 * i1, s2 = xv <= 1.0 ? i2 : e2 * i2;
    const double c1 = xv >= 0.0 ? e1 * i1 : i1, c2 = xv <= 1.0 ? e2 * i2 : i2;
    const double gv = s1 * s2, ov = c1 + s1 * c2;
    const double dg = gv * (c1 - c2) * inv_tau;
    *g = I::chain(gv, dg, x);
    *omg = I::chain(ov, -dg, x);
    return;
  } else {
    const I xi = to_ind<I>(x);
    const I e1 = exp_d(-fabs(xi) * I(inv_tau));               // sigma(x/tau) pair
    const I e2 = partner_exp(xi, e1, C, inv_C, inv_tau, pair);  // sigma((1-x)/tau) pair
    const I i1 = rcp_d(I(1.0) + e1), i2 = rcp_d(I(1.0) + e2);
    const bool ge0 = pv(x) >= 0.0, le1 = pv(x) <= 1.0;
    const I s1 = ge0 ? i1 : e1 * i1, c1 = ge0 ? e1 * i1 : i1;
    const I s2 = le1 ? i2 : e2 * i2, c2 = le1 ? e2 * i2 : i2;
    *g = s1 * s2;
    *omg = c1 + s1 * c2;
  }
}

// Product of indicators and its complement: 1 - ab = (1 - a) + a (1 - b).
template <class I>
__device__ __forceinline__ void within_and(const I& a, const I& oma, const I& b, const I& omb, I* g,
                                           I* omg) {
  *g = a * b;
  *omg = oma + a * omb;
}

// argmin over n costs: soft (argmin_s, smooth_ops.hpp:126-144) or first-min
// one-hot (argmin_hard, 210-218). Returns the winner = first argmax weight.
// Costs in T; weights in I from the T-exact differences m - cost_i.
template <int N, class T, class I>
__device__ __forceinline__ int pick_min(const T (&cost)[N], I (&w)[N], double inv_tau, int hard) {
  if constexpr (is_dual<T>::value && std::is_same_v<T, I>) {
    if (!hard) {  // Dual: primal softmin weights, dw_i = w_i (sum_j w_j dc_j - dc_i) / tau
      int best = 0;
      double m = cost[0].v;
#pragma unroll
      for (int i = 1; i < N; ++i)
        if (cost[i].v < m) {
          best = i;
          m = cost[i].v;
        }
      double wv[N], total = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        wv[i] = i == best ? 1.0 : exp_d((m - cost[i].v) * inv_tau);
        total += wv[i];
      }
      const double inv = rcp_d(total);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        wv[i] *= inv;
        w[i].v = wv[i];
      }
      constexpr int ND = sizeof(cost[0].d) / sizeof(double);
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        double avg = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) avg = fma(wv[j], cost[j].d[d], avg);
#pragma unroll
        for (int i = 0; i < N; ++i) w[i].d[d] = wv[i] * inv_tau * (avg - cost[i].d[d]);
      }
      return best;
    }
  }
  int best = 0;
  T m = cost[0];
#pragma unroll
  for (int i = 1; i < N; ++i)
    if (pv(cost[i]) < pv(m)) {
      best = i;
      m = cost[i];
    }
  if (hard) {
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = i == best ? 1.0 : 0.0;
    return best;
  }
  I total = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    w[i] = i == best ? I(1.0) : exp_d(to_ind<I>((m - cost[i]) * inv_tau));  // exp(0) = 1 at the minimum
    total += w[i];
  }
  const I inv = rcp_d(total);
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] *= inv;
  return best;
}

template <class T>
struct QpSolT {
  T a1, a2;
  T gamma;
  int label;
};
using QpSol = QpSolT<double>;

// solve_box_qp_2 (witness.hpp:74-121), erratum-fixed cost 4 (witness.hpp:99).
// kIeee: IEEE quotients instead of the one-Newton reciprocals (the unconstrained
// solve of a near-parallel pair at lambda = 1e-6 amplifies a 1e-12 quotient
// error ~1e4-fold; the reference-precision K6 solver opts in).
template <class T, class I = T, bool kIeee = false, int kH = -1>
__device__ __forceinline__ QpSolT<T> solve_box_qp_2(const T& q1, const T& q2, const T& q3, const T& c1,
                                                    const T& c2, const DevCfg& c) {
  T q2_over_q1, q2_over_q3, c1_over_q1, c2_over_q3, a1u, a2u;
  if constexpr (kIeee) {
    q2_over_q1 = q2 / q1;
    q2_over_q3 = q2 / q3;
    c1_over_q1 = c1 / q1;
    c2_over_q3 = c2 / q3;
    a1u = (q2 * c2_over_q3 - c1) / (q1 - q2 * q2_over_q3);
    a2u = (q2 * c1_over_q1 - c2) / (q3 - q2 * q2_over_q1);
  } else {
    const T i1 = rcp_d(q1), i3 = rcp_d(q3);
    q2_over_q1 = q2 * i1;
    q2_over_q3 = q2 * i3;
    c1_over_q1 = c1 * i1;
    c2_over_q3 = c2 * i3;
    a1u = div_d(q2 * c2_over_q3 - c1, q1 - q2 * q2_over_q3);
    a2u = div_d(q2 * c1_over_q1 - c2, q3 - q2 * q2_over_q1);
  }
  const T a1_1_a2 = clip01<T, I, kH>(-(q2_over_q3 + c2_over_q3), c);
  const T a1_0_a2 = clip01<T, I, kH>(-c2_over_q3, c);
  const T a2_1_a1 = clip01<T, I, kH>(-(q2_over_q1 + c1_over_q1), c);
  const T a2_0_a1 = clip01<T, I, kH>(-c1_over_q1, c);
  const T cost[4] = {
      0.5 * (q1 + 2.0 * q2 * a1_1_a2 + q3 * a1_1_a2 * a1_1_a2) + c1 + c2 * a1_1_a2,
      0.5 * q3 * a1_0_a2 * a1_0_a2 + c2 * a1_0_a2,
      0.5 * (q1 * a2_1_a1 * a2_1_a1 + 2.0 * q2 * a2_1_a1 + q3) + c1 * a2_1_a1 + c2,
      0.5 * q1 * a2_0_a1 * a2_0_a1 + c1 * a2_0_a1,
  };
  I wi[4];
  const int best = pick_min<4>(cost, wi, c.inv_tau_min, hard_mode<kH>(c));
  const T w[4] = {T(wi[0]), T(wi[1]), T(wi[2]), T(wi[3])};
  // constrained = sum_i w_i cand_i (witness.hpp:101-113)
  const T k0 = w[0] + w[2] * a2_1_a1 + w[3] * a2_0_a1;
  const T k1 = w[0] * a1_1_a2 + w[1] * a1_0_a2 + w[2];
  I g1, o1, g2, o2, in, out;
  within01<T, I>(a1u, c.inv_tau_comp, c.comp_C, c.inv_comp_C, c.pair_exp, hard_mode<kH>(c), &g1, &o1);
  within01<T, I>(a2u, c.inv_tau_comp, c.comp_C, c.inv_comp_C, c.pair_exp, hard_mode<kH>(c), &g2, &o2);
  within_and(g1, o1, g2, o2, &in, &out);
  QpSolT<T> s;
  s.a1 = a1u * T(in) + k0 * T(out);
  s.a2 = a2u * T(in) + k1 * T(out);
  s.gamma = T(in);
  s.label = best | ((pv(in) >= 0.5) << 2);
  return s;
}

// ee_witness Q/c construction (witness.hpp:137-158) for edges given in a
// common frame: Q = A^T A + lambda I, c = b^T A - lambda/2, A = [t1, -t2].
template <class T = double, class I = T, bool kIeee = false, int kH = -1>
__device__ __forceinline__ QpSolT<T> ee_qp(vec3<T> e1a, vec3<T> e1b, vec3<T> e2a, vec3<T> e2b,
                                           const DevCfg& c) {
  const vec3<T> t1 = e1b - e1a;
  const vec3<T> t2n = e2a - e2b;
  const vec3<T> b = e1a - e2a;
  return solve_box_qp_2<T, I, kIeee, kH>(ddot(t1, t1) + c.lambda, ddot(t1, t2n), ddot(t2n, t2n) + c.lambda,
                              ddot(b, t1) - 0.5 * c.lambda, ddot(b, t2n) - 0.5 * c.lambda, c);
}

// vf_witness (witness.hpp:163-227): clipped edge projections over the full
// edge length, soft/hard argmin of distances, plane projection, barycentric
// inside test, blend. Returns the closest point; label as above over 3.
// Geometry FP64 (normalisations by the one-Newton rsqrt, 1e-12 relative);
// indicators in I.
template <class I = double, int kH = -1>
__device__ __forceinline__ double3 vf_witness(double3 v, double3 t0, double3 t1, double3 t2,
                                              const DevCfg& c, int* label) {
  const double3 d10 = t1 - t0, d21 = t2 - t1, d20 = t2 - t0;
  const double3 dv0 = v - t0, dv1 = v - t1;
  const double guard = 1e-12;  // SmoothingConfig::kEdgeNormalEps
  const double l10 = ddot(d10, d10) + guard, l21 = ddot(d21, d21) + guard, l20 = ddot(d20, d20) + guard;
  const double r10 = rsqrt_d(l10), r21 = rsqrt_d(l21), r20 = rsqrt_d(l20);
  const double len10 = l10 * r10, len21 = l21 * r21, len20 = l20 * r20;
  const double3 u10 = dscale(d10, r10), u21 = dscale(d21, r21), u20 = dscale(d20, r20);
  // clip over [0, len] (arc-length parameterisation, witness.hpp:181-189):
  // softplus(s) - softplus(s - len) = [max(s,0) - max(s-len,0)]
  //   + tau log((1 + exp(-|s|/tau)) / (1 + exp(-|s-len|/tau)))
  auto clip_len = [&](double s, double len) -> double {
    if (hard_mode<kH>(c)) return fmin(fmax(s, 0.0), len);
    const I a = exp_d(to_ind<I>(-fabs(s) * c.inv_tau_clip));
    const I b = exp_d(to_ind<I>(-fabs(s - len) * c.inv_tau_clip));
    const I corr = I(c.tau_clip) * log_d((I(1.0) + a) * rcp_d(I(1.0) + b));
    return (pos0(s) - pos0(s - len)) + (double)corr;
  };
  const double3 on1 = t0 + u10 * clip_len(ddot(dv0, u10), len10);
  const double3 on2 = t1 + u21 * clip_len(ddot(dv1, u21), len21);
  const double3 on3 = t0 + u20 * clip_len(ddot(dv0, u20), len20);
  const double3 q1 = v - on1, q2 = v - on2, q3 = v - on3;
  // distances as x rsqrt(x) (1.3e-12 relative: they only enter the softmin
  // weights, scaled by 1/tau_min) instead of three IEEE square roots
  auto dist = [](double x) { return x > 0.0 ? x * rsqrt_d(x) : 0.0; };
  const double cost[3] = {dist(ddot(q1, q1)), dist(ddot(q2, q2)), dist(ddot(q3, q3))};
  I w[3];
  const int best = pick_min<3>(cost, w, c.inv_tau_min, hard_mode<kH>(c));
  const double3 cons = on1 * (double)w[0] + on2 * (double)w[1] + on3 * (double)w[2];
  const double3 n_raw = d3(d10.y * d20.z - d10.z * d20.y, d10.z * d20.x - d10.x * d20.z,
                           d10.x * d20.y - d10.y * d20.x);
  const double rn = rsqrt_d(ddot(n_raw, n_raw) + guard);  // 1 / n_norm
  const double3 n = dscale(n_raw, rn);
  const double3 dvp0 = dv0 - n * ddot(dv0, n);
  const double3 plane = t0 + dvp0;
  auto cross = [](double3 a, double3 b) {
    return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
  };
  const double bv = ddot(cross(d10, dvp0), n) * rn;
  const double bu = ddot(cross(dvp0, d20), n) * rn;
  const double bw = 1.0 - bu - bv;
  I gu, ou, gv, ov, gw, ow, guv, ouv, in, out;
  within01<double, I>(bu, c.inv_tau_comp, c.comp_C, c.inv_comp_C, c.pair_exp, hard_mode<kH>(c), &gu, &ou);
  within01<double, I>(bv, c.inv_tau_comp, c.comp_C, c.inv_comp_C, c.pair_exp, hard_mode<kH>(c), &gv, &ov);
  within01<double, I>(bw, c.inv_tau_comp, c.comp_C, c.inv_comp_C, c.pair_exp, hard_mode<kH>(c), &gw, &ow);
  within_and(gu, ou, gv, ov, &guv, &ouv);
  within_and(guv, ouv, gw, ow, &in, &out);
  if (label) *label = best | ((pv(in) >= 0.5) << 2);
  return plane * (double)in + cons * (double)out;
}

}  // namespace cmgb
