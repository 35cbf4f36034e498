// Branch-free analytical active-set witness solvers (witness.hpp:74-227).
//
// Linear algebra in FP64 (the unconstrained minimiser -Q^-1 c cancels badly
// for near-parallel edges at lambda = 1e-6); the smooth operators' SFU work
// (softplus / sigmoid / softmin weights) in FP32 on FP64-exact arguments.
// The soft and hard modes are selected by a warp-uniform flag.
#pragma once

#include "../common.h"
#include "dmath.cuh"

namespace cmgb {

// clip01 (witness.hpp:45-52): clip_s(x, 0, 1, tau) =
//   softplus(x) - softplus(x - 1), softplus(y) = max(y, 0) + tau log1p(exp(-|y|/tau)).
__device__ __forceinline__ double clip01(double x, const DevCfg& c) {
  if (c.hard_ops) return fmin(fmax(x, 0.0), 1.0);
  const double xm1 = x - 1.0;
  const double exact = fmax(x, 0.0) - fmax(xm1, 0.0);
  const float corr = softplus_corr((float)fabs(x) * c.inv_tau_clip, c.tau_clip) -
                     softplus_corr((float)fabs(xm1) * c.inv_tau_clip, c.tau_clip);
  return exact + (double)corr;
}

// within01 (witness.hpp:54-61): sigma(x/tau) sigma((1-x)/tau) | [0 <= x <= 1].
__device__ __forceinline__ float within01(double x, float inv_tau, int hard) {
  if (hard) return (x >= 0.0 && x <= 1.0) ? 1.0f : 0.0f;
  return sigmoidf((float)x * inv_tau) * sigmoidf((float)(1.0 - x) * inv_tau);
}

// argmin over n costs: soft (argmin_s, smooth_ops.hpp:126-144) or first-min
// one-hot (argmin_hard, 210-218). Returns the label (argmax weight, first).
template <int N>
__device__ __forceinline__ int pick_min(const double (&cost)[N], float (&w)[N], float inv_tau,
                                        int hard) {
  int best = 0;
#pragma unroll
  for (int i = 1; i < N; ++i)
    if (cost[i] < cost[best]) best = i;
  if (hard) {
#pragma unroll
    for (int i = 0; i < N; ++i) w[i] = i == best ? 1.0f : 0.0f;
    return best;
  }
  const double m = cost[best];
  float total = 0.0f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    w[i] = __expf((float)(m - cost[i]) * inv_tau);
    total += w[i];
  }
  const float inv = rcpf(total);
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] *= inv;
  return best;  // exp(0) is the unique maximum weight except at exact ties
}

struct QpSol {
  double a1, a2;
  float gamma;
  int label;
};

// solve_box_qp_2 (witness.hpp:74-121), erratum-fixed cost 4 (witness.hpp:99).
__device__ __forceinline__ QpSol solve_box_qp_2(double q1, double q2, double q3, double c1,
                                                double c2, const DevCfg& c) {
  const double inv_q1 = 1.0 / q1, inv_q3 = 1.0 / q3;
  const double q2_over_q1 = q2 * inv_q1, q2_over_q3 = q2 * inv_q3;
  const double c1_over_q1 = c1 * inv_q1, c2_over_q3 = c2 * inv_q3;
  const double a1u = (q2 * c2_over_q3 - c1) / (q1 - q2 * q2_over_q3);
  const double a2u = (q2 * c1_over_q1 - c2) / (q3 - q2 * q2_over_q1);
  const double a1_1_a2 = clip01(-(q2_over_q3 + c2_over_q3), c);
  const double a1_0_a2 = clip01(-c2_over_q3, c);
  const double a2_1_a1 = clip01(-(q2_over_q1 + c1_over_q1), c);
  const double a2_0_a1 = clip01(-c1_over_q1, c);
  const double cost[4] = {
      0.5 * (q1 + 2.0 * q2 * a1_1_a2 + q3 * a1_1_a2 * a1_1_a2) + c1 + c2 * a1_1_a2,
      0.5 * q3 * a1_0_a2 * a1_0_a2 + c2 * a1_0_a2,
      0.5 * (q1 * a2_1_a1 * a2_1_a1 + 2.0 * q2 * a2_1_a1 + q3) + c1 * a2_1_a1 + c2,
      0.5 * q1 * a2_0_a1 * a2_0_a1 + c1 * a2_0_a1,
  };
  float w[4];
  const int best = pick_min<4>(cost, w, c.inv_tau_min, c.hard_ops);
  const double k0 = (double)w[0] + (double)w[2] * a2_1_a1 + (double)w[3] * a2_0_a1;
  const double k1 = (double)w[0] * a1_1_a2 + (double)w[1] * a1_0_a2 + (double)w[2];
  const float inside =
      within01(a1u, c.inv_tau_comp, c.hard_ops) * within01(a2u, c.inv_tau_comp, c.hard_ops);
  const double in = (double)inside, out = 1.0 - in;
  QpSol s;
  s.a1 = a1u * in + k0 * out;
  s.a2 = a2u * in + k1 * out;
  s.gamma = inside;
  s.label = best | ((inside >= 0.5f) << 2);
  return s;
}

// ee_witness Q/c construction (witness.hpp:137-158) for edges given in a
// common frame: Q = A^T A + lambda I, c = b^T A - lambda/2, A = [t1, -t2].
__device__ __forceinline__ QpSol ee_qp(double3 e1a, double3 e1b, double3 e2a, double3 e2b,
                                       const DevCfg& c) {
  const double3 t1 = e1b - e1a;
  const double3 t2n = e2a - e2b;
  const double3 b = e1a - e2a;
  return solve_box_qp_2(ddot(t1, t1) + c.lambda, ddot(t1, t2n), ddot(t2n, t2n) + c.lambda,
                        ddot(b, t1) - 0.5 * c.lambda, ddot(b, t2n) - 0.5 * c.lambda, c);
}

// vf_witness (witness.hpp:163-227): clipped edge projections over the full
// edge length, soft/hard argmin of distances, plane projection, barycentric
// inside test, blend. Returns the closest point; label as above over 3.
__device__ __forceinline__ double3 vf_witness(double3 v, double3 t0, double3 t1, double3 t2,
                                              const DevCfg& c, int* label) {
  const double3 d10 = t1 - t0, d21 = t2 - t1, d20 = t2 - t0;
  const double3 dv0 = v - t0, dv1 = v - t1;
  const double guard = 1e-12;
  const double len10 = sqrt(ddot(d10, d10) + guard);
  const double len21 = sqrt(ddot(d21, d21) + guard);
  const double len20 = sqrt(ddot(d20, d20) + guard);
  const double3 u10 = d10 * (1.0 / len10), u21 = d21 * (1.0 / len21), u20 = d20 * (1.0 / len20);
  auto clip_len = [&](double s, double len) -> double {
    if (c.hard_ops) return fmin(fmax(s, 0.0), len);
    const double sm = s - len;
    const double exact = fmax(s, 0.0) - fmax(sm, 0.0);
    const float corr = softplus_corr((float)fabs(s) * c.inv_tau_clip, c.tau_clip) -
                       softplus_corr((float)fabs(sm) * c.inv_tau_clip, c.tau_clip);
    return exact + (double)corr;
  };
  const double3 on1 = t0 + u10 * clip_len(ddot(dv0, u10), len10);
  const double3 on2 = t1 + u21 * clip_len(ddot(dv1, u21), len21);
  const double3 on3 = t0 + u20 * clip_len(ddot(dv0, u20), len20);
  const double3 r1 = v - on1, r2 = v - on2, r3 = v - on3;
  const double cost[3] = {sqrt(ddot(r1, r1)), sqrt(ddot(r2, r2)), sqrt(ddot(r3, r3))};
  float w[3];
  const int best = pick_min<3>(cost, w, c.inv_tau_min, c.hard_ops);
  const double3 cons = on1 * (double)w[0] + on2 * (double)w[1] + on3 * (double)w[2];
  const double3 n_raw = d3(d10.y * d20.z - d10.z * d20.y, d10.z * d20.x - d10.x * d20.z,
                           d10.x * d20.y - d10.y * d20.x);
  const double n_norm = sqrt(ddot(n_raw, n_raw) + guard);
  const double3 n = n_raw * (1.0 / n_norm);
  const double3 dvp0 = dv0 - n * ddot(dv0, n);
  const double3 plane = t0 + dvp0;
  auto cross = [](double3 a, double3 b) {
    return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
  };
  const double bv = ddot(cross(d10, dvp0), n) / n_norm;
  const double bu = ddot(cross(dvp0, d20), n) / n_norm;
  const double bw = 1.0 - bu - bv;
  const float inside = within01(bu, c.inv_tau_comp, c.hard_ops) *
                       within01(bv, c.inv_tau_comp, c.hard_ops) *
                       within01(bw, c.inv_tau_comp, c.hard_ops);
  if (label) *label = best | ((inside >= 0.5f) << 2);
  const double in = (double)inside;
  return plane * in + cons * (1.0 - in);
}

}  // namespace cmgb
