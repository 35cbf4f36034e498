// Batched demo integrator: DemoSim::step (src/demosim.cpp:81-138) for every env
// of a batch, on the manifolds the scene batch leaves in device memory.
//
//   penalty_kernel   16 lanes per (env, pair): penalty_forces (demosim.cpp:31-66)
//                    over the pair's fixed-layout contacts, fixed-order warp
//                    reduction -> the pair's two wrenches + deepest penetration
//   integrate_kernel one thread per env: per body, wrench sum in pair order, then
//                    semi-implicit Euler on SE(3) (108-133) + finite check
//
// FP64 throughout (the contacts arrive as the ABI's FP32 outputs).
#include <cuda_runtime.h>

#include "launch_util.cuh"

#include "../common.h"
#include "../device/dmath.cuh"
#include "../device/pose.cuh"

namespace cmgb {

namespace {

__device__ __forceinline__ void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

// softplus_s (smooth_ops.hpp:66-81), both arms as in the reference; below
// e^-40 log1p(e) = e to double precision, above it log(1 + e) by log_d (the
// absolute error of forming 1 + e, ~1e-16, is what matters: it is scaled by tau).
__device__ __forceinline__ double softplus_ref(double x, double tau) {
  const double scaled = x / tau;
  const double e = exp_d(-fabs(scaled));
  const double l = e < 4e-18 ? e : log_d(1.0 + e);
  return scaled > 0.0 ? x + tau * l : tau * l;
}

// A 16-lane group per env (two envs per warp). The group first reads every
// contact's activity and deepest-penetration term and lists the active rows
// (activity >= 1e-12; the reference skips the others, demosim.cpp:40-41) in
// row order in shared memory, then deals them to its lanes: inactive rows
// leave no lane idle.
constexpr int kPenaltyLanes = 16;
constexpr int kPenaltyThreads = 256;
constexpr int kPenaltyMaxC = 256;  // rows per pair the list holds (more: every row is visited)

__global__ void __launch_bounds__(kPenaltyThreads, 3) penalty_kernel(const __grid_constant__ PenaltyArgs a) {
  __shared__ uint16_t act_list[kPenaltyThreads / kPenaltyLanes][kPenaltyMaxC];
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kPenaltyLanes;
  const int lane = threadIdx.x & (kPenaltyLanes - 1);
  const int grp = threadIdx.x / kPenaltyLanes;
  if (e >= a.n_env) return;  // a whole 16-lane group exits; the shuffles below use the group's mask
  const unsigned gm = 0xFFFFu << (threadIdx.x & 16);
  const DemoParamsDev& P = a.prm;
  // transforms[i].t is the COM (demosim.cpp:84, 96-97)
  const double* f1 = a.frames1 + 12 * e;
  const double* f2 = a.frames2 + 12 * e;
  const double com1[3] = {f1[9], f1[10], f1[11]};
  const double com2[3] = {f2[9], f2[10], f2[11]};
  const double* vel1 = a.vel + (e * a.nb + a.bi) * 6;
  const double* vel2 = a.vel + (e * a.nb + a.bj) * 6;
  const float* rows = a.contacts + e * a.C * 8;
  const bool listed = a.C <= kPenaltyMaxC;
  double deep = 0.0;
  int n_act = 0;
  // pass 1: activity of every row; the first kPre blocks of 16 rows are loaded
  // before any is used (independent loads in flight: the kernel is latency-bound)
  constexpr int kPre = 4;
  float pa[kPre], pd[kPre];
#pragma unroll
  for (int b = 0; b < kPre; ++b) {
    const int r = b * kPenaltyLanes + lane;
    pa[b] = r < a.C ? rows[r * 8 + 7] : 0.0f;
    pd[b] = r < a.C ? rows[r * 8 + 3] : 0.0f;
  }
  auto take = [&](int r, double act, double dist) {
    const bool on = r < a.C && act >= 1e-12;
    if (r < a.C && act > 0.5) deep = fmin(deep, dist);
    const unsigned bits = __ballot_sync(gm, on) >> (threadIdx.x & 16);
    if (listed && on) act_list[grp][n_act + __popc(bits & ((1u << lane) - 1u))] = (uint16_t)r;
    n_act += __popc(bits);
  };
#pragma unroll
  for (int b = 0; b < kPre; ++b)
    if (b * kPenaltyLanes < a.C) take(b * kPenaltyLanes + lane, pa[b], pd[b]);
  for (int r0 = kPre * kPenaltyLanes; r0 < a.C; r0 += kPenaltyLanes) {
    const int r = r0 + lane;
    take(r, r < a.C ? rows[r * 8 + 7] : 0.0f, r < a.C ? rows[r * 8 + 3] : 0.0f);
  }
  __syncwarp(gm);
  double acc[12];  // force1, torque1, force2, torque2
#pragma unroll
  for (int k = 0; k < 12; ++k) acc[k] = 0.0;
  const int n_rows = listed ? n_act : a.C;
  for (int k = lane; k < n_rows; k += kPenaltyLanes) {  // pass 2: the active rows
    const int r = listed ? (int)act_list[grp][k] : k;
    const float4* cp = reinterpret_cast<const float4*>(rows + r * 8);
    const float4 c0 = cp[0], c1 = cp[1];
    const double act = c1.w, dist = c0.w;
    if (act < 1e-12) continue;  // (unlisted path only)
    const double pt[3] = {c0.x, c0.y, c0.z};
    const double pressure = P.stiffness * softplus_ref(-dist, P.tau_force);
    const double nraw[3] = {c1.x, c1.y, c1.z};
    const double sc = rsqrt_d(1e-12 + (nraw[0] * nraw[0] + nraw[1] * nraw[1] + nraw[2] * nraw[2]));
    const double nh[3] = {nraw[0] * sc, nraw[1] * sc, nraw[2] * sc};
    // side of contact r in the fixed layout (manifold.hpp:14-17)
    const bool side1 = r < a.n1 ? true : (r < a.n1 + a.n2 ? false : (((r - a.n1 - a.n2) & 1) == 0));
    const double* vo = side1 ? vel1 : vel2;
    const double* vt = side1 ? vel2 : vel1;
    const double* co = side1 ? com1 : com2;
    const double* ct = side1 ? com2 : com1;
    double ro[3] = {pt[0] - co[0], pt[1] - co[1], pt[2] - co[2]};
    double rt[3] = {pt[0] - ct[0], pt[1] - ct[1], pt[2] - ct[2]};
    double wo[3], wt[3];
    const double Wo[3] = {vo[3], vo[4], vo[5]}, Wt[3] = {vt[3], vt[4], vt[5]};
    cross3(Wo, ro, wo);
    cross3(Wt, rt, wt);
    const double vrel[3] = {vo[0] + wo[0] - (vt[0] + wt[0]), vo[1] + wo[1] - (vt[1] + wt[1]),
                            vo[2] + wo[2] - (vt[2] + wt[2])};
    const double vn = vrel[0] * nh[0] + vrel[1] * nh[1] + vrel[2] * nh[2];
    const double fn = fmax(act * (pressure - P.damping * vn), 0.0);
    const double vtg[3] = {vrel[0] - nh[0] * vn, vrel[1] - nh[1] * vn, vrel[2] - nh[2] * vn};
    const double vtn = sqrt(vtg[0] * vtg[0] + vtg[1] * vtg[1] + vtg[2] * vtg[2]);
    const double ft = fmin(P.friction * fn, P.friction_viscous * vtn);
    const double q = ft * rcp_d(vtn + 1e-12);  // (vtg / den) ft with one reciprocal
    const double F[3] = {nh[0] * fn - vtg[0] * q, nh[1] * fn - vtg[1] * q, nh[2] * fn - vtg[2] * q};
    double to[3], tt[3];
    cross3(ro, F, to);
    cross3(rt, F, tt);
    // the own body gains (F, r_o x F), the other loses (F, r_t x F); selects,
    // not a pointer into acc (which would put it in local memory)
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) {
      const double sf = side1 ? F[k2] : -F[k2];
      acc[k2] += sf;
      acc[3 + k2] += side1 ? to[k2] : -tt[k2];
      acc[6 + k2] -= sf;
      acc[9 + k2] += side1 ? -tt[k2] : to[k2];
    }
  }
  // fixed-order butterfly reduction within the env's 16 lanes (deterministic)
#pragma unroll
  for (int o = kPenaltyLanes / 2; o > 0; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 12; ++k) acc[k] += __shfl_xor_sync(gm, acc[k], o);
    deep = fmin(deep, __shfl_xor_sync(gm, deep, o));
  }
  if (lane == 0) {
    double* w = a.wrench + e * 12;
#pragma unroll
    for (int k = 0; k < 12; ++k) w[k] = acc[k];
    a.deepest[e] = deep;
  }
}

__global__ void __launch_bounds__(128) integrate_kernel(const __grid_constant__ IntegrateArgs a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.n_env) return;
  double d = 0.0;  // deepest_penetration over the env's pairs (demosim.cpp:86, 94-95)
  for (int q = 0; q < a.n_pairs; ++q) d = fmin(d, a.pair_deepest[(int64_t)q * a.n_env + e]);
  if (a.deepest) a.deepest[e] = d;
  bool fin = true;
  for (int b = 0; b < a.nb; ++b) {
    if (a.is_static[b]) continue;
    // wrench: pair contributions in pair order (demosim.cpp:96-103)
    double F[3] = {0, 0, 0}, T[3] = {0, 0, 0};
    for (int q = 0; q < a.n_pairs; ++q) {
      const int side = a.pair_i[q] == b ? 0 : (a.pair_j[q] == b ? 1 : -1);
      if (side < 0) continue;
      const double* w = a.wrench + ((int64_t)q * a.n_env + e) * 12 + 6 * side;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        F[k] += w[k];
        T[k] += w[3 + k];
      }
    }
    double* pose = a.poses + (e * a.nb + b) * 6;
    double* v = a.vel + (e * a.nb + b) * 6;
    double xi[6], R[9], t[3];
#pragma unroll
    for (int k = 0; k < 6; ++k) xi[k] = pose[k];
    se3_exp_d(xi, R, t);
    const double m = a.mass[b];
    const double dt = a.dt;
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] += dt * (F[k] / m + a.gravity[k]);
    // I_world = R diag(I) R^T, no gyroscopic term (demosim.cpp:116-126)
    const double tb[3] = {R[0] * T[0] + R[3] * T[1] + R[6] * T[2], R[1] * T[0] + R[4] * T[1] + R[7] * T[2],
                          R[2] * T[0] + R[5] * T[1] + R[8] * T[2]};
    const double wb[3] = {tb[0] / a.inertia[3 * b], tb[1] / a.inertia[3 * b + 1], tb[2] / a.inertia[3 * b + 2]};
    const double wd[3] = {R[0] * wb[0] + R[1] * wb[1] + R[2] * wb[2], R[3] * wb[0] + R[4] * wb[1] + R[5] * wb[2],
                          R[6] * wb[0] + R[7] * wb[1] + R[8] * wb[2]};
#pragma unroll
    for (int k = 0; k < 3; ++k) v[3 + k] += dt * wd[k];
    const double tn[3] = {t[0] + v[0] * dt, t[1] + v[1] * dt, t[2] + v[2] * dt};
    const double wdt[3] = {v[3] * dt, v[4] * dt, v[5] * dt};
    double dR[9], Rn[9];
    so3_exp_dev(wdt, dR);
    matmul3(dR, R, Rn);
    se3_log_dev(Rn, tn, pose);
    fin = fin && isfinite(tn[0]) && isfinite(tn[1]) && isfinite(tn[2]) && isfinite(v[3]) && isfinite(v[4]) &&
          isfinite(v[5]) && isfinite(v[0]);
  }
  if (a.ok) a.ok[e] = fin ? 1 : 0;
}

}  // namespace

int launch_penalty(const PenaltyArgs& a, void* stream) {
  if (a.n_env <= 0) return 0;
  const int64_t threads = a.n_env * kPenaltyLanes;
  note_launch();
  penalty_kernel<<<(unsigned)((threads + kPenaltyThreads - 1) / kPenaltyThreads), kPenaltyThreads, 0,
                   static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_integrate(const IntegrateArgs& a, void* stream) {
  const int64_t n = a.n_env;
  if (n <= 0) return 0;
  note_launch();
  integrate_kernel<<<(unsigned)((n + 127) / 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace cmgb
