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

// softplus_s (smooth_ops.hpp:66-81), both arms as in the reference; the
// exponential is exp_d and below e^-40 log1p(e) = e to double precision.
__device__ __forceinline__ double softplus_ref(double x, double tau) {
  const double scaled = x / tau;
  const double e = exp_d(-fabs(scaled));
  const double l = e < 4e-18 ? e : log1p(e);
  return scaled > 0.0 ? x + tau * l : tau * l;
}

// A 16-lane group per env (two envs per warp): 48-contact pair manifolds are
// 3 contacts per lane with no idle second pass.
constexpr int kPenaltyLanes = 16;

__global__ void __launch_bounds__(256) penalty_kernel(const __grid_constant__ PenaltyArgs a) {
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kPenaltyLanes;
  const int lane = threadIdx.x & (kPenaltyLanes - 1);
  if (e >= a.n_env) return;  // a whole 16-lane group exits; the shuffles below use the group's mask
  const DemoParamsDev& P = a.prm;
  // transforms[i].t is the COM (demosim.cpp:84, 96-97)
  const double* f1 = a.frames1 + 12 * e;
  const double* f2 = a.frames2 + 12 * e;
  const double com1[3] = {f1[9], f1[10], f1[11]};
  const double com2[3] = {f2[9], f2[10], f2[11]};
  const double* vel1 = a.vel + (e * a.nb + a.bi) * 6;
  const double* vel2 = a.vel + (e * a.nb + a.bj) * 6;
  double acc[12];  // force1, torque1, force2, torque2
#pragma unroll
  for (int k = 0; k < 12; ++k) acc[k] = 0.0;
  double deep = 0.0;
  for (int r = lane; r < a.C; r += kPenaltyLanes) {
    const float4* cp = reinterpret_cast<const float4*>(a.contacts + (e * a.C + r) * 8);
    const float4 c0 = cp[0], c1 = cp[1];
    const double act = c1.w, dist = c0.w;
    if (act > 0.5) deep = fmin(deep, dist);
    if (act < 1e-12) continue;
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
    const double den = vtn + 1e-12;
    const double F[3] = {nh[0] * fn - vtg[0] / den * ft, nh[1] * fn - vtg[1] / den * ft,
                         nh[2] * fn - vtg[2] / den * ft};
    double to[3], tt[3];
    cross3(ro, F, to);
    cross3(rt, F, tt);
    double* own = acc + (side1 ? 0 : 6);
    double* oth = acc + (side1 ? 6 : 0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      own[k] += F[k];
      own[3 + k] += to[k];
      oth[k] -= F[k];
      oth[3 + k] -= tt[k];
    }
  }
  // fixed-order butterfly reduction within the env's 16 lanes (deterministic)
  const unsigned gm = 0xFFFFu << (threadIdx.x & 16);
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
  penalty_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(a);
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
