// Device scalar helpers for sm_100a.
//
// Precision policy: geometry that suffers cancellation (pose
// transforms, QP linear algebra, witness points, sphere-trace accumulation,
// the E-E separation vector) is FP64; SDF fields and the smooth operators'
// transcendentals are FP32 on the SFU (MUFU.EX2/LG2/RSQ/RCP).
#pragma once

#include <cuda_runtime.h>
#include <math.h>

namespace cmgb {

__device__ __forceinline__ float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2f(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcpf(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rsqf(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// x^p for a general real exponent via the SFU (x > 0).
__device__ __forceinline__ float powg(float x, float p) { return ex2f(p * lg2f(x)); }

// x^(n-1) for a small positive integer n (repeated squaring, no SFU);
// the branch is warp-uniform (one SDF per launch side).
__device__ __forceinline__ float powi_m1(float x, int n) {
  switch (n) {
    case 1: return 1.0f;
    case 2: return x;
    case 3: return x * x;
    case 4: { const float x2 = x * x; return x2 * x; }
    case 5: { const float x2 = x * x; return x2 * x2; }
    case 10: { const float x2 = x * x, x4 = x2 * x2, x8 = x4 * x4; return x8 * x; }
    case 20: { const float x2 = x * x, x4 = x2 * x2, x8 = x4 * x4, x16 = x8 * x8; return (x16 * x2) * x; }
    default: {
      float r = 1.0f, b = x;
      int e = n - 1;
#pragma unroll 1
      while (e) {
        if (e & 1) r *= b;
        b *= b;
        e >>= 1;
      }
      return r;
    }
  }
}

// (x^p, x^(p-1)): integer fast path when n > 0, else SFU pow.
__device__ __forceinline__ void pow_pair(float x, int n, float p, float& xp, float& xpm1) {
  if (n > 0) {
    xpm1 = powi_m1(x, n);
    xp = xpm1 * x;
  } else {
    xp = powg(x, p);
    xpm1 = xp * rcpf(x);
  }
}

// stable_sigmoid (smooth_ops.hpp:22-35): both arms evaluate the same function.
__device__ __forceinline__ float sigmoidf(float x) {
  const float e = __expf(-fabsf(x));
  const float inv = __frcp_rn(1.0f + e);
  return x >= 0.0f ? inv : e * inv;
}

// softplus correction tau*log1p(exp(-|x|/tau)) (smooth_ops.hpp:66-81 with the
// max(x,0) part taken exactly in FP64 by the caller).
__device__ __forceinline__ float softplus_corr(float ax_over_tau, float tau) {
  return tau * log1pf(__expf(-ax_over_tau));
}

// tanh (sign_s, smooth_ops.hpp:57-62): accurate libdevice form (2 ulp).
__device__ __forceinline__ float tanh_acc(float x) { return tanhf(x); }

__device__ __forceinline__ double3 d3(double x, double y, double z) { return make_double3(x, y, z); }
__device__ __forceinline__ double3 operator+(double3 a, double3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ double3 operator-(double3 a, double3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double3 operator*(double3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ double ddot(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

__device__ __forceinline__ float3 f3(float x, float y, float z) { return make_float3(x, y, z); }
__device__ __forceinline__ float fdot(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ float3 to_f3(double3 a) { return f3((float)a.x, (float)a.y, (float)a.z); }

// Row-major 3x3 (vec3.hpp:88-92 / 125-130).
__device__ __forceinline__ double3 mul_R(const double* R, double3 v) {
  return d3(R[0] * v.x + R[1] * v.y + R[2] * v.z, R[3] * v.x + R[4] * v.y + R[5] * v.z,
            R[6] * v.x + R[7] * v.y + R[8] * v.z);
}
__device__ __forceinline__ double3 mul_Rt(const double* R, double3 v) {
  return d3(R[0] * v.x + R[3] * v.y + R[6] * v.z, R[1] * v.x + R[4] * v.y + R[7] * v.z,
            R[2] * v.x + R[5] * v.y + R[8] * v.z);
}
__device__ __forceinline__ float3 mul_R_f(const double* R, float3 v) {
  return f3((float)R[0] * v.x + (float)R[1] * v.y + (float)R[2] * v.z,
            (float)R[3] * v.x + (float)R[4] * v.y + (float)R[5] * v.z,
            (float)R[6] * v.x + (float)R[7] * v.y + (float)R[8] * v.z);
}

// se3_exp (pose.hpp:37-91) in FP64; series branch below theta^2 = 1e-8.
__device__ __forceinline__ void se3_exp_d(const double* xi, double* R, double* t) {
  const double wx = xi[3], wy = xi[4], wz = xi[5];
  const double th2 = wx * wx + wy * wy + wz * wz;
  double a, b, c;
  if (th2 < 1e-8) {
    a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    c = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
  } else {
    const double th = sqrt(th2);
    double s, co;
    sincos(th, &s, &co);
    a = s / th;
    b = (1.0 - co) / th2;
    c = (1.0 - a) / th2;
  }
  const double W[9] = {0.0, -wz, wy, wz, 0.0, -wx, -wy, wx, 0.0};
  double W2[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      W2[3 * i + j] = W[3 * i] * W[j] + W[3 * i + 1] * W[3 + j] + W[3 * i + 2] * W[6 + j];
  double V[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double id = (i % 4 == 0) ? 1.0 : 0.0;
    R[i] = (id + W[i] * a) + W2[i] * b;
    V[i] = (id + W[i] * b) + W2[i] * c;
  }
  const double3 r = mul_R(V, d3(xi[0], xi[1], xi[2]));
  t[0] = r.x;
  t[1] = r.y;
  t[2] = r.z;
}

}  // namespace cmgb
