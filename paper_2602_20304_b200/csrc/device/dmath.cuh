// Device scalar helpers for sm_100a.
//
// Precision policy: every quantity that the reference's outputs
// are ill-conditioned in (pose transforms, SDF field cores and gradient
// directions, QP linear algebra, witness points, sphere-trace accumulation,
// the E-E separation vector) is FP64 on the B200's half-rate DFMA pipe; the
// bounded transcendental corrections (sigmoid / softplus / softmin weights,
// expm1 / log1p of small arguments) run in FP32 on the SFU (MUFU.EX2/LG2/RSQ/
// RCP).
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

// FP64 reciprocal / reciprocal square root for finite, normal, positive-range
// arguments: MUFU.RCP64H / RSQ64H seed (rcp/rsqrt.approx.ftz.f64; measured max
// relative error 2^-20.0 / 2^-20.1 on B200, tools/mufu_f64_precision.cu) + one
// Newton step -> <= 1.3e-12 relative (measured 9.7e-13 / 1.25e-12). Every use
// sits where 1e-12 relative is below the ~1e-10 absolute witness budget
// (DESIGN.md §4): QP reciprocals / quotients, log_d's atanh argument,
// indicator normalisations, the trace's normalisations (whose scale error only
// moves points along the normal, which later iterations remove). An FP32 seed
// would overflow for |grad f|^2 > 3.4e38.
__device__ __forceinline__ double rcp_d(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return fma(y, fma(-x, y, 1.0), y);
}
__device__ __forceinline__ double rsqrt_d(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y * fma(-0.5 * x, y * y, 1.5);
}
__device__ __forceinline__ double div_d(double a, double b) { return a * rcp_d(b); }

// exp(x) in FP64 for x <= ~709: x = k ln2 + r, |r| <= ln2/2 (Cody-Waite split
// of ln2), e^r by a degree-8 near-minimax polynomial (Chebyshev interpolation,
// tools/minimax_coeffs.py: max relative error 1.1e-12), 2^k spliced into the
// exponent field. exp(x < -708) returns 0 (the true value is < 2.3e-308).
// ~13 FP64 instructions, no branches beyond the underflow select. 1e-12 is
// the precision every use needs: the exponentials are soft
// indicator / weight / log-sum-exp terms whose relative error moves witness
// points and fields by <= ~tau x 1e-12 (the witness budget is ~1e-10 absolute);
// the libdevice version carries 1-ulp accuracy and full special-case handling
// the arguments never need.
// FP64 literals live in the constant bank so DFMA/DMUL read them as c[][]
// operands (an immediate double costs two UMOVs + a uniform-pipe dependency).
struct MathConsts {
  double exp_c[9];  // degree 8 .. 0 (Horner order)
  double log_c[6];  // atanh(s)/s = Q(s^2), degree 5 .. 0 in s^2
  double log2e, ln2_hi, ln2_lo, ln2, sqrt2, floor30, floor20;
};
static __constant__ MathConsts kMC = {
    {2.4876164022625967e-05, 0.00019915866926782682, 0.0013888821677630362, 0.008333266097949614,
     0.041666666890957, 0.16666666891045775, 0.49999999999797934, 0.9999999999797852, 1.0},
    {0.09804047819876527, 0.11087124955038745, 0.14286083072937864, 0.1999999744591619,
     0.3333333333978963, 0.9999999999999736},
    1.4426950408889634, 6.93147180369123816490e-01, 1.90821492927058770002e-10,
    6.93147180559945309417e-01, 1.4142135623730951, 1e-30, 1e-20};

__device__ __forceinline__ double exp_d(double x) {
  // k = rint(x log2e) by the 1.5 * 2^52 shifter: the sum's low word is k as an
  // integer (no FRND / F2I round trip), the difference k as a double
  const double t = fma(x, kMC.log2e, 6755399441055744.0);
  const double k = t - 6755399441055744.0;
  double r = fma(-k, kMC.ln2_hi, x);
  r = fma(-k, kMC.ln2_lo, r);
  double p = kMC.exp_c[0];
#pragma unroll
  for (int i = 1; i < 9; ++i) p = fma(p, r, kMC.exp_c[i]);
  const int ki = __double2loint(t);
  const double s = __hiloint2double(__double2hiint(p) + (ki << 20), __double2loint(p));
  return x < -708.0 ? 0.0 : s;
}

// log(v) in FP64 for finite v > 0: v = 2^e m, m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh(s) = 2 s Q(s^2), s = (m - 1)/(m + 1), |s| <= 0.1716, Q a
// degree-5 near-minimax polynomial in s^2 (max relative error 2.7e-14).
__device__ __forceinline__ double log_d(double v) {
  int hi = __double2hiint(v);
  int e = ((hi >> 20) & 0x7ff) - 1023;
  hi = (hi & 0x000fffff) | 0x3ff00000;  // m in [1, 2)
  double m = __hiloint2double(hi, __double2loint(v));
  if (m > kMC.sqrt2) {
    m *= 0.5;
    e += 1;
  }
  const double s = (m - 1.0) * rcp_d(m + 1.0);
  const double s2 = s * s;
  double p = kMC.log_c[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) p = fma(p, s2, kMC.log_c[i]);
  return fma((double)e, kMC.ln2, 2.0 * s * p);
}

// Primal of a scalar (the Dual<N> overload lives in dual.cuh): branches of the
// templated routines read it, like the reference's HardBranchScope reads.
__device__ __forceinline__ double pv(double x) { return x; }
__device__ __forceinline__ double pv(float x) { return x; }

// FP32 members of the overload sets (the K6 witness batches' soft indicators,
// witness.cuh): SFU forms. Their arguments are FP64 values rounded to FP32,
// which already costs |x| 6e-8 relative in exp; ex2/lg2/rcp.approx stay within
// that budget (alpha error <= tau_clip * 1e-6 on the witness points).
// (ftz forms without the denormal range fix-ups of __expf / __logf: the
// arguments are <= 0 -- a result below 2^-126 is a weight that does not count
// -- or quotients in (1/2, 2))
__device__ __forceinline__ float exp_d(float x) { return ex2f(x * 1.44269504088896341f); }
__device__ __forceinline__ float log_d(float x) { return lg2f(x) * 0.693147180559945309f; }
__device__ __forceinline__ float rcp_d(float x) { return rcpf(x); }

// stable_sigmoid (smooth_ops.hpp:22-35), FP64: both arms evaluate the same
// function; returns sigma(x) and its complement 1 - sigma(x) = sigma(-x), each
// to full relative precision (the blends need the small one exactly).
template <class T>
__device__ __forceinline__ void sigmoid_pair_d(const T& x, T* s, T* c) {
  const T e = exp_d(-fabs(x));
  const T inv = rcp_d(1.0 + e);
  const T small = e * inv;
  *s = pv(x) >= 0.0 ? inv : small;
  *c = pv(x) >= 0.0 ? small : inv;
}
template <class T>
__device__ __forceinline__ T sigmoid_d(const T& x) {
  T s, c;
  sigmoid_pair_d(x, &s, &c);
  return s;
}

// softplus_s (smooth_ops.hpp:66-81): max(x, 0) + tau log1p(exp(-|x|/tau)); both
// reference arms are this function.
__device__ __forceinline__ double softplus_d(double x, double tau, double inv_tau) {
  return fmax(x, 0.0) + tau * log_d(1.0 + exp_d(-fabs(x) * inv_tau));
}

__device__ __forceinline__ double3 d3(double x, double y, double z) { return make_double3(x, y, z); }
__device__ __forceinline__ double3 operator+(double3 a, double3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ double3 operator-(double3 a, double3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double3 operator*(double3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ double ddot(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double3 dscale(double3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ float3 to_f3v(double3 a) { return make_float3((float)a.x, (float)a.y, (float)a.z); }

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
// T = double (frames kernel) or Dual<N> (pose tangents, manifold_jvp.cu).
template <class T>
__device__ __forceinline__ void se3_exp_d(const T* xi, T* R, T* t) {
  const T wx = xi[3], wy = xi[4], wz = xi[5];
  const T th2 = wx * wx + wy * wy + wz * wz;
  T a, b, c;
  if (pv(th2) < 1e-8) {
    a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    c = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
  } else {
    const T th = sqrt(th2);
    T s, co;
    sincos(th, &s, &co);
    a = s / th;
    b = (1.0 - co) / th2;
    c = (1.0 - a) / th2;
  }
  const T W[9] = {0.0, -wz, wy, wz, 0.0, -wx, -wy, wx, 0.0};
  T W2[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      W2[3 * i + j] = W[3 * i] * W[j] + W[3 * i + 1] * W[3 + j] + W[3 * i + 2] * W[6 + j];
  T V[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const double id = (i % 4 == 0) ? 1.0 : 0.0;
    R[i] = (id + W[i] * a) + W2[i] * b;
    V[i] = (id + W[i] * b) + W2[i] * c;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) t[i] = V[3 * i] * xi[0] + V[3 * i + 1] * xi[1] + V[3 * i + 2] * xi[2];
}

}  // namespace cmgb
