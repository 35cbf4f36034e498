// Forward-mode derivative-carrying scalar for the pose-Jacobian (JVP) path.
//
// The reference templates every kernel on its scalar and runs it with
// Dual<12> seeded at the two 6-D pose vectors (dual.hpp:47-130, 249-263). On
// the device the JVP kernel (manifold_jvp.cuh) instead seeds Dual<N> at the
// low-dimensional bottlenecks of the pipeline -- Dual<3> at a body point,
// Dual<5> at the witness QP's (Q, c), Dual<1> per pose coordinate in se3_exp
// -- and chains the 12 pose directions through the resulting Jacobians. Semantics follow
// dual.hpp: comparisons / branches read the primal only (callers use pv()),
// fabs has subgradient 0 at the kink (dual.hpp:236-246).
//
// Elementary functions evaluate the primal with the same FP64 device routines
// as the value path (exp_d, log_d, rcp_d, rsqrt_d; dmath.cuh) and apply the
// analytic chain rule to the tangents, so the primal of a Dual run is
// bit-identical to the double run.
//
// Vectors: vec3<double> is CUDA's double3 (the value kernels keep their exact
// code); vec3<Dual<N>> is V3<Dual<N>>. Templated device code builds vectors
// with mk3<T>() and reads primals with pv().
#pragma once

#include <type_traits>

#include "dmath.cuh"

namespace cmgb {

template <int N>
struct Dual {
  double v;
  double d[N];

  __device__ __forceinline__ Dual() {}
  __device__ __forceinline__ Dual(double x) : v(x) {  // NOLINT: implicit promotion intended
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = 0.0;
  }
  static __device__ __forceinline__ Dual make(double v, const double (&t)[N]) {
    Dual r;
    r.v = v;
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = t[i];
    return r;
  }
  // v + s * (tangents of x): the chain rule of every unary function below.
  static __device__ __forceinline__ Dual chain(double v, double s, const Dual& x) {
    Dual r;
    r.v = v;
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = s * x.d[i];
    return r;
  }

  friend __device__ __forceinline__ Dual operator+(const Dual& a, const Dual& b) {
    Dual r;
    r.v = a.v + b.v;
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = a.d[i] + b.d[i];
    return r;
  }
  friend __device__ __forceinline__ Dual operator-(const Dual& a, const Dual& b) {
    Dual r;
    r.v = a.v - b.v;
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = a.d[i] - b.d[i];
    return r;
  }
  friend __device__ __forceinline__ Dual operator-(const Dual& a) {
    Dual r;
    r.v = -a.v;
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = -a.d[i];
    return r;
  }
  friend __device__ __forceinline__ Dual operator*(const Dual& a, const Dual& b) {
    Dual r;
    r.v = a.v * b.v;
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = fma(a.v, b.d[i], a.d[i] * b.v);
    return r;
  }
  // a / b via the FP64 reciprocal of the value path (div_d)
  friend __device__ __forceinline__ Dual operator/(const Dual& a, const Dual& b) {
    const double inv = rcp_d(b.v);
    Dual r;
    r.v = a.v * inv;
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = (a.d[i] - r.v * b.d[i]) * inv;
    return r;
  }
  __device__ __forceinline__ Dual& operator+=(const Dual& o) { return *this = *this + o; }
  __device__ __forceinline__ Dual& operator-=(const Dual& o) { return *this = *this - o; }
  __device__ __forceinline__ Dual& operator*=(const Dual& o) { return *this = *this * o; }

  // fused a * b + c: the primal is one FP64 fma, as in the value path
  friend __device__ __forceinline__ Dual fma(const Dual& a, const Dual& b, const Dual& c) {
    Dual r;
    r.v = fma(a.v, b.v, c.v);
#pragma unroll
    for (int i = 0; i < N; ++i) r.d[i] = fma(a.v, b.d[i], fma(a.d[i], b.v, c.d[i]));
    return r;
  }
  friend __device__ __forceinline__ Dual exp_d(const Dual& x) {
    const double e = exp_d(x.v);
    return chain(e, e, x);
  }
  // exp / log of the LSE and top-K weights: the lean FP64 routines (<= 1 ulp
  // from libdevice's; dmath.cuh)
  friend __device__ __forceinline__ Dual exp(const Dual& x) {
    const double e = exp_d(x.v);
    return chain(e, e, x);
  }
  friend __device__ __forceinline__ Dual log_d(const Dual& x) { return chain(log_d(x.v), rcp_d(x.v), x); }
  friend __device__ __forceinline__ Dual log(const Dual& x) { return chain(log_d(x.v), rcp_d(x.v), x); }
  friend __device__ __forceinline__ Dual log1p(const Dual& x) {
    return chain(::log1p(x.v), rcp_d(1.0 + x.v), x);
  }
  friend __device__ __forceinline__ Dual expm1(const Dual& x) {
    const double e = ::expm1(x.v);
    return chain(e, 1.0 + e, x);
  }
  friend __device__ __forceinline__ Dual rcp_d(const Dual& x) {
    const double r = rcp_d(x.v);
    return chain(r, -r * r, x);
  }
  friend __device__ __forceinline__ Dual div_d(const Dual& a, const Dual& b) { return a / b; }
  friend __device__ __forceinline__ Dual rsqrt_d(const Dual& x) {
    const double r = rsqrt_d(x.v);
    return chain(r, -0.5 * r * r * r, x);
  }
  friend __device__ __forceinline__ Dual sqrt(const Dual& x) {
    const double s = ::sqrt(x.v);
    return chain(s, 0.5 * rcp_d(s), x);
  }
  friend __device__ __forceinline__ Dual tanh(const Dual& x) {
    const double t = ::tanh(x.v);
    return chain(t, 1.0 - t * t, x);
  }
  // pow with a constant exponent (dual.hpp:224-234)
  friend __device__ __forceinline__ Dual pow(const Dual& x, double p) {
    // x > 0 on every use (squared coordinates + floor): exp_d(p log_d x), and
    // the derivative p x^(p-1) = p y / x from the same value (sdf.cuh pow_rt)
    const double y = exp_d(p * log_d(x.v));
    return chain(y, p * y * rcp_d(x.v), x);
  }
  // |x| with subgradient 0 at the kink (dual.hpp:236-246)
  friend __device__ __forceinline__ Dual fabs(const Dual& x) {
    const double s = x.v < 0.0 ? -1.0 : (x.v > 0.0 ? 1.0 : 0.0);
    return chain(::fabs(x.v), s, x);
  }
  // max / min select a whole operand by primal (std::max semantics)
  friend __device__ __forceinline__ Dual fmax(const Dual& a, const Dual& b) { return a.v < b.v ? b : a; }
  friend __device__ __forceinline__ Dual fmin(const Dual& a, const Dual& b) { return b.v < a.v ? b : a; }
  friend __device__ __forceinline__ void sincos(const Dual& x, Dual* s, Dual* c) {
    double sv, cv;
    ::sincos(x.v, &sv, &cv);
    *s = chain(sv, cv, x);
    *c = chain(cv, -sv, x);
  }
};

template <class T>
struct is_dual : std::false_type {};
template <int N>
struct is_dual<Dual<N>> : std::true_type {};

template <int N>
__device__ __forceinline__ double pv(const Dual<N>& x) { return x.v; }

// ---- 3-vectors over T ---------------------------------------------------------
template <class T>
struct V3 {
  T x, y, z;
};
template <class T>
struct Vec3Of {
  using type = V3<T>;
};
template <>
struct Vec3Of<double> {
  using type = double3;
};
template <class T>
using vec3 = typename Vec3Of<T>::type;

template <class T>
__device__ __forceinline__ vec3<T> mk3(const T& x, const T& y, const T& z) {
  if constexpr (std::is_same_v<T, double>) return make_double3(x, y, z);
  else return V3<T>{x, y, z};
}

template <class T>
__device__ __forceinline__ V3<T> operator+(const V3<T>& a, const V3<T>& b) {
  return V3<T>{a.x + b.x, a.y + b.y, a.z + b.z};
}
template <class T>
__device__ __forceinline__ V3<T> operator-(const V3<T>& a, const V3<T>& b) {
  return V3<T>{a.x - b.x, a.y - b.y, a.z - b.z};
}
template <class T, class S>
__device__ __forceinline__ V3<T> operator*(const V3<T>& a, const S& s) {
  return V3<T>{a.x * s, a.y * s, a.z * s};
}
template <class T>
__device__ __forceinline__ T ddot(const V3<T>& a, const V3<T>& b) {
  return a.x * b.x + a.y * b.y + a.z * b.z;
}
template <class T, class S>
__device__ __forceinline__ V3<T> dscale(const V3<T>& a, const S& s) {
  return V3<T>{a.x * s, a.y * s, a.z * s};
}
// Row-major 3x3 (vec3.hpp:88-92 / 125-130); M is double (fixed leaf frames)
// or T (posed frames).
template <class M, class T>
__device__ __forceinline__ V3<T> mul_R(const M* R, const V3<T>& v) {
  return V3<T>{R[0] * v.x + R[1] * v.y + R[2] * v.z, R[3] * v.x + R[4] * v.y + R[5] * v.z,
               R[6] * v.x + R[7] * v.y + R[8] * v.z};
}
template <class M, class T>
__device__ __forceinline__ V3<T> mul_Rt(const M* R, const V3<T>& v) {
  return V3<T>{R[0] * v.x + R[3] * v.y + R[6] * v.z, R[1] * v.x + R[4] * v.y + R[7] * v.z,
               R[2] * v.x + R[5] * v.y + R[8] * v.z};
}

}  // namespace cmgb
