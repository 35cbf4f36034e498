// Device evaluation of the smooth analytical SDF programs.
//
// Query flavours, as in the reference (sdf.hpp:177-195):
//   kValue         phi                         (scores, pen sigmoids)
//   kGrad          phi + true grad phi         (sphere tracing, sdf.hpp:318-326)
//   kNormalSource  phi + composed normal field (SQ leaves give grad f, 233-288)
//   kNormalOnly    normal field only (lone SQ leaf: phi skipped)
// Gradients are analytic (the reference nests a Dual<3>: the derivative of the
// same expression graph).
//
// Precision: phi feeds the fixed-count sphere trace, whose
// tangential drift is phi * (direction error), and the E-E signed normal
// amplifies witness errors by (1/|de|)(1 + 1/tau_sign); matching the FP64
// reference to 1e-5 needs ~1e-10 absolute. The field is therefore FP64
// throughout (integer-power chains instead of pow for the superquadric,
// 1 - f^p4 = -expm1(p4 log1p(f - 1)) without cancellation, FP64 plane / RBF
// distances, LSE / RBF weights). FP64 reciprocal square roots are SFU seeds
// refined by one Newton step.
#pragma once

#include "../common.h"
#include "dmath.cuh"
#include "dual.cuh"

namespace cmgb {

// Every routine is templated on the scalar T: double for the value kernels,
// Dual<N> for the pose-Jacobian kernel (dual.cuh). T = double compiles to the
// same code as a plain double implementation.
template <class T>
struct SdfOutT {
  T v;
  vec3<T> g;
};
using SdfOut = SdfOutT<double>;

// max(m, x) for the log-sum-exp shifts: one compare + selects for double
// (fmax's NaN handling costs five instructions; the same value for every
// non-NaN x); Dual keeps its fmax (the tangent of the larger arm).
template <class T>
__device__ __forceinline__ T max_sel(const T& m, const T& x) {
  if constexpr (std::is_same_v<T, double>) return x > m ? x : m;
  else return fmax(m, x);
}

// x^n for a small positive integer n (warp-uniform), FP64 products.
template <class T>
__device__ __forceinline__ T ipow_d(const T& x, int n) {
  switch (n) {
    case 1: return x;
    case 2: return x * x;
    case 4: { const T x2 = x * x; return x2 * x2; }
    case 5: { const T x2 = x * x; return x2 * x2 * x; }
    case 9: { const T x2 = x * x, x4 = x2 * x2; return x4 * x4 * x; }
    case 10: { const T x2 = x * x, x4 = x2 * x2; return x4 * x4 * x2; }
    case 19: { const T x2 = x * x, x4 = x2 * x2, x8 = x4 * x4, x16 = x8 * x8; return x16 * x2 * x; }
    case 20: { const T x2 = x * x, x4 = x2 * x2, x8 = x4 * x4, x16 = x8 * x8; return x16 * x4; }
    default: {
      T r = 1.0, b = x;
#pragma unroll 1
      for (int e = n; e; e >>= 1) {
        if (e & 1) r *= b;
        b *= b;
      }
      return r;
    }
  }
}

// Compile-time integer power (N > 0) for specialised superquadric kinds.
template <int N, class T>
__device__ __forceinline__ T cpow(const T& x) {
  if constexpr (N == 1) return x;
  else if constexpr (N % 2 == 0) { const T h = cpow<N / 2>(x); return h * h; }
  else return cpow<N - 1>(x) * x;
}

// (x^p, x^(p-1)) in FP64: integer chains (no SFU) or libdevice pow.
// Runtime-exponent x^p for x > 0 (the squared-coordinate floor keeps it so):
// exp_d(p log_d(x)), relative error ~|p log x| 3e-14 + 1e-12 -- the same
// budget as the integer-exponent chains' Newton step, at a fifth of
// libdevice pow's cost; Dual arguments keep their overload.
template <class T>
__device__ __forceinline__ T pow_rt(const T& x, double p) {
  if constexpr (std::is_same_v<T, double>) return exp_d(p * log_d(x));
  else return pow(x, p);
}

template <class T>
__device__ __forceinline__ void pow_pair_d(const T& x, int n, double p, T& xp, T& xpm1) {
  if (n > 0) {
    xpm1 = n == 1 ? T(1.0) : ipow_d(x, n - 1);
    xp = xpm1 * x;
  } else {
    xp = pow_rt(x, p);
    xpm1 = div_d(xp, x);
  }
}

// (x^p, x^(p-1)): compile-time exponent N > 0, or runtime (N == 0).
template <int N, class T>
__device__ __forceinline__ void pow_pair_t(const T& x, int n, double p, T& xp, T& xpm1) {
  if constexpr (N == 0) {
    pow_pair_d(x, n, p, xp, xpm1);
  } else if constexpr (N == 1) {
    xpm1 = 1.0;
    xp = x;
  } else {
    xpm1 = cpow<N - 1>(x);
    xp = xpm1 * x;
  }
}

// Dual overload for compile-time exponents N >= 2: the primal chain is the
// double one (bit-identical to the Dual products), the tangents take the
// analytic derivatives N x^(N-1), (N-1) x^(N-2) -- 2 scalings instead of
// carrying the tangents through every product of the chain.
template <int N, int ND, std::enable_if_t<(N >= 2), int> = 0>
__device__ __forceinline__ void pow_pair_t(const Dual<ND>& x, int, double, Dual<ND>& xp, Dual<ND>& xpm1) {
  const double a = cpow<N - 1>(x.v);
  const double b = N >= 3 ? cpow<(N >= 3 ? N - 2 : 1)>(x.v) : 1.0;
  xpm1 = Dual<ND>::chain(a, (double)(N - 1) * b, x);
  xp = Dual<ND>::chain(a * x.v, (double)N * a, x);
}

// 1 - f^p4 for f > 0, p4 < 0, cancellation-free near the surface (f -> 1).
// When n = -1/p4 is an exact integer (eps1 = 0.1 -> 20, 0.2 -> 10, 1 -> 2),
// f^p4 = 1/r with r = f^(1/n): an FP32 SFU seed refined by one FP64 Newton
// step on r^n = f (relative error ~ (n-1)/2 * (3e-7)^2), then
//   1 - f^p4 = (r - 1) / r        (r - 1 exact in FP64).
// Otherwise -expm1(p4 ln f) with ln f = log1p(f - 1) near the surface.
// Also returns 1/r (= f^p4) for the gradient.
template <int N4 = 0>
__device__ __forceinline__ double one_minus_pow(double f, double p4, int n_rt, double* F,
                                                double* inv_f = nullptr) {
  const int n = N4 > 0 ? N4 : n_rt;
  if constexpr (N4 == 2) {  // eps1 = 1 (ellipsoids): F = f^(-1/2) is one Newton-refined reciprocal square root
    const double Fv = rsqrt_d(f);
    *F = Fv;
    if (inv_f) *inv_f = Fv * Fv;
    return 1.0 - Fv;
  }
  if (n > 0) {
    // F = f^(-1/n). Seed F0 = 2^(-log2(f)/n): log2 from the exponent bits +
    // SFU lg2 of the mantissa, 2^q spliced from bits (any normal f). One
    // Newton step on F^-n = f:  F = F0 (1 + (1 - f F0^n) / n), relative error
    // ~ (n+1)/2 delta0^2 ~ 1e-12; then 1 - F is exact in FP64.
    const int hi = __double2hiint(f);
    const int ex = ((hi >> 20) & 0x7ff) - 1023;
    const float mant = __int_as_float(((hi & 0x000fffff) << 3) | 0x3f800000);  // top mantissa bits
    const float l = -((float)ex + lg2f(mant)) * (1.0f / (float)n);
    const float q = floorf(l);
    const double F0 = (double)ex2f(l - q) * __hiloint2double(((int)q + 1023) << 20, 0);
    const double Fn = N4 > 0 ? cpow<(N4 > 0 ? N4 : 1)>(F0) : ipow_d(F0, n);
    const double e = fma(-f, Fn, 1.0);  // f F0^n = 1 - e, |e| ~ n delta0
    const double Fv = fma(F0 * e, 1.0 / (double)n, F0);
    *F = Fv;
    // 1/f = F0^n / (1 - e) = F0^n (1 + e + e^2 + ...): two FMAs, error e^3
    if (inv_f) *inv_f = fma(Fn, fma(e, e, e), Fn);
    return 1.0 - Fv;
  }
  // ln f by log_d: forming 1 + d rounds by ~1e-16 ABSOLUTE, which is all
  // 1 - f^p4 needs (it feeds phi additively); expm1 by a Taylor polynomial
  // below |y| = 1e-3 (error y^5/120) and exp_d(y) - 1 above (absolute ~1e-12,
  // the Newton-step level of the integer branch)
  const double y = p4 * log_d(f);
  const double em1 = fabs(y) < 1e-3 ? y * fma(y, fma(y, fma(y, 1.0 / 24.0, 1.0 / 6.0), 0.5), 1.0) : exp_d(y) - 1.0;
  *F = 1.0 + em1;
  if (inv_f) *inv_f = rcp_d(f);
  return -em1;
}

// Dual overload: primal by the routine above (bit-identical to the value
// path), tangents by the chain rule d(f^p4) = p4 f^p4 / f df.
template <int N4 = 0, int N>
__device__ __forceinline__ Dual<N> one_minus_pow(const Dual<N>& f, double p4, int n_rt, Dual<N>* F,
                                                 Dual<N>* inv_f = nullptr) {
  double Fv, rf;
  const double om = one_minus_pow<N4>(f.v, p4, n_rt, &Fv, &rf);
  const double s = p4 * Fv * rf;
  *F = Dual<N>::chain(Fv, s, f);
  if (inv_f) *inv_f = Dual<N>::chain(rf, -rf * rf, f);
  return Dual<N>::chain(om, -s, f);
}

// Superquadric leaf (sdf.hpp:85-108). p in the BODY frame (FP64). N1..N4 > 0
// compile in the exponents (kSqE01); 0 reads them from the descriptor.
template <int FL, int N1 = 0, int N2 = 0, int N3 = 0, int N4 = 0, class T = double, int kFrame = -1>
__device__ __forceinline__ SdfOutT<T> sq_leaf(const DevSq& q, vec3<T> p) {
  // apply_inverse; kFrame 2: the leaf is known to be translation only (R = I
  // exactly, so p - t is the same result; the capsule's caps)
  if constexpr (kFrame == 2) p = p - mk3<T>(q.t[0], q.t[1], q.t[2]);
  else if (q.has_frame) p = mul_Rt(q.R, p - mk3<T>(q.t[0], q.t[1], q.t[2]));
  const T xn = p.x * q.inv_ax[0], yn = p.y * q.inv_ax[1], zn = p.z * q.inv_ax[2];
  const T x2 = fma(xn, xn, T(kMC.floor30)), y2 = fma(yn, yn, T(kMC.floor30)), z2 = fma(zn, zn, T(kMC.floor30));
  T A, Am1, B, Bm1, G, Gm1, Cz, Czm1;
  pow_pair_t<N1>(x2, q.n1, q.p1, A, Am1);
  pow_pair_t<N1>(y2, q.n1, q.p1, B, Bm1);
  const T g = A + B;
  pow_pair_t<N2>(g, q.n2, q.p2, G, Gm1);
  pow_pair_t<N3>(z2, q.n3, q.p3, Cz, Czm1);
  const T f = G + Cz;
  SdfOutT<T> out;
  out.v = 0.0;
  out.g = mk3<T>(0.0, 0.0, 0.0);
  if (FL == kValue) {
    const T r2 = fma(xn, xn, fma(yn, yn, fma(zn, zn, T(kMC.floor20))));
    T F;
    out.v = one_minus_pow<N4>(f, q.p4, q.n4, &F) * rsqrt_d(r2);  // (1 - f^p4) / |x~|
    return out;
  }
  // grad f w.r.t. the normalised coordinates (d(x2^p1)/dxn = 2 p1 x2^(p1-1) xn);
  // the body-frame gradient is diag(1/axes) times it.
  const T cxy = q.c_xy * Gm1;
  if (FL == kNormalOnly || FL == kNormalSource) {
    const vec3<T> dfn = mk3<T>(cxy * Am1 * xn, cxy * Bm1 * yn, q.c_z * Czm1 * zn);
    const vec3<T> df = mk3<T>(dfn.x * q.inv_ax[0], dfn.y * q.inv_ax[1], dfn.z * q.inv_ax[2]);
    if (FL == kNormalSource) {
      const T r2 = fma(xn, xn, fma(yn, yn, fma(zn, zn, T(kMC.floor20))));
      T F;
      out.v = one_minus_pow<N4>(f, q.p4, q.n4, &F) * rsqrt_d(r2);
    }
    out.g = (kFrame != 2 && q.has_frame) ? mul_R(q.R, df) : df;
    return out;
  }
  // kGrad: grad phi = diag(1/axes) (-p4 (F/f) grad_n f - phi x~ / r) / r
  const T r2 = fma(xn, xn, fma(yn, yn, fma(zn, zn, T(kMC.floor20))));
  const T rinv = rsqrt_d(r2);
  T F, inv_f;
  const T omF = one_minus_pow<N4>(f, q.p4, q.n4, &F, &inv_f);
  const T phi = omF * rinv;
  out.v = phi;
  const T k = -q.p4 * F * inv_f;
  const T h = phi * rinv;
  const T sx = q.inv_ax[0] * rinv, sy = q.inv_ax[1] * rinv, sz = q.inv_ax[2] * rinv;
  // component i: s_i x~_i (k c A_i' - h) with c A_i' x~_i = d f / d x~_i (factored: 2 fewer products each)
  const T kxy = k * cxy, kz = k * q.c_z;
  const vec3<T> gl = mk3<T>(sx * (xn * fma(kxy, Am1, -h)), sy * (yn * fma(kxy, Bm1, -h)),
                            sz * (zn * fma(kz, Czm1, -h)));
  out.g = (kFrame != 2 && q.has_frame) ? mul_R(q.R, gl) : gl;
  return out;
}

// Convex polyhedron leaf: LSE over plane distances (sdf.hpp:110-117).
// Pool per plane: double4 (n.x, n.y, n.z, n . point); distances in FP64.
template <int FL, class T = double>
__device__ __forceinline__ SdfOutT<T> cp_leaf(const DevNode& nd, const double4* pool, vec3<T> p) {
  const double4* pl = pool + nd.offset;
  T m = -INFINITY;
#pragma unroll 1
  for (int i = 0; i < nd.count; ++i) {
    const double4 q = pl[i];
    m = max_sel(m, fma(T(q.x), p.x, fma(T(q.y), p.y, fma(T(q.z), p.z, T(-q.w)))));
  }
  T acc = 0.0;
  vec3<T> g = mk3<T>(0.0, 0.0, 0.0);
#pragma unroll 1
  for (int i = 0; i < nd.count; ++i) {
    const double4 q = pl[i];
    const T d = fma(T(q.x), p.x, fma(T(q.y), p.y, fma(T(q.z), p.z, T(-q.w))));
    const T e = exp_d((d - m) * nd.inv_tau_d);
    acc += e;
    if (FL != kValue) g = g + mk3<T>(e * q.x, e * q.y, e * q.z);
  }
  SdfOutT<T> out;
  out.v = m + nd.tau_d * log_d(acc);
  out.g = mk3<T>(0.0, 0.0, 0.0);
  if (FL != kValue) out.g = dscale(g, rcp_d(acc));
  return out;
}

// kBoxCp: cp_leaf for the 6 axis-aligned box planes. With unit normals the
// FMA dot of cp_leaf is exactly +-p_i - w_k (the zero products add exact
// zeros) and the gradient sum is (e0 - e1, e2 - e3, e4 - e5): bit-identical to
// cp_leaf without the plane loads and 18 of its 24 FMAs per pass.
template <int FL, class T = double>
__device__ __forceinline__ SdfOutT<T> box_cp_leaf(const DevNode& nd, vec3<T> p) {
  const T d[6] = {p.x - nd.box_w[0], -p.x - nd.box_w[1], p.y - nd.box_w[2],
                  -p.y - nd.box_w[3], p.z - nd.box_w[4], -p.z - nd.box_w[5]};
  T m = -INFINITY;
#pragma unroll
  for (int i = 0; i < 6; ++i) m = max_sel(m, d[i]);
  T e[6], acc = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    e[i] = exp_d((d[i] - m) * nd.inv_tau_d);
    acc += e[i];
  }
  SdfOutT<T> out;
  out.v = m + nd.tau_d * log_d(acc);
  out.g = mk3<T>(0.0, 0.0, 0.0);
  if (FL != kValue) out.g = dscale(mk3<T>(e[0] - e[1], e[2] - e[3], e[4] - e[5]), rcp_d(acc));
  return out;
}

// Oriented pointcloud leaf (sdf.hpp:119-132). Pool per point: double4
// (p, -1/(2 th^2)), double4 (n, 1/th^2). Sums in FP64.
template <int FL, class T = double>
__device__ __forceinline__ SdfOutT<T> opc_leaf(const DevNode& nd, const double4* pool, vec3<T> p) {
  const double4* pt = pool + nd.offset;
  T num = 0.0, den = 1e-30;
  vec3<T> dnum = mk3<T>(0.0, 0.0, 0.0), dden = mk3<T>(0.0, 0.0, 0.0);
#pragma unroll 1
  for (int i = 0; i < nd.count; ++i) {
    const double4 a = pt[2 * i], b = pt[2 * i + 1];
    const T rx = p.x - a.x, ry = p.y - a.y, rz = p.z - a.z;
    const T arg = (rx * rx + ry * ry + rz * rz) * a.w;
    const T w = exp_d(arg);
    const T nr = b.x * rx + b.y * ry + b.z * rz;
    num = fma(w, nr, num);
    den += w;
    if (FL != kValue) {
      const T s = -w * b.w;  // dw = -w r / th^2
      dnum = dnum + mk3<T>(s * rx * nr + w * b.x, s * ry * nr + w * b.y, s * rz * nr + w * b.z);
      dden = dden + mk3<T>(s * rx, s * ry, s * rz);
    }
  }
  SdfOutT<T> out;
  const T inv = rcp_d(den);
  out.v = num * inv;
  out.g = mk3<T>(0.0, 0.0, 0.0);
  if (FL != kValue)
    out.g = mk3<T>((dnum.x - out.v * dden.x) * inv, (dnum.y - out.v * dden.y) * inv,
               (dnum.z - out.v * dden.z) * inv);
  return out;
}

template <int FL, class T = double>
__device__ __forceinline__ SdfOutT<T> leaf_eval(const DevNode& nd, const double4* pool, vec3<T> p) {
  if (nd.op == 0) return sq_leaf<FL, 0, 0, 0, 0, T>(nd.sq, p);
  if (nd.op == 1) return cp_leaf<FL, T>(nd, pool, p);
  return opc_leaf<FL, T>(nd, pool, p);
}

// Full program evaluation in the BODY frame. KIND (SdfKind) is a compile-time
// specialisation chosen on the host per surface: each kernel instantiation
// carries only the field code it needs (I-cache footprint).
// The generic postfix interpreter; Nodes = the parameter block's node array
// (indexed in constant space, as before) or a device-memory pointer.
template <int FL, class T, class Nodes>
__device__ __forceinline__ SdfOutT<T> interpret(const Nodes& nodes, int n_nodes, const double4* pool, vec3<T> p) {
  constexpr bool kWantG = FL != kValue;
  T sv[kMaxStack];
  vec3<T> sg[kMaxStack];
  int sp = 0;
#pragma unroll 1
  for (int i = 0; i < n_nodes; ++i) {
    const DevNode& nd = nodes[i];
    if (nd.op <= 2) {
      const SdfOutT<T> r = leaf_eval<FL, T>(nd, pool, p);
      sv[sp] = r.v;
      sg[sp] = r.g;
      ++sp;
    } else if (nd.op == 3) {  // union: softmin weights, first minimum
      const int n = nd.count, base = sp - n;
      T m = sv[base];
#pragma unroll 1
      for (int k = 1; k < n; ++k) m = fmin(m, sv[base + k]);
      T acc = 0.0;
      vec3<T> g = mk3<T>(0.0, 0.0, 0.0);
#pragma unroll 1
      for (int k = 0; k < n; ++k) {
        const T arg = (m - sv[base + k]) * nd.inv_tau_d;
        const T e = exp_d(arg);
        acc += e;
        if (kWantG) g = g + dscale(sg[base + k], e);
      }
      sp = base;
      sv[sp] = m - nd.tau_d * log_d(acc);
      sg[sp] = kWantG ? dscale(g, rcp_d(acc)) : mk3<T>(0.0, 0.0, 0.0);
      ++sp;
    } else {  // subtraction: args (phi+, -phi-), softmax weights
      const int a = sp - 2, b = sp - 1;
      const T a0 = sv[a], a1 = -sv[b];
      const T m = fmax(a0, a1);
      const T e0 = exp_d((a0 - m) * nd.inv_tau_d);
      const T e1 = exp_d((a1 - m) * nd.inv_tau_d);
      const T acc = e0 + e1;
      sv[a] = m + nd.tau_d * log_d(acc);
      if (kWantG) {
        const T inv = rcp_d(acc);
        sg[a] = dscale(sg[a], e0 * inv) - dscale(sg[b], e1 * inv);
      }
      sp = a + 1;
    }
  }
  SdfOutT<T> out;
  out.v = sv[0];
  out.g = sg[0];
  return out;
}

template <int FL_IN, int KIND, class T = double>
__device__ SdfOutT<T> sdf_eval(const DevSdf& s, vec3<T> p) {
  if constexpr (KIND == kSingleSq) return sq_leaf<FL_IN, 0, 0, 0, 0, T>(s.nodes[0].sq, p);
  if constexpr (ct_sq(KIND)) {
    constexpr SqExpTuple e = sq_exps(KIND);
    return sq_leaf<FL_IN, e.n1, e.n2, e.n3, e.n4, T>(s.nodes[0].sq, p);
  }
  // kNormalOnly skips phi only for a lone SQ leaf; compositions need the values.
  constexpr int FL = FL_IN == kNormalOnly ? kNormalSource : FL_IN;
  constexpr bool kWantG = FL != kValue;
  if constexpr (KIND == kCapsule) {
    // union of three compile-time superquadric leaves (sdf.hpp smooth union:
    // m - tau log sum exp((m - v_i) / tau), m = min v_i, gradient blended by the
    // same weights), accumulated online so only one leaf's result is live at a
    // time (the three-leaf form spills at the 64-register budget): the running
    // minimum m with sum S = sum exp((m - v_i) / tau) and blended gradient G;
    // a new leaf below m rescales both by exp((v - m) / tau). Two exponentials
    // (the reference's exp(0) of the minimum is 1 exactly) instead of three.
    constexpr SqExpTuple a = sq_exps(kSqCyl), b = sq_exps(kSqEll);
    const DevNode& un = s.nodes[3];
    const SdfOutT<T> r0 = sq_leaf<FL, a.n1, a.n2, a.n3, a.n4, T>(s.nodes[0].sq, p);
    T m = r0.v, acc = 1.0;
    vec3<T> g = r0.g;
    auto add = [&](const SdfOutT<T>& r) {
      const T d = r.v - m;
      const bool below = pv(d) < 0.0;
      const T e = exp_d(-fabs(d) * un.inv_tau_d);  // exp((m - v) / tau) or exp((v - m) / tau)
      if (below) {  // new minimum: rescale the running sums
        acc = fma(acc, e, T(1.0));
        if constexpr (kWantG) g = dscale(g, e) + r.g;
        m = r.v;
      } else {
        acc += e;
        if constexpr (kWantG) g = g + dscale(r.g, e);
      }
    };
    add(sq_leaf<FL, b.n1, b.n2, b.n3, b.n4, T, 2>(s.nodes[1].sq, p));  // caps: translation only (host)
    add(sq_leaf<FL, b.n1, b.n2, b.n3, b.n4, T, 2>(s.nodes[2].sq, p));
    SdfOutT<T> out;
    out.v = m - un.tau_d * log_d(acc);
    out.g = mk3<T>(0.0, 0.0, 0.0);
    if constexpr (kWantG) out.g = dscale(g, rcp_d(acc));
    return out;
  }
  if constexpr (KIND == kSingleCp) return cp_leaf<FL, T>(s.nodes[0], s.pool, p);
  if constexpr (KIND == kBoxCp) return box_cp_leaf<FL, T>(s.nodes[0], p);
  // Generic postfix interpreter (union: -LSE(-phi), subtraction: LSE(phi+, -phi-);
  // sdf.hpp:222-230, 260-287). Warp-uniform control flow. Nodes from the
  // parameter block, or from device memory for programs above kMaxNodes.
  if (s.ext) return interpret<FL, T>(s.ext, s.n_nodes, s.pool, p);
  return interpret<FL, T>(s.nodes, s.n_nodes, s.pool, p);
}

}  // namespace cmgb
