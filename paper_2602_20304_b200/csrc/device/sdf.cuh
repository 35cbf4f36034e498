// Device evaluation of the smooth analytical SDF programs (FP32).
//
// Three query flavours, as in the reference (sdf.hpp:177-195):
//   kValue         phi                       (penetration scores / pen sigmoids)
//   kGrad          phi, true grad phi        (sphere tracing, sdf.hpp:318-326)
//   kNormalSource  phi, composed normal field; SQ leaves contribute grad f
//                  (sdf.hpp:233-288)
// Gradients are analytic (the reference nests a Dual<3>; the derivative of
// the same expression graph).
#pragma once

#include "../common.h"
#include "dmath.cuh"

namespace cmgb {

struct SdfOut {
  float v;
  float3 g;
};

// Superquadric leaf in its canonical frame (sdf.hpp:85-108).
template <int FL>
__device__ __forceinline__ SdfOut sq_leaf(const DevSq& q, float3 p) {
  if (q.has_frame) {  // Transform::apply_inverse: R^T (p - t)
    const float dx = p.x - q.t[0], dy = p.y - q.t[1], dz = p.z - q.t[2];
    p = f3(q.R[0] * dx + q.R[3] * dy + q.R[6] * dz, q.R[1] * dx + q.R[4] * dy + q.R[7] * dz,
           q.R[2] * dx + q.R[5] * dy + q.R[8] * dz);
  }
  const float xn = p.x * q.inv_ax[0], yn = p.y * q.inv_ax[1], zn = p.z * q.inv_ax[2];
  const float x2 = fmaf(xn, xn, 1e-30f), y2 = fmaf(yn, yn, 1e-30f), z2 = fmaf(zn, zn, 1e-30f);
  float A, Am1, B, Bm1, G, Gm1, Cz, Czm1;
  pow_pair(x2, q.n1, q.p1, A, Am1);
  pow_pair(y2, q.n1, q.p1, B, Bm1);
  const float g = A + B;
  pow_pair(g, q.n2, q.p2, G, Gm1);
  pow_pair(z2, q.n3, q.p3, Cz, Czm1);
  const float f = G + Cz;
  SdfOut out;
  // df/dp through the normalisation (d x2^p1 = p1 x2^(p1-1) 2 xn / ax).
  const float cxy = 2.0f * q.p1 * q.p2 * Gm1;
  const float dfx = cxy * Am1 * xn * q.inv_ax[0];
  const float dfy = cxy * Bm1 * yn * q.inv_ax[1];
  const float dfz = 2.0f * q.p3 * Czm1 * zn * q.inv_ax[2];
  if (FL != kNormalOnly) {  // V-S contacts need phi with the normal source
    const float r2 = fmaf(xn, xn, fmaf(yn, yn, fmaf(zn, zn, 1e-20f)));
    const float rinv = rsqf(r2);
    float F;
    if (q.p4kind == kPowRsqrt) F = rsqf(f);
    else if (q.p4kind == kPowRcp) F = rcpf(f);
    else F = powg(f, q.p4);
    out.v = (1.0f - F) * rinv;
    if (FL == kGrad) {
      // grad phi = (-p4 F/f grad f - phi * (x~/axes) / r) / r
      const float k = -q.p4 * F * rcpf(f);
      const float h = out.v * rinv;
      float3 gl = f3((k * dfx - h * xn * q.inv_ax[0]) * rinv, (k * dfy - h * yn * q.inv_ax[1]) * rinv,
                     (k * dfz - h * zn * q.inv_ax[2]) * rinv);
      if (q.has_frame)
        gl = f3(q.R[0] * gl.x + q.R[1] * gl.y + q.R[2] * gl.z, q.R[3] * gl.x + q.R[4] * gl.y + q.R[5] * gl.z,
                q.R[6] * gl.x + q.R[7] * gl.y + q.R[8] * gl.z);
      out.g = gl;
    }
  }
  if (FL == kNormalSource || FL == kNormalOnly) {
    float3 gl = f3(dfx, dfy, dfz);
    if (q.has_frame)
      gl = f3(q.R[0] * gl.x + q.R[1] * gl.y + q.R[2] * gl.z, q.R[3] * gl.x + q.R[4] * gl.y + q.R[5] * gl.z,
              q.R[6] * gl.x + q.R[7] * gl.y + q.R[8] * gl.z);
    out.g = gl;
  }
  return out;
}

// Convex polyhedron leaf: LSE over plane distances (sdf.hpp:110-117).
// Pool entry per plane: (n.x, n.y, n.z, n . point).
template <int FL>
__device__ __forceinline__ SdfOut cp_leaf(const DevNode& nd, const float4* pool, float3 p) {
  const float4* pl = pool + nd.offset;
  float m = -INFINITY;
#pragma unroll 1
  for (int i = 0; i < nd.count; ++i) {
    const float4 q = pl[i];
    const float d = fmaf(q.x, p.x, fmaf(q.y, p.y, fmaf(q.z, p.z, -q.w)));
    m = fmaxf(m, d);
  }
  float acc = 0.0f;
  float3 g = f3(0.f, 0.f, 0.f);
#pragma unroll 1
  for (int i = 0; i < nd.count; ++i) {
    const float4 q = pl[i];
    const float d = fmaf(q.x, p.x, fmaf(q.y, p.y, fmaf(q.z, p.z, -q.w)));
    const float e = __expf((d - m) * nd.inv_tau);
    acc += e;
    if (FL != kValue) {
      g.x = fmaf(e, q.x, g.x);
      g.y = fmaf(e, q.y, g.y);
      g.z = fmaf(e, q.z, g.z);
    }
  }
  SdfOut out;
  out.v = m + nd.tau * __logf(acc);
  if (FL != kValue) {
    const float inv = rcpf(acc);
    out.g = f3(g.x * inv, g.y * inv, g.z * inv);
  }
  return out;
}

// Oriented pointcloud leaf: Gaussian-RBF weighted plane distances
// (sdf.hpp:119-132). Pool per point: (p, -1/(2 th^2)), (n, 1/th^2).
template <int FL>
__device__ __forceinline__ SdfOut opc_leaf(const DevNode& nd, const float4* pool, float3 p) {
  const float4* pt = pool + nd.offset;
  float num = 0.0f, den = 1e-30f;
  float3 dnum = f3(0.f, 0.f, 0.f), dden = f3(0.f, 0.f, 0.f);
#pragma unroll 1
  for (int i = 0; i < nd.count; ++i) {
    const float4 a = pt[2 * i], b = pt[2 * i + 1];
    const float rx = p.x - a.x, ry = p.y - a.y, rz = p.z - a.z;
    const float w = __expf((rx * rx + ry * ry + rz * rz) * a.w);
    const float nr = b.x * rx + b.y * ry + b.z * rz;
    num = fmaf(w, nr, num);
    den += w;
    if (FL != kValue) {
      const float s = -w * b.w;  // dw = -w r / th^2
      dnum.x += s * rx * nr + w * b.x;
      dnum.y += s * ry * nr + w * b.y;
      dnum.z += s * rz * nr + w * b.z;
      dden.x += s * rx;
      dden.y += s * ry;
      dden.z += s * rz;
    }
  }
  SdfOut out;
  const float inv = __frcp_rn(den);
  out.v = num * inv;
  if (FL != kValue)
    out.g = f3((dnum.x - out.v * dden.x) * inv, (dnum.y - out.v * dden.y) * inv,
               (dnum.z - out.v * dden.z) * inv);
  return out;
}

template <int FL>
__device__ __forceinline__ SdfOut leaf_eval(const DevNode& nd, const float4* pool, float3 p) {
  if (nd.op == 0) return sq_leaf<FL>(nd.sq, p);
  if (nd.op == 1) return cp_leaf<FL>(nd, pool, p);
  return opc_leaf<FL>(nd, pool, p);
}

// Full program evaluation in the BODY frame.
template <int FL_IN>
__device__ SdfOut sdf_eval(const DevSdf& s, float3 p) {
  if (s.kind == kSingleSq) return sq_leaf<FL_IN>(s.nodes[0].sq, p);
  // kNormalOnly skips phi only for a lone SQ leaf; compositions need the values.
  constexpr int FL = FL_IN == kNormalOnly ? kNormalSource : FL_IN;
  if (s.kind == kSingleCp) return cp_leaf<FL>(s.nodes[0], s.pool, p);
  // Generic postfix interpreter (union: -LSE(-phi), subtraction: LSE(phi+, -phi-);
  // sdf.hpp:222-230, 260-287). Warp-uniform control flow.
  float sv[kMaxStack], sx[kMaxStack], sy[kMaxStack], sz[kMaxStack];
  int sp = 0;
#pragma unroll 1
  for (int i = 0; i < s.n_nodes; ++i) {
    const DevNode& nd = s.nodes[i];
    if (nd.op <= 2) {
      const SdfOut r = leaf_eval<FL>(nd, s.pool, p);
      sv[sp] = r.v;
      if (FL != kValue) { sx[sp] = r.g.x; sy[sp] = r.g.y; sz[sp] = r.g.z; }
      ++sp;
    } else if (nd.op == 3) {  // union: weights softmin(phi_i / tau), first minimum
      const int n = nd.count, base = sp - n;
      float m = sv[base];
#pragma unroll 1
      for (int k = 1; k < n; ++k) m = fminf(m, sv[base + k]);
      float acc = 0.f, gx = 0.f, gy = 0.f, gz = 0.f;
#pragma unroll 1
      for (int k = 0; k < n; ++k) {
        const float e = __expf((m - sv[base + k]) * nd.inv_tau);
        acc += e;
        if (FL != kValue) { gx = fmaf(e, sx[base + k], gx); gy = fmaf(e, sy[base + k], gy); gz = fmaf(e, sz[base + k], gz); }
      }
      sp = base;
      sv[sp] = m - nd.tau * __logf(acc);
      if (FL != kValue) {
        const float inv = rcpf(acc);
        sx[sp] = gx * inv; sy[sp] = gy * inv; sz[sp] = gz * inv;
      }
      ++sp;
    } else {  // subtraction: args (phi+, -phi-), softmax weights
      const int a = sp - 2, b = sp - 1;
      const float a0 = sv[a], a1 = -sv[b];
      const float m = fmaxf(a0, a1);
      const float e0 = __expf((a0 - m) * nd.inv_tau), e1 = __expf((a1 - m) * nd.inv_tau);
      const float acc = e0 + e1;
      sv[a] = m + nd.tau * __logf(acc);
      if (FL != kValue) {
        const float inv = rcpf(acc);
        const float w0 = e0 * inv, w1 = e1 * inv;
        sx[a] = w0 * sx[a] - w1 * sx[b];
        sy[a] = w0 * sy[a] - w1 * sy[b];
        sz[a] = w0 * sz[a] - w1 * sz[b];
      }
      sp = a + 1;
    }
  }
  SdfOut out;
  out.v = sv[0];
  out.g = FL != kValue ? f3(sx[0], sy[0], sz[0]) : f3(0.f, 0.f, 0.f);
  return out;
}

}  // namespace cmgb
