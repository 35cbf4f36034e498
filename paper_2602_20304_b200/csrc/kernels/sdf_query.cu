// Batched SDF queries and sphere tracing on one surface: SmoothSdf::value /
// value_and_gradient / value_and_normal_source (sdf.hpp:177-195) and
// sphere_trace_project against a posed SDF (sdf.hpp:318-326), one thread per
// point, through the same device field code as the manifold kernel (the
// surface's compile-time SDF kind included).
#include <cuda_runtime.h>

#include "launch_util.cuh"

#include "../common.h"
#include "../device/dmath.cuh"
#include "../device/sdf.cuh"

namespace cmgb {

namespace {

template <int FL, int KIND>
__global__ void __launch_bounds__(256) sdf_query_kernel(const __grid_constant__ SdfQueryParams q) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q.n) return;
  const double3 p = d3(q.points[3 * i], q.points[3 * i + 1], q.points[3 * i + 2]);
  const SdfOut s = sdf_eval<FL, KIND>(q.sdf, p);
  double* o = q.out + 4 * i;
  o[0] = s.v;
  o[1] = FL == kValue ? 0.0 : s.g.x;
  o[2] = FL == kValue ? 0.0 : s.g.y;
  o[3] = FL == kValue ? 0.0 : s.g.z;
}

// World point -> body frame, the manifold kernel's trace step (sdf.hpp:318-326
// in the body frame: rotations preserve the normalisation), -> world.
template <int KIND>
__global__ void __launch_bounds__(256) sphere_trace_kernel(const __grid_constant__ SdfQueryParams q) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q.n) return;
  const double3 pw = d3(q.points[3 * i], q.points[3 * i + 1], q.points[3 * i + 2]);
  double3 p = mul_Rt(q.R, pw - d3(q.t[0], q.t[1], q.t[2]));
  for (int k = 0; k < q.iters; ++k) {
    const SdfOut s = sdf_eval<kGrad, KIND>(q.sdf, p);
    const double sc = rsqrt_d(q.tau + ddot(s.g, s.g)) * s.v;
    p = d3(fma(-s.g.x, sc, p.x), fma(-s.g.y, sc, p.y), fma(-s.g.z, sc, p.z));
  }
  const double3 r = mul_R(q.R, p) + d3(q.t[0], q.t[1], q.t[2]);
  q.out[3 * i] = r.x;
  q.out[3 * i + 1] = r.y;
  q.out[3 * i + 2] = r.z;
}

template <int KIND>
int launch_query_kind(const SdfQueryParams& q, int mode, cudaStream_t s) {
  const unsigned grid = (unsigned)((q.n + 255) / 256);
  switch (mode) {
    case 0: note_launch(); sdf_query_kernel<kValue, KIND><<<grid, 256, 0, s>>>(q); break;
    case 1: note_launch(); sdf_query_kernel<kGrad, KIND><<<grid, 256, 0, s>>>(q); break;
    case 2: note_launch(); sdf_query_kernel<kNormalSource, KIND><<<grid, 256, 0, s>>>(q); break;
    default: note_launch(); sphere_trace_kernel<KIND><<<grid, 256, 0, s>>>(q); break;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace

// mode 0 / 1 / 2: value / gradient / normal source; 3: sphere trace.
int launch_sdf_query(const SdfQueryParams& q, int mode, void* stream) {
  if (q.n <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (q.sdf.kind) {
    case kSqE01: return launch_query_kind<kSqE01>(q, mode, s);
    case kSingleSq: return launch_query_kind<kSingleSq>(q, mode, s);
    case kSingleCp: return launch_query_kind<kSingleCp>(q, mode, s);
    case kBoxCp: return launch_query_kind<kBoxCp>(q, mode, s);
    default: return launch_query_kind<kGeneric>(q, mode, s);
  }
}

}  // namespace cmgb
