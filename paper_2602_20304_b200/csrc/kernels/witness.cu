// K6: batched witness points — run_ee_batch / run_vf_batch (src/batch.cpp:53-98)
// over ee_witness / vf_witness (include/cmg/witness.hpp:137-227).
//
// One thread per pair, grid-stride over a persistent grid (SM count x
// resident blocks). The pair stream is HBM-bound (96 B FP64 in + 24 B FP32
// out per E-E pair): input tiles arrive by TMA bulk copy into a double buffer
// (device/bulk.cuh), outputs are staged so stores are full lines.
#include <cuda_runtime.h>

#include "../common.h"
#include "launch_util.cuh"
#include "../device/bulk.cuh"
#include "../device/witness.cuh"

namespace cmgb {

namespace {

// 128 threads, one pair each per tile; two input tiles in flight per CTA.
constexpr int kWitnessThreads = 128;

template <typename T>
__device__ __forceinline__ double3 load3(const T* p) {
  return d3((double)p[0], (double)p[1], (double)p[2]);
}

struct EeSolve {
  using Out = float;
  static constexpr int kOut = 6;
  template <int kH, typename T>
  __device__ __forceinline__ static void run(const WitnessParams& p, const T* q, int64_t idx, float* o) {
    const double3 e1a = load3(q), e1b = load3(q + 3), e2a = load3(q + 6), e2b = load3(q + 9);
    const QpSol s = ee_qp<double, float, false, kH>(e1a, e1b, e2a, e2b, p.cfg);  // FP32 indicators (witness.cuh)
    const double3 p1 = e1a + (e1b - e1a) * s.a1;  // edge_point (witness.hpp:130-133)
    const double3 p2 = e2a + (e2b - e2a) * s.a2;
    o[0] = (float)p1.x; o[1] = (float)p1.y; o[2] = (float)p1.z;
    o[3] = (float)p2.x; o[4] = (float)p2.y; o[5] = (float)p2.z;
    if (p.alpha_gamma) {
      float* ag = p.alpha_gamma + 3 * idx;
      ag[0] = (float)s.a1;
      ag[1] = (float)s.a2;
      ag[2] = (float)s.gamma;
    }
    if (p.labels) p.labels[idx] = s.label;
  }
};

// Reference-precision E-E witness (FP64 indicators and outputs): what
// ee_witness<double> returns, for callers that difference the witness points
// (the rotating-edge sweep's theta-derivative, sweep.cpp:44-56).
struct EeSolve64 {
  using Out = double;
  static constexpr int kOut = 6;
  template <int kH, typename T>
  __device__ __forceinline__ static void run(const WitnessParams& p, const T* q, int64_t idx, double* o) {
    const double3 e1a = load3(q), e1b = load3(q + 3), e2a = load3(q + 6), e2b = load3(q + 9);
    const QpSol s = ee_qp<double, double, true, kH>(e1a, e1b, e2a, e2b, p.cfg);
    const double3 p1 = e1a + (e1b - e1a) * s.a1;
    const double3 p2 = e2a + (e2b - e2a) * s.a2;
    o[0] = p1.x; o[1] = p1.y; o[2] = p1.z;
    o[3] = p2.x; o[4] = p2.y; o[5] = p2.z;
    if (p.alpha_gamma_f64) {
      double* ag = static_cast<double*>(p.alpha_gamma_f64) + 3 * idx;
      ag[0] = s.a1;
      ag[1] = s.a2;
      ag[2] = s.gamma;
    }
    if (p.labels) p.labels[idx] = s.label;
  }
};

struct VfSolve {
  using Out = float;
  static constexpr int kOut = 3;
  template <int kH, typename T>
  __device__ __forceinline__ static void run(const WitnessParams& p, const T* q, int64_t idx, float* o) {
    int label;
    const double3 r = vf_witness<float, kH>(load3(q), load3(q + 3), load3(q + 6), load3(q + 9), p.cfg, &label);
    o[0] = (float)r.x; o[1] = (float)r.y; o[2] = (float)r.z;
    if (p.labels) p.labels[idx] = label;
  }
};

// Persistent grid-stride over tiles of kWitnessThreads pairs. The input tiles
// (96 B / pair FP64, 48 B FP32) arrive by TMA bulk copies into a kStages-deep
// ring: kStages - 1 tiles stream in while the CTA solves the current one.
// Outputs are staged in shared memory so the global stores are full lines.
constexpr int kStages = 2;  // measured: deeper rings cost resident CTAs (4 stages: 16 warps/SM, -40%)

// kH: the solver's operator mode (hard_ops) fixed at compile time.
template <typename T, class Solve, int kH>
__global__ void __launch_bounds__(kWitnessThreads) witness_kernel(const __grid_constant__ WitnessParams p) {
  constexpr int W = Solve::kOut;
  using Out = typename Solve::Out;
  extern __shared__ __align__(128) unsigned char dsm[];  // kStages input tiles, then the output tile
  T(*tile)[kWitnessThreads * 12] = reinterpret_cast<T(*)[kWitnessThreads * 12]>(dsm);
  Out* otile = reinterpret_cast<Out*>(dsm + sizeof(T) * kStages * kWitnessThreads * 12);
  __shared__ __align__(8) uint64_t bar[kStages];
  const T* __restrict__ in = static_cast<const T*>(p.pairs);
  const int tid = threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kWitnessThreads;
  int64_t first = (int64_t)blockIdx.x * kWitnessThreads;
  auto issue = [&](int64_t f, int b) {
    const int cnt = (int)(p.n - f < kWitnessThreads ? p.n - f : kWitnessThreads);
    const uint32_t bytes = (uint32_t)(cnt * 12 * sizeof(T));  // 48 / 96 B per pair: multiple of 16
    mbar_arrive_expect_tx(&bar[b], bytes);
    bulk_g2s(tile[b], in + f * 12, bytes, &bar[b]);
  };
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < kStages; ++b) mbar_init(&bar[b], 1);
    mbar_fence_init();
#pragma unroll
    for (int k = 0; k < kStages - 1; ++k)
      if (first + k * stride < p.n) issue(first + k * stride, k);
  }
  __syncthreads();
  for (int it = 0; first < p.n; first += stride, ++it) {
    const int b = it % kStages;
    // refill the buffer consumed by the previous iteration (its readers
    // finished at that iteration's first barrier)
    const int64_t ahead = first + (int64_t)(kStages - 1) * stride;
    if (tid == 0 && ahead < p.n) {
      fence_proxy_async_smem();
      issue(ahead, (it + kStages - 1) % kStages);
    }
    const int count = (int)(p.n - first < kWitnessThreads ? p.n - first : kWitnessThreads);
    mbar_wait(&bar[b], (it / kStages) & 1);
    if (tid < count) Solve::template run<kH>(p, tile[b] + 12 * tid, first + tid, otile + W * tid);
    __syncthreads();
    Out* __restrict__ out = static_cast<Out*>(p.out_any) + first * W;
    for (int k = tid; k < count * W; k += kWitnessThreads) out[k] = otile[k];
    __syncthreads();
  }
}

template <typename T, class Solve, int kH>
int launch_witness_mode(const WitnessParams& p, cudaStream_t s) {
  constexpr size_t smem = sizeof(T) * kStages * kWitnessThreads * 12 +
                          sizeof(typename Solve::Out) * kWitnessThreads * Solve::kOut;
  static PerDeviceInt cap_cache;  // persistent grid: SMs x resident CTAs, per device
  const int cap = cap_cache.get([] {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaFuncSetAttribute(witness_kernel<T, Solve, kH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, witness_kernel<T, Solve, kH>, kWitnessThreads, smem);
    return sms * (per_sm > 0 ? per_sm : 1);
  });
  const int64_t need = (p.n + kWitnessThreads - 1) / kWitnessThreads;
  const int grid = (int)(need < cap ? (need > 0 ? need : 1) : cap);
  note_launch();
  witness_kernel<T, Solve, kH><<<grid, kWitnessThreads, smem, s>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

template <typename T, class Solve>
int launch_witness(const WitnessParams& p, cudaStream_t s) {
  return p.cfg.hard_ops ? launch_witness_mode<T, Solve, 1>(p, s) : launch_witness_mode<T, Solve, 0>(p, s);
}

// FP32 -> FP64 widening of the V-F outputs for the host-buffer call (the
// reference's run_vf_batch writes doubles): on the device, so the D2H of a
// pipeline chunk lands in the caller's buffer directly.
__global__ void widen_kernel(const float* __restrict__ src, double* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (double)src[i];
}

}  // namespace

int launch_widen(const float* src, double* dst, int64_t n, void* stream) {
  if (n <= 0) return 0;
  const int64_t need = (n + 255) / 256;
  const int grid = (int)(need < 148 * 8 ? need : 148 * 8);
  note_launch();
  widen_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, dst, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_ee_witness(const WitnessParams& p, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p.fp64 ? launch_witness<double, EeSolve>(p, s) : launch_witness<float, EeSolve>(p, s);
}

int launch_ee_witness_f64(const WitnessParams& p, void* stream) {
  return launch_witness<double, EeSolve64>(p, static_cast<cudaStream_t>(stream));
}

int launch_vf_witness(const WitnessParams& p, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return p.fp64 ? launch_witness<double, VfSolve>(p, s) : launch_witness<float, VfSolve>(p, s);
}

}  // namespace cmgb
