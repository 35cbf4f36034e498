// K6: batched witness points — run_ee_batch / run_vf_batch (src/batch.cpp:53-98)
// over ee_witness / vf_witness (include/cmg/witness.hpp:137-227).
//
// One thread per pair, grid-stride over a persistent grid (SM count x
// resident blocks). The pair stream is HBM-bound (96 B FP64 in + 24 B FP32
// out per E-E pair), so each warp's loads/stores are staged through shared
// memory to keep every global transaction a full 128-byte line.
#include <cuda_runtime.h>

#include "../common.h"
#include "../device/witness.cuh"

namespace cmgb {

namespace {

constexpr int kWitnessThreads = 256;

template <typename T>
__device__ __forceinline__ double3 load3(const T* p) {
  return d3((double)p[0], (double)p[1], (double)p[2]);
}

// Cooperative, coalesced copy of a block's contiguous input tile into smem.
template <typename T>
__device__ __forceinline__ void stage_in(const T* __restrict__ src, T* dst, int64_t first,
                                         int count, int width) {
  const int64_t base = first * width;
  const int total = count * width;
  for (int i = threadIdx.x; i < total; i += blockDim.x) dst[i] = src[base + i];
}

template <typename T>
__global__ void __launch_bounds__(kWitnessThreads)
    ee_witness_kernel(const __grid_constant__ WitnessParams p) {
  __shared__ T tile[kWitnessThreads * 12];
  __shared__ float otile[kWitnessThreads * 6];
  const T* __restrict__ in = static_cast<const T*>(p.pairs);
  for (int64_t first = (int64_t)blockIdx.x * kWitnessThreads; first < p.n;
       first += (int64_t)gridDim.x * kWitnessThreads) {
    const int count = (int)(p.n - first < kWitnessThreads ? p.n - first : kWitnessThreads);
    stage_in(in, tile, first, count, 12);
    __syncthreads();
    const int i = threadIdx.x;
    if (i < count) {
      const T* q = tile + 12 * i;
      const double3 e1a = load3(q), e1b = load3(q + 3), e2a = load3(q + 6), e2b = load3(q + 9);
      const QpSol s = ee_qp(e1a, e1b, e2a, e2b, p.cfg);
      const double3 p1 = e1a + (e1b - e1a) * s.a1;  // edge_point (witness.hpp:130-133)
      const double3 p2 = e2a + (e2b - e2a) * s.a2;
      float* o = otile + 6 * i;
      o[0] = (float)p1.x; o[1] = (float)p1.y; o[2] = (float)p1.z;
      o[3] = (float)p2.x; o[4] = (float)p2.y; o[5] = (float)p2.z;
      if (p.alpha_gamma) {
        float* ag = p.alpha_gamma + 3 * (first + i);
        ag[0] = (float)s.a1;
        ag[1] = (float)s.a2;
        ag[2] = s.gamma;
      }
      if (p.labels) p.labels[first + i] = s.label;
    }
    __syncthreads();
    float* __restrict__ out = p.out + first * 6;
    for (int k = threadIdx.x; k < count * 6; k += blockDim.x) out[k] = otile[k];
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(kWitnessThreads)
    vf_witness_kernel(const __grid_constant__ WitnessParams p) {
  __shared__ T tile[kWitnessThreads * 12];
  __shared__ float otile[kWitnessThreads * 3];
  const T* __restrict__ in = static_cast<const T*>(p.pairs);
  for (int64_t first = (int64_t)blockIdx.x * kWitnessThreads; first < p.n;
       first += (int64_t)gridDim.x * kWitnessThreads) {
    const int count = (int)(p.n - first < kWitnessThreads ? p.n - first : kWitnessThreads);
    stage_in(in, tile, first, count, 12);
    __syncthreads();
    const int i = threadIdx.x;
    if (i < count) {
      const T* q = tile + 12 * i;
      int label;
      const double3 r = vf_witness(load3(q), load3(q + 3), load3(q + 6), load3(q + 9), p.cfg,
                                   &label);
      float* o = otile + 3 * i;
      o[0] = (float)r.x; o[1] = (float)r.y; o[2] = (float)r.z;
      if (p.labels) p.labels[first + i] = label;
    }
    __syncthreads();
    float* __restrict__ out = p.out + first * 3;
    for (int k = threadIdx.x; k < count * 3; k += blockDim.x) out[k] = otile[k];
    __syncthreads();
  }
}

int grid_for(int64_t n, const void* kernel) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kWitnessThreads, 0);
  const int64_t need = (n + kWitnessThreads - 1) / kWitnessThreads;
  const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  return (int)(need < cap ? (need > 0 ? need : 1) : cap);
}

}  // namespace

int launch_ee_witness(const WitnessParams& p, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p.fp64) {
    const void* k = (const void*)ee_witness_kernel<double>;
    ee_witness_kernel<double><<<grid_for(p.n, k), kWitnessThreads, 0, s>>>(p);
  } else {
    const void* k = (const void*)ee_witness_kernel<float>;
    ee_witness_kernel<float><<<grid_for(p.n, k), kWitnessThreads, 0, s>>>(p);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_vf_witness(const WitnessParams& p, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p.fp64) {
    const void* k = (const void*)vf_witness_kernel<double>;
    vf_witness_kernel<double><<<grid_for(p.n, k), kWitnessThreads, 0, s>>>(p);
  } else {
    const void* k = (const void*)vf_witness_kernel<float>;
    vf_witness_kernel<float><<<grid_for(p.n, k), kWitnessThreads, 0, s>>>(p);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace cmgb
