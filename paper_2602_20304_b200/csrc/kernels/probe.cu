// Roofline denominators not in MEASURED_PEAKS.json: sustained FP32 (FFMA) and
// FP64 (DFMA) throughput of this GPU at its current clocks, measured with
// independent FMA chains (8 per thread) on a full-occupancy grid.
#include <cuda_runtime.h>

#include "../../../include/cmgb_probe.h"
#include "launch_util.cuh"

namespace {

template <typename T>
__global__ void __launch_bounds__(256) fma_chain(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (T)(threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = x[k] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == (T)-1.2345) out[threadIdx.x] = s;  // keep the chains live
}

template <typename T>
double run(int iters, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  T* out = nullptr;
  cudaMalloc(&out, 256 * sizeof(T));
  const int grid = sms * 8;
  fma_chain<T><<<grid, 256, 0, s>>>(out, 64, (T)0.999, (T)0.001);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  fma_chain<T><<<grid, 256, 0, s>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  const double flops = 2.0 * 8.0 * iters * (double)grid * 256.0;
  return ms > 0.f ? flops / (ms * 1e-3) / 1e12 : 0.0;
}

}  // namespace

extern "C" int cmgb_probe_fma_tflops(int32_t fp64, int32_t iters, double* tflops, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  *tflops = fp64 ? run<double>(iters, s) : run<float>(iters, s);
  return cudaGetLastError() == cudaSuccess ? 0 : 3;
}

extern "C" uint64_t cmgb_kernel_launches(void) { return cmgb::launch_counter().load(std::memory_order_relaxed); }
