// Host-side launch helpers shared by the kernel files.
#pragma once

#include <atomic>
#include <cstdint>

#include <cuda_runtime.h>

namespace cmgb {

// Host-side count of this library's kernel launches (exported as
// cmgb_kernel_launches): bench.py reads it around its timed regions, so the
// launch count it reports is measured, not claimed.
inline std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}
inline void note_launch() { launch_counter().fetch_add(1, std::memory_order_relaxed); }

// Runs f() once per CUDA device (function attributes such as the dynamic
// shared-memory limit are per device); idempotent f, so a racing second call is
// harmless.
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  template <class F>
  void operator()(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    f();
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
};

// Per-device cached integer (e.g. a persistent-grid size), computed on first use.
struct PerDeviceInt {
  std::atomic<int> v[64] = {};
  template <class F>
  int get(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::atomic<int>& slot = v[dev & 63];
    int x = slot.load(std::memory_order_acquire);
    if (x == 0) {
      x = f();
      slot.store(x, std::memory_order_release);
    }
    return x;
  }
};

// The current device's shared-memory budgets, cached per device: the opt-in
// maximum per block (the dynamic-smem attribute every kernel sets, and the
// largest per-env working set a plan may use) and the capacity per SM (what
// the resident-CTA targets divide; the runtime reserves 1 KB per CTA).
inline int smem_optin_per_block() {
  static PerDeviceInt c;
  return c.get([] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v > 0 ? v : 48 * 1024;
  });
}
inline int smem_per_sm() {
  static PerDeviceInt c;
  return c.get([] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    return v > 0 ? v : 48 * 1024;
  });
}
constexpr int kSmemReservedPerCta = 1024;

// Lets kernel `fn` take the device's full opt-in shared memory as dynamic
// shared memory (less its static shared memory: the sum may not exceed the
// opt-in limit, or the attribute call fails).
template <class K>
inline void allow_max_dynamic_smem(K* fn) {
  cudaFuncAttributes a{};
  const int st = cudaFuncGetAttributes(&a, fn) == cudaSuccess ? (int)a.sharedSizeBytes : 0;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin_per_block() - st);
}

}  // namespace cmgb
