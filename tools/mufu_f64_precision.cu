// Measures the relative error of the FP64 MUFU seeds (rcp/rsqrt.approx.ftz.f64)
// and of one / two Newton steps on them (developer tool; decides how many
// refinement steps dmath.cuh needs). nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(int n, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // log-uniform x in [1e-6, 1e6]
  double x = exp(-13.8155 + 27.631 * ((double)i + 0.5) / n);
  double y, r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double ex = 1.0 / sqrt(x);
  double hx = 0.5 * x;
  double y1 = y * fma(-hx, y * y, 1.5);
  double y2 = y1 * fma(-hx, y1 * y1, 1.5);
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double er = 1.0 / x;
  double e = fma(-x, r, 1.0);
  double r1 = fma(r, e, r);
  double e2 = fma(-x, r1, 1.0);
  double r2 = fma(r1, e2, r1);
  out[6 * i + 0] = fabs(y / ex - 1);
  out[6 * i + 1] = fabs(y1 / ex - 1);
  out[6 * i + 2] = fabs(y2 / ex - 1);
  out[6 * i + 3] = fabs(r / er - 1);
  out[6 * i + 4] = fabs(r1 / er - 1);
  out[6 * i + 5] = fabs(r2 / er - 1);
}

int main() {
  const int n = 1 << 22;
  double* d;
  cudaMalloc(&d, sizeof(double) * 6 * n);
  k<<<n / 256, 256>>>(n, d);
  double* h = new double[6 * (size_t)n];
  cudaMemcpy(h, d, sizeof(double) * 6 * n, cudaMemcpyDeviceToHost);
  const char* names[6] = {"rsqrt seed", "rsqrt 1 NR", "rsqrt 2 NR", "rcp seed", "rcp 1 NR", "rcp 2 NR"};
  for (int j = 0; j < 6; ++j) {
    double m = 0;
    for (int i = 0; i < n; ++i) m = fmax(m, h[6 * i + j]);
    printf("%-12s max rel err %.3e (2^%.1f)\n", names[j], m, m > 0 ? log2(m) : -999.0);
  }
  return 0;
}
