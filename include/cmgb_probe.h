/*
 * cmgb_probe.h — measurement helpers for bench.py (not part of the reference
 * boundary): sustained FMA throughput used as the compute-roofline
 * denominator (MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).
 */
#ifndef CMGB_PROBE_H_
#define CMGB_PROBE_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* TFLOP/s (2 flops per FMA) of a full-grid FFMA (fp64 = 0) / DFMA (fp64 = 1) chain. */
int cmgb_probe_fma_tflops(int32_t fp64, int32_t iters, double* tflops, void* cuda_stream);
/* Kernel launches this library has issued so far (all devices, all threads;
 * the probe's own launches excluded): bench.py's gpu_launches. */
uint64_t cmgb_kernel_launches(void);
#ifdef __cplusplus
}
#endif
#endif
