// SE(3) / SO(3) helpers of the demo integrator (src/pose.cpp), FP64 with the
// reference's branches: so3_exp (pose.hpp:54-61, exp_coeffs 25-47), so3_log
// (pose.cpp:10-33: clamp, small-angle and near-pi branches), se3_log (35-50).
// Matrices row-major double[9].
#pragma once

#include "dmath.cuh"

namespace cmgb {

// A = sin(t)/t, B = (1-cos(t))/t^2 with the series below t^2 = 1e-8.
__device__ __forceinline__ void exp_ab(double th2, double& a, double& b) {
  if (th2 < 1e-8) {
    a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
  } else {
    const double th = sqrt(th2);
    double s, c;
    sincos(th, &s, &c);
    a = s / th;
    b = (1.0 - c) / th2;
  }
}

__device__ __forceinline__ void skew(const double* w, double* W) {
  W[0] = 0.0;   W[1] = -w[2]; W[2] = w[1];
  W[3] = w[2];  W[4] = 0.0;   W[5] = -w[0];
  W[6] = -w[1]; W[7] = w[0];  W[8] = 0.0;
}

__device__ __forceinline__ void matmul3(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}

// so3_exp: R = I + [w]x a + [w]x^2 b
__device__ __forceinline__ void so3_exp_dev(const double* w, double* R) {
  const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  double a, b;
  exp_ab(th2, a, b);
  double W[9], W2[9];
  skew(w, W);
  matmul3(W, W, W2);
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = ((i % 4 == 0) ? 1.0 : 0.0) + W[i] * a + W2[i] * b;
}

// so3_log (pose.cpp:10-33)
__device__ __forceinline__ void so3_log_dev(const double* r, double* w) {
  const double trace = r[0] + r[4] + r[8];
  const double cos_theta = fmin(fmax(0.5 * (trace - 1.0), -1.0), 1.0);
  const double theta = acos(cos_theta);
  const double vee[3] = {r[7] - r[5], r[2] - r[6], r[3] - r[1]};
  if (theta < 1e-8) {
    w[0] = vee[0] * 0.5; w[1] = vee[1] * 0.5; w[2] = vee[2] * 0.5;
    return;
  }
  if (theta > 3.14159265358979323846 - 1e-6) {
    double s[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) s[i] = r[i];
    s[0] += 1.0; s[4] += 1.0; s[8] += 1.0;
    int k = 0;
    if (s[4] > s[4 * k]) k = 1;
    if (s[8] > s[4 * k]) k = 2;
    const double ax[3] = {s[k], s[3 + k], s[6 + k]};
    const double nrm = sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    w[0] = ax[0] / nrm * theta; w[1] = ax[1] / nrm * theta; w[2] = ax[2] / nrm * theta;
    return;
  }
  const double f = 0.5 * theta / sin(theta);
  w[0] = vee[0] * f; w[1] = vee[1] * f; w[2] = vee[2] * f;
}

// se3_log (pose.cpp:35-50): pose = [V^-1 t; w]
__device__ __forceinline__ void se3_log_dev(const double* R, const double* t, double* pose) {
  double w[3];
  so3_log_dev(R, w);
  const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
  double W[9], W2[9];
  skew(w, W);
  matmul3(W, W, W2);
  double coeff;
  if (th2 < 1e-8) {
    coeff = 1.0 / 12.0;
  } else {
    const double th = sqrt(th2);
    const double half = 0.5 * th;
    coeff = (1.0 - half * cos(half) / sin(half)) / th2;
  }
  double Vi[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) Vi[i] = ((i % 4 == 0) ? 1.0 : 0.0) + W[i] * -0.5 + W2[i] * coeff;
#pragma unroll
  for (int i = 0; i < 3; ++i) pose[i] = Vi[3 * i] * t[0] + Vi[3 * i + 1] * t[1] + Vi[3 * i + 2] * t[2];
  pose[3] = w[0]; pose[4] = w[1]; pose[5] = w[2];
}

}  // namespace cmgb
