// common.cuh — device helpers shared by the kernels of libpsgd_b200.so.
#pragma once
#include <cstdint>
#include "../../include/psgd_b200.h"

namespace psgd {

__device__ __forceinline__ bool finite1(float x) {
  return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// sum over the lane's 16 register rows: four independent FMA chains (the padded
// rows are zero, so every lane runs the same straight-line code)
__device__ __forceinline__ double dot16(const double (&a)[16], const double (&b)[16]) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int k = 0; k < 16; k += 4) {
    s0 = fma(a[k], b[k], s0);
    s1 = fma(a[k + 1], b[k + 1], s1);
    s2 = fma(a[k + 2], b[k + 2], s2);
    s3 = fma(a[k + 3], b[k + 3], s3);
  }
  return (s0 + s1) + (s2 + s3);
}

// ---- register-resident warp MGS for n <= 512, r <= 4 (linalg.py:61-90): lane l
// owns rows l + 32 k (k < 16, zero beyond n); every dot product is 16 FMAs plus
// one shuffle reduction.  Same sequence, threshold and seeded replacement loop
// (linalg.py:82-88, draws from `repl`, column j of attempt a at
// repl[(a * rcols + j) * n]) as mgs_inplace.  One straight-line body for every
// (n, r): the kernel's code stays small enough for the instruction cache (a
// variant per (n, r) made K2 fetch ~1 MB of SASS per launch).
__device__ __forceinline__ void warp_mgs_rt(const float* __restrict__ P, int n, int r, double inv_div,
                                            const double* __restrict__ repl, int rcols, float* __restrict__ out,
                                            int* status) {
  const int lane = threadIdx.x & 31;
  double x[4][16];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int i = lane + 32 * k;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float v = (i < n && j < r) ? __ldcg(P + i * r + j) : 0.f;
      bad |= !finite1(v);
      x[j][k] = (double)v * inv_div;
    }
  }
  if (__any_sync(0xffffffffu, bad)) {  // linalg.py:35-36 (ContractViolation)
    if (lane == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j >= r) break;
    double before = sqrt(warp_sum(dot16(x[j], x[j])));
    double nrm = before;
    for (int attempt = 0;; ++attempt) {  // attempt a > 0: after the a-th replacement draw
      if (attempt > 0 || j > 0) {
#pragma unroll
        for (int i2 = 0; i2 < j; ++i2) {
          const double c = warp_sum(dot16(x[i2], x[j]));
#pragma unroll
          for (int k = 0; k < 16; ++k) x[j][k] -= c * x[i2][k];
        }
        nrm = sqrt(warp_sum(dot16(x[j], x[j])));
      }
      if (!(nrm < 1e-12 * (before + 1.0))) break;  // linalg.py:82-88
      if (attempt == PSGD_REPL_ATTEMPTS) {  // the table holds attempts 0 .. PSGD_REPL_ATTEMPTS - 1
        if (lane == 0) atomicOr(status, PSGD_STATUS_REPLACEMENT);
        break;
      }
      const double* rv = repl + ((long long)attempt * rcols + j) * n;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int i = lane + 32 * k;
        x[j][k] = i < n ? rv[i] : 0.0;
      }
      before = 1.0;
    }
    const double inv = 1.0 / nrm;
#pragma unroll
    for (int k = 0; k < 16; ++k) x[j][k] *= inv;
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int i = lane + 32 * k;
    if (i < n)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < r) out[i * r + j] = (float)x[j][k];
  }
}

// P-hat of one matrix by one warp when n <= 512 and r <= 4; false otherwise
__device__ __forceinline__ bool warp_mgs(const float* P, int n, int r, double inv_div, const double* repl,
                                         int rcols, float* out, int* status) {
  if (n > 512 || r > 4) return false;
  warp_mgs_rt(P, n, r, inv_div, repl, rcols, out, status);
  return true;
}

}  // namespace psgd
