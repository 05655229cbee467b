// common.cuh — device helpers shared by the translation units of libpsgd_b200.so.
#pragma once
#include <cstdint>
#include "../../include/psgd_b200.h"

namespace psgd {

__device__ __forceinline__ bool finite1(float x) {
  return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}

// ---- register-resident warp MGS (n <= 32 * RPL, r == R <= 4): each lane
// owns rows lane + 32 k; dot products are RPL fused multiply-adds plus one
// shuffle reduction, so the whole orthogonalisation of a 512 x 2 P is ~1 us.
// Same sequence, threshold and replacement rule as mgs_inplace (linalg.py:61-90).
template <int RPL, int R, class T = float>
__device__ __forceinline__ void warp_mgs_reg(const T* __restrict__ P, int n, double inv_div,
                                             const double* __restrict__ repl, int rcols, float* __restrict__ out,
                                             int* status) {
  const int lane = threadIdx.x & 31;
  double x[R][RPL];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int i = lane + 32 * k;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const T v = i < n ? __ldcg(P + i * R + j) : T(0);
      bad |= !isfinite(v);
      x[j][k] = (double)v * inv_div;
    }
  }
  if (__any_sync(0xffffffffu, bad)) {  // linalg.py:35-36 (ContractViolation)
    if (lane == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
    return;
  }
  auto wsum = [](double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  };
#pragma unroll
  for (int j = 0; j < R; ++j) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < RPL; ++k) s = fma(x[j][k], x[j][k], s);
    double before = sqrt(wsum(s));
    double nrm = before;
    for (int attempt = 0;; ++attempt) {  // attempt a > 0: after the a-th replacement draw
      if (attempt > 0 || j > 0) {
#pragma unroll
        for (int i2 = 0; i2 < j; ++i2) {
          double d = 0.0;
#pragma unroll
          for (int k = 0; k < RPL; ++k) d = fma(x[i2][k], x[j][k], d);
          const double c = wsum(d);
#pragma unroll
          for (int k = 0; k < RPL; ++k) x[j][k] -= c * x[i2][k];
        }
        s = 0.0;
#pragma unroll
        for (int k = 0; k < RPL; ++k) s = fma(x[j][k], x[j][k], s);
        nrm = sqrt(wsum(s));
      }
      if (!(nrm < 1e-12 * (before + 1.0))) break;  // linalg.py:82-88
      if (attempt == PSGD_REPL_ATTEMPTS) {  // the table holds attempts 0 .. PSGD_REPL_ATTEMPTS - 1
        if (lane == 0) atomicOr(status, PSGD_STATUS_REPLACEMENT);
        break;
      }
      const double* rv = repl + ((long long)attempt * rcols + j) * n;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int i = lane + 32 * k;
        x[j][k] = i < n ? rv[i] : 0.0;
      }
      before = 1.0;
    }
    const double inv = 1.0 / nrm;
#pragma unroll
    for (int k = 0; k < RPL; ++k) x[j][k] *= inv;
  }
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int i = lane + 32 * k;
    if (i < n)
#pragma unroll
      for (int j = 0; j < R; ++j) out[i * R + j] = (float)x[j][k];
  }
}

template <int R, class T = float>
__device__ __forceinline__ bool warp_mgs_dispatch_r(int rpl_log2, const T* P, int n, double inv_div,
                                                    const double* repl, int rcols, float* out, int* status) {
  switch (rpl_log2) {
    case 0: warp_mgs_reg<1, R, T>(P, n, inv_div, repl, rcols, out, status); return true;
    case 1: warp_mgs_reg<2, R, T>(P, n, inv_div, repl, rcols, out, status); return true;
    case 2: warp_mgs_reg<4, R, T>(P, n, inv_div, repl, rcols, out, status); return true;
    case 3: warp_mgs_reg<8, R, T>(P, n, inv_div, repl, rcols, out, status); return true;
    case 4: warp_mgs_reg<16, R, T>(P, n, inv_div, repl, rcols, out, status); return true;
    default: return false;
  }
}

// P-hat of one matrix by one warp when n <= 512 and r <= 4; false otherwise
__device__ __forceinline__ bool warp_mgs(const float* P, int n, int r, double inv_div, const double* repl,
                                         int rcols, float* out, int* status) {
  if (n > 512 || r > 4) return false;
  int l = 0;
  while ((32 << l) < n) ++l;
  switch (r) {
    case 1: return warp_mgs_dispatch_r<1>(l, P, n, inv_div, repl, rcols, out, status);
    case 2: return warp_mgs_dispatch_r<2>(l, P, n, inv_div, repl, rcols, out, status);
    case 3: return warp_mgs_dispatch_r<3>(l, P, n, inv_div, repl, rcols, out, status);
    default: return warp_mgs_dispatch_r<4>(l, P, n, inv_div, repl, rcols, out, status);
  }
}


}  // namespace psgd
