// l2_probe2.cu — is delta still in L2 when the next kernel reads it?  And what
// does a plain read of ~45-90 MB reach from a cold (dirty-flushed) L2?
// (B200, sm_100a; run on the GPU box: ./tools/l2_probe2)
//
// F : 256 MiB memset (L2 full of dirty lines, as bench.py's flush)
// W : read g, e (evict_first) ; write d = g + e with store policy P
// Rd: read d only (sum -> tiny output), forward or reverse order
// Cases (median of 40, CUDA events around Rd):
//   cold      F, Rd              (d not in L2)
//   after-W   F, W, Rd           (d just written by W)
// Store policy P: 0 plain, 1 evict_last, 2 evict_normal; reverse: Rd newest first.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_normal() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ float4 ld_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

__global__ void kW(const float4* g, const float4* e, float4* d, long long n4, int pol) {
  const uint64_t pf = pol_first(), pl = pol == 1 ? pol_last() : pol_normal();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 a = ld_hint(g + i, pf), b = ld_hint(e + i, pf);
    float4 c = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    if (pol == 0) d[i] = c; else st_hint(d + i, c, pl);
  }
}
// 4 independent float4 loads per thread per iteration
__global__ void kRd(const float4* d, float* out, long long n4, int rev) {
  float s = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i0 + 3 * stride < n4; i0 += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      v[u] = __ldcs(d + (rev ? n4 - 1 - i : i));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i0 < n4; i0 += stride) {
    const float4 v = __ldcs(d + (rev ? n4 - 1 - i0 : i0));
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 12345.f) out[0] = s;
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 11164352LL;  // ResNet-18 matrix elements
  const long long n4 = n / 4;
  float *g, *e, *d, *fl, *out;
  const size_t B = n * 4, FL = 256ull << 20;
  CK(cudaMalloc(&g, B)); CK(cudaMalloc(&e, B)); CK(cudaMalloc(&d, 2 * B));
  CK(cudaMalloc(&fl, FL)); CK(cudaMalloc(&out, 64));
  CK(cudaMemset(g, 0, B)); CK(cudaMemset(e, 0, B)); CK(cudaMemset(d, 0, 2 * B));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t ev[2];
  for (auto& x : ev) CK(cudaEventCreate(&x));
  const int gridW = 148 * 8, blk = 256;
  printf("n=%lld (%.1f MB per array)\n", n, B / 1e6);
  for (int grid_mult : {4, 8, 16}) {
    for (int rd2 : {0, 1}) {  // rd2: Rd reads 2B (90 MB) of cold data instead of B
      std::vector<float> t;
      for (int it = 0; it < 50; ++it) {
        CK(cudaMemsetAsync(fl, it & 0xff, FL, st));
        CK(cudaEventRecord(ev[0], st));
        kRd<<<148 * grid_mult, blk, 0, st>>>((const float4*)d, out, rd2 ? 2 * n4 : n4, 0);
        CK(cudaEventRecord(ev[1], st));
        CK(cudaStreamSynchronize(st));
        float a;
        CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
        if (it >= 10) t.push_back(a * 1e3f);
      }
      std::sort(t.begin(), t.end());
      const double bytes = (rd2 ? 2.0 : 1.0) * B;
      printf("cold read %.1f MB, %d CTAs/SM: %.2f us (%.0f GB/s)\n", bytes / 1e6, grid_mult, t[t.size() / 2],
             bytes / (t[t.size() / 2] * 1e-6) / 1e9);
    }
  }
  for (int pol = 0; pol < 3; ++pol)
    for (int rev = 0; rev < 2; ++rev) {
      std::vector<float> t;
      for (int it = 0; it < 50; ++it) {
        CK(cudaMemsetAsync(fl, it & 0xff, FL, st));
        kW<<<gridW, blk, 0, st>>>((const float4*)g, (const float4*)e, (float4*)d, n4, pol);
        CK(cudaEventRecord(ev[0], st));
        kRd<<<148 * 8, blk, 0, st>>>((const float4*)d, out, n4, rev);
        CK(cudaEventRecord(ev[1], st));
        CK(cudaStreamSynchronize(st));
        float a;
        CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
        if (it >= 10) t.push_back(a * 1e3f);
      }
      std::sort(t.begin(), t.end());
      printf("after-W  store policy %d  %s: Rd %.2f us (%.0f GB/s)\n", pol, rev ? "reverse" : "forward",
             t[t.size() / 2], B / (t[t.size() / 2] * 1e-6) / 1e9);
    }
  return 0;
}
