// l2_probe.cu — does a K1-style producer's delta survive in L2 until a K3-style
// consumer reads it?  (B200, sm_100a; run on the GPU box: ./tools/l2_probe)
//
// W: read g, e (evict_first) ; write d = g + e (policy under test)
// R: read d ; write e2 = d - 1, m = d + 1 (streaming stores)
// Before every W, a 256 MiB write flushes L2 (leaves it full of dirty lines, as
// bench.py does).  Reported: W and R times (CUDA events around each launch,
// median of 50), R's implied rate.  Modes:
//   0  plain stores for d
//   1  st.global.L2::cache_hint evict_last for d
//   2  mode 1 + cudaLimitPersistingL2CacheSize = max + stream access-policy
//      window over d (hitProp persisting)
//   3  mode 0 + access-policy window only
//   4  mode 0, R sweeps d in reverse order (most recently written first)
//   5  mode 1, R in reverse order
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ float4 ld_hint(const float4* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(float4* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

__global__ void kW(const float4* g, const float4* e, float4* d, long long n4, int mode) {
  const uint64_t pf = pol_first(), pl = pol_last();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 a = ld_hint(g + i, pf), b = ld_hint(e + i, pf);
    float4 c = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    if (mode == 1 || mode == 2) st_hint(d + i, c, pl); else d[i] = c;
  }
}
__global__ void kR(const float4* d, float4* e2, float4* m, long long n4, int rev) {
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n4; i0 += (long long)gridDim.x * blockDim.x) {
    const long long i = rev ? n4 - 1 - i0 : i0;
    float4 v = d[i];
    __stcs(e2 + i, make_float4(v.x - 1, v.y - 1, v.z - 1, v.w - 1));
    __stcs(m + i, make_float4(v.x + 1, v.y + 1, v.z + 1, v.w + 1));
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 11164352LL;  // ResNet-18 matrix elements
  const long long n4 = n / 4;
  float *g, *e, *d, *e2, *m, *fl;
  const size_t B = n * 4, FL = 256ull << 20;
  CK(cudaMalloc(&g, B)); CK(cudaMalloc(&e, B)); CK(cudaMalloc(&d, B)); CK(cudaMalloc(&e2, B)); CK(cudaMalloc(&m, B));
  CK(cudaMalloc(&fl, FL));
  CK(cudaMemset(g, 0, B)); CK(cudaMemset(e, 0, B));
  int dev = 0, l2 = 0, maxp = 0;
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
  printf("n=%lld (%.1f MB per array)  L2 %d B  max persisting %d B\n", n, B / 1e6, l2, maxp);
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t ev[3];
  for (auto& x : ev) CK(cudaEventCreate(&x));
  const int grid = 148 * 8, blk = 256;
  for (int mode = 0; mode < 6; ++mode) {
    if (mode == 4) {
      CK(cudaCtxResetPersistingL2Cache());
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
      cudaStreamAttrValue av{};
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
    }
    if (mode == 2 || mode == 3) {
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp));
      cudaStreamAttrValue av{};
      av.accessPolicyWindow.base_ptr = d;
      av.accessPolicyWindow.num_bytes = std::min<size_t>(B, (size_t)maxp);
      av.accessPolicyWindow.hitRatio = 1.0f;
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
    }
    std::vector<float> tw, tr;
    for (int it = 0; it < 60; ++it) {
      CK(cudaMemsetAsync(fl, it & 0xff, FL, st));
      if (mode == 2 || mode == 3) CK(cudaCtxResetPersistingL2Cache());
      CK(cudaEventRecord(ev[0], st));
      kW<<<grid, blk, 0, st>>>((const float4*)g, (const float4*)e, (float4*)d, n4, mode == 5 ? 1 : mode);
      CK(cudaEventRecord(ev[1], st));
      kR<<<grid, blk, 0, st>>>((const float4*)d, (float4*)e2, (float4*)m, n4, mode >= 4);
      CK(cudaEventRecord(ev[2], st));
      CK(cudaStreamSynchronize(st));
      float a, b;
      CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
      CK(cudaEventElapsedTime(&b, ev[1], ev[2]));
      if (it >= 10) { tw.push_back(a * 1e3f); tr.push_back(b * 1e3f); }
    }
    std::sort(tw.begin(), tw.end());
    std::sort(tr.begin(), tr.end());
    const float w = tw[tw.size() / 2], r = tr[tr.size() / 2];
    printf("mode %d: W %.2f us (%.0f GB/s)  R %.2f us (%.0f GB/s over 3 arrays)  W+R %.2f us\n", mode, w,
           3 * B / (w * 1e-6) / 1e9, r, 3 * B / (r * 1e-6) / 1e9, w + r);
  }
  return 0;
}
