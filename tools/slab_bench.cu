// slab_bench: DRAM read efficiency of column-slab access (the resident kernel's
// phase 1 pattern) vs. segment width.  Each CTA (512 threads, one per SM x
// waves) reads column slabs [c0, c0 + C) x all 512 rows of 512 x 4608 fp32
// matrices, two arrays (g, e), 8 rows per thread in flight; C = 4 * CQ.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/slab_bench tools/slab_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <vector>

constexpr int N = 512, M = 4096, NMAT = 6;

template <int CQL>
__global__ void __launch_bounds__(512, 1) slabs(const float* __restrict__ g, const float* __restrict__ e,
                                                 float* __restrict__ out, int nslab_per_mat, int total) {
  constexpr int CQ = 1 << CQL, RG = 512 >> CQL, C = 4 * CQ;
  const int t = threadIdx.x, cq = t & (CQ - 1), rg = t >> CQL;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s = blockIdx.x; s < total; s += gridDim.x) {
    const int mat = s / nslab_per_mat, c0 = (s % nslab_per_mat) * C;
    const long long base = (long long)mat * N * M + c0 + 4 * cq;
    for (int j0 = 0; j0 < N / RG; j0 += 8) {
      float4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int row = rg + RG * (j0 + u);
        if (j0 + u < N / RG) {
          a[u] = __ldcs(reinterpret_cast<const float4*>(g + base + (long long)row * M));
          b[u] = __ldcs(reinterpret_cast<const float4*>(e + base + (long long)row * M));
        } else {
          a[u] = b[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x += a[u].x + b[u].x;
        acc.y += a[u].y + b[u].y;
        acc.z += a[u].z + b[u].z;
        acc.w += a[u].w + b[u].w;
      }
    }
  }
  out[blockIdx.x * 512 + t] = acc.x + acc.y + acc.z + acc.w;
}

// contiguous reference: each CTA streams whole rows
__global__ void __launch_bounds__(512, 1) rows(const float* __restrict__ g, const float* __restrict__ e,
                                                float* __restrict__ out, long long n4) {
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* e4 = reinterpret_cast<const float4*>(e);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const long long stride = (long long)gridDim.x * 512;
  for (long long i0 = (long long)blockIdx.x * 512 + threadIdx.x; i0 < n4; i0 += 8 * stride) {
    float4 a[8], b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long i = i0 + u * stride;
      a[u] = i < n4 ? __ldcs(g4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      b[u] = i < n4 ? __ldcs(e4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc.x += a[u].x + b[u].x;
      acc.y += a[u].y + b[u].y;
      acc.z += a[u].z + b[u].z;
      acc.w += a[u].w + b[u].w;
    }
  }
  out[blockIdx.x * 512 + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

__global__ void readflush(const float4* __restrict__ p, long long n4, float* out) {
  float acc = 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    acc += p[i].x;
  if (acc == 12345.f) out[0] = acc;
}
int g_mode = 1;  // 0 none, 1 write flush, 2 write + read (clean L2)
float* g_rf = nullptr;
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar)) : "memory");
}
// 2-D TMA: the resident kernel's slot = box of C cols x RG rows (8 KB) of g and of e
template <int CQL>
__global__ void __launch_bounds__(544, 1) tma_slabs(const __grid_constant__ CUtensorMap mg, const __grid_constant__ CUtensorMap me,
                                                    float* __restrict__ out, int nslab_per_mat, int total, int stages) {
  constexpr int CQ = 1 << CQL, RG = 512 >> CQL, C = 4 * CQ, NS = N / RG;
  extern __shared__ __align__(128) unsigned char sm[];
  float4* buf = reinterpret_cast<float4*>(sm);  // stages x 2 x 512 float4
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * 2 * 8192);
  uint64_t* empty = full + stages;
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 16); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 16) {
    if ((t & 31) == 0) {
      int k = 0;
      for (int s = blockIdx.x; s < total; s += gridDim.x) {
        const int mat = s / nslab_per_mat, c0 = (s % nslab_per_mat) * C;
        for (int j = 0; j < NS; ++j, ++k) {
          const int st = k % stages; const uint32_t ph = (k / stages) & 1;
          mbar_wait(&empty[st], ph ^ 1);
          mbar_expect_tx(&full[st], 16384);
          tma_2d(buf + (size_t)st * 1024, &mg, c0, mat * N + j * RG, &full[st]);
          tma_2d(buf + (size_t)st * 1024 + 512, &me, c0, mat * N + j * RG, &full[st]);
        }
      }
    }
    return;
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int k = 0;
  for (int s = blockIdx.x; s < total; s += gridDim.x)
    for (int j = 0; j < NS; ++j, ++k) {
      const int st = k % stages; const uint32_t ph = (k / stages) & 1;
      mbar_wait(&full[st], ph);
      const float4 a = buf[(size_t)st * 1024 + t], b = buf[(size_t)st * 1024 + 512 + t];
      __syncwarp();
      if ((t & 31) == 0) mbar_arrive(&empty[st]);
      acc.x += a.x + b.x; acc.y += a.y + b.y; acc.z += a.z + b.z; acc.w += a.w + b.w;
    }
  out[blockIdx.x * 512 + t] = acc.x + acc.y + acc.z + acc.w;
}

template <class F>
float timeit(F f, float* flush, size_t fl) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> ts;
  for (int it = 0; it < 12; ++it) {
    if (g_mode >= 1) cudaMemsetAsync(flush, it, fl);
    if (g_mode == 2) readflush<<<148 * 4, 512>>>(reinterpret_cast<const float4*>(g_rf), (long long)(fl / 16), flush);
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it >= 2) ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main() {
  const size_t elems = (size_t)NMAT * N * M, bytes = 2 * elems * 4;
  float *g, *e, *out, *flush;
  cudaMalloc(&g, elems * 4);
  cudaMalloc(&e, elems * 4);
  cudaMalloc(&out, 148 * 4 * 512 * 4);
  const size_t fl = 256 << 20;
  cudaMalloc(&flush, fl);
  cudaMemset(g, 0, elems * 4);
  cudaMemset(e, 0, elems * 4);
  cudaMalloc(&g_rf, fl);
  cudaMemset(g_rf, 0, fl);
  for (int mode = 0; mode < 3; ++mode) {
    g_mode = mode;
    float ms = timeit([&] { rows<<<148, 512>>>(g, e, out, (long long)elems / 4); }, flush, fl);
    printf("rows, flush mode %d (0 none, 1 write, 2 write+read): %7.2f us  %7.1f GB/s\n", mode, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  }
  g_mode = 2;
  for (int grid : {148, 296}) {
    float ms = timeit([&] { rows<<<grid, 512>>>(g, e, out, (long long)elems / 4); }, flush, fl);
    printf("rows (contiguous)     grid %3d: %7.2f us  %7.1f GB/s\n", grid, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  }
#define RUN(CQL)                                                                                              \
  {                                                                                                           \
    const int C = 4 << CQL, nsl = M / C;                                                                     \
    float ms = timeit([&] { slabs<CQL><<<148, 512>>>(g, e, out, nsl, nsl * NMAT); }, flush, fl);             \
    printf("slab C=%4d (%4d B)    grid 148: %7.2f us  %7.1f GB/s\n", C, C * 4, ms * 1e3, bytes / (ms * 1e-3) / 1e9); \
  }
  RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9)
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
#define TRUN(CQL, ST)                                                                                              \
  {                                                                                                                \
    const int C = 4 << CQL, RG = 512 >> CQL, nsl = M / C;                                                         \
    CUtensorMap mg, me;                                                                                            \
    cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)N * NMAT};                                                    \
    cuuint64_t strides[1] = {(cuuint64_t)M * 4};                                                                   \
    cuuint32_t box[2] = {(cuuint32_t)C, (cuuint32_t)RG};                                                           \
    cuuint32_t es[2] = {1, 1};                                                                                     \
    encode(&mg, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,       \
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);       \
    encode(&me, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, e, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,       \
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);       \
    const int smem = ST * 16384 + 2 * ST * 8;                                                                      \
    cudaFuncSetAttribute(tma_slabs<CQL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                      \
    float ms = timeit([&] { tma_slabs<CQL><<<148, 544, smem>>>(mg, me, out, nsl, nsl * NMAT, ST); }, flush, fl);   \
    printf("TMA2D C=%4d (%4d B rows) stages %d (%3d KB): %7.2f us  %7.1f GB/s  %s\n", C, C * 4, ST, ST * 16, ms * 1e3, \
           bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));                                   \
  }
  TRUN(3, 4) TRUN(4, 4) TRUN(5, 4) TRUN(3, 8) TRUN(4, 8) TRUN(5, 8) TRUN(4, 12) TRUN(5, 12)
  return 0;
}
