// Microbenchmark: read-streaming throughput of (a) cp.async.bulk (TMA 1-D) into a
// smem ring with mbarriers, (b) plain LDG.128 loops, on this B200.  Informs the
// K1/K3 pipeline design.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/tma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar)) : "memory");
}

// 2-D tiles: the matrix (rows x cols fp32) is cut into column slabs of bx columns;
// each slab is loaded as ceil(rows/by) boxes of bx x by.
__global__ void tma_tiles(const __grid_constant__ CUtensorMap map, int rows, int cols, int bx, int by, int stages, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int nbox = (rows + by - 1) / by;
  const int sbytes = nbox * by * bx * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * sbytes);
  uint64_t* empty = full + stages;
  const int nslab = cols / bx;
  const int per = (nslab + gridDim.x - 1) / gridDim.x;
  const int cb = blockIdx.x * per, ce = min(nslab, cb + per);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw - 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == nw - 1) {
    if ((threadIdx.x & 31) == 0)
      for (int k = cb; k < ce; ++k) {
        const int s = (k - cb) % stages; const uint32_t ph = ((k - cb) / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], sbytes);
        for (int b = 0; b < nbox; ++b) tma_2d(sm + (size_t)s * sbytes + (size_t)b * by * bx * 4, &map, k * bx, b * by, &full[s]);
      }
    return;
  }
  float acc = 0.f;
  for (int k = cb; k < ce; ++k) {
    const int s = (k - cb) % stages; const uint32_t ph = ((k - cb) / stages) & 1;
    mbar_wait(&full[s], ph);
    acc += reinterpret_cast<const float*>(sm + (size_t)s * sbytes)[threadIdx.x];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void tma_stream_hint(const char* src, long long total, int cbytes, int stages, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * cbytes);
  uint64_t* empty = full + stages;
  const long long nch = total / cbytes;
  const long long per = (nch + gridDim.x - 1) / gridDim.x;
  const long long cb = blockIdx.x * per, ce = min(nch, cb + per);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw - 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == nw - 1) {
    if ((threadIdx.x & 31) == 0)
      for (long long k = cb; k < ce; ++k) {
        const int s = (k - cb) % stages; const uint32_t ph = ((k - cb) / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], cbytes);
        tma_load_hint(sm + (size_t)s * cbytes, src + k * cbytes, cbytes, &full[s]);
      }
    return;
  }
  float acc = 0.f;
  for (long long k = cb; k < ce; ++k) {
    const int s = (k - cb) % stages; const uint32_t ph = ((k - cb) / stages) & 1;
    mbar_wait(&full[s], ph);
    acc += reinterpret_cast<const float*>(sm + (size_t)s * cbytes)[threadIdx.x];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 12345.f) sink[0] = acc;
}

// each CTA streams a contiguous range of `chunks` chunks of `cbytes` bytes
__global__ void tma_stream(const char* src, long long total, int cbytes, int stages, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * cbytes);
  uint64_t* empty = full + stages;
  const long long nch = total / cbytes;
  const long long per = (nch + gridDim.x - 1) / gridDim.x;
  const long long cb = blockIdx.x * per, ce = min(nch, cb + per);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw - 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == nw - 1) {
    if ((threadIdx.x & 31) == 0)
      for (long long k = cb; k < ce; ++k) {
        const int s = (k - cb) % stages; const uint32_t ph = ((k - cb) / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], cbytes);
        tma_load(sm + (size_t)s * cbytes, src + k * cbytes, cbytes, &full[s]);
      }
    return;
  }
  float acc = 0.f;
  for (long long k = cb; k < ce; ++k) {
    const int s = (k - cb) % stages; const uint32_t ph = ((k - cb) / stages) & 1;
    mbar_wait(&full[s], ph);
    acc += reinterpret_cast<const float*>(sm + (size_t)s * cbytes)[threadIdx.x];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void ldg_stream(const float4* src, long long n4, float* sink) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(src + i);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

__global__ void copy_stream(const float4* src, float4* dst, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
}

int main(int argc, char** argv) {
  const long long total = argc > 1 ? atoll(argv[1]) : (1LL << 30);  // bytes read
  char* src; float* sink; char* dst; char* flush;
  cudaMalloc(&src, total); cudaMalloc(&dst, total); cudaMalloc(&sink, 64); cudaMalloc(&flush, 256 << 20);
  cudaMemset(src, 1, total);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto fn) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemsetAsync(flush, it, 256 << 20);
      cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (it > 0 && ms < best) best = ms;
    }
    return best;
  };
  printf("SMs %d\n", nsm);
  for (int tb : {256, 512}) for (int occ : {4, 8}) {
    float ms = timeit([&] { ldg_stream<<<nsm * occ, tb>>>((const float4*)src, total / 16, sink); });
    printf("LDG.128 read  tb=%d ctas/sm=%d : %.1f GB/s\n", tb, occ, total / ms / 1e6);
  }
  {
    float ms = timeit([&] { copy_stream<<<nsm * 8, 256>>>((const float4*)src, (float4*)dst, total / 16); });
    printf("LDG/STG copy (r+w)          : %.1f GB/s\n", 2.0 * total / ms / 1e6);
  }
  for (int cb : {16384, 36864, 49152}) for (int st : {2, 3, 4, 6}) for (int ctas : {1, 2}) {
    size_t smem = (size_t)st * cb + 2 * st * 8;
    if (smem * ctas > 220 * 1024) continue;
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float ms = timeit([&] { tma_stream<<<nsm * ctas, 256, smem>>>(src, total, cb, st, sink); });
    cudaError_t e = cudaGetLastError();
    printf("TMA bulk chunk=%6d stages=%d ctas/sm=%d (in flight %4zu KB/SM): %.1f GB/s %s\n", cb, st, ctas,
           (size_t)st * cb * ctas / 1024, total / ms / 1e6, e ? cudaGetErrorString(e) : "");
  }
  for (int cb : {16384, 36864}) for (int st : {3, 4}) {
    size_t smem = (size_t)st * cb + 2 * st * 8;
    if (smem > 220 * 1024) continue;
    cudaFuncSetAttribute(tma_stream_hint, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float ms = timeit([&] { tma_stream_hint<<<nsm, 256, smem>>>(src, total, cb, st, sink); });
    printf("TMA bulk+evict_first chunk=%6d stages=%d: %.1f GB/s\n", cb, st, total / ms / 1e6);
  }
  // 2-D tiles out of a (rows x 4608) fp32 matrix
  void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int cols = 4608;
  const int rows = (int)(total / 4 / cols) / 512 * 512;
  for (int bx : {32, 64, 128}) for (int by : {64, 128, 256}) for (int st : {2, 3}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)512};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
    cuuint32_t es[2] = {1, 1};
    // treat the buffer as many stacked 512 x 4608 matrices: use one map per 512-row block via y offset
    dims[1] = rows;
    CUresult cr = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int srows = 512;
    const size_t sbytes = (size_t)((srows + by - 1) / by) * by * bx * 4;
    size_t smem = st * sbytes + 2 * st * 8;
    if (smem > 220 * 1024 || cr) { printf("skip bx=%d by=%d st=%d (%d)\n", bx, by, st, (int)cr); continue; }
    cudaFuncSetAttribute(tma_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // only the first 512 rows x all columns: 9.4 MB -> repeat via many CTAs? keep simple: one slab set
    float ms = timeit([&] { tma_tiles<<<nsm, 256, smem>>>(map, srows, cols, bx, by, st, sink); });
    printf("TMA 2D box %3dx%3d stages=%d (slab %zu KB): %.1f GB/s over %.1f MB\n", bx, by, st, sbytes / 1024,
           (double)srows * cols * 4 / ms / 1e6, srows * cols * 4 / 1e6);
  }
  return 0;
}
