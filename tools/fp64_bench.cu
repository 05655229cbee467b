// fp64 vs fp32 FMA throughput / latency on this part (informs the GS design)
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void chain(T* out, int iters, long long* cyc) {
  T a = threadIdx.x * (T)1e-3, b = (T)1.0000001, c = (T)1e-7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = a * b + c; }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
template <typename T>
__global__ void thru(T* out, int iters) {
  T a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const T b = (T)1.0000001, c = (T)1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c;
    a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  double* d; float* f; long long* cyc; long long h;
  cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 26); cudaMalloc(&cyc, 8);
  const int it = 1 << 14;
  chain<double><<<1, 32>>>(d, it, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / it);
  chain<float><<<1, 32>>>(f, it, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", (double)h / it);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); thru<double><<<148 * 8, 256>>>(d, it); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("DFMA throughput: %.2f TFLOP/s\n", 2.0 * 8 * it * 148 * 8 * 256 / ms / 1e9);
    cudaEventRecord(a); thru<float><<<148 * 8, 256>>>(f, it); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("FFMA throughput: %.2f TFLOP/s\n", 2.0 * 8 * it * 148 * 8 * 256 / ms / 1e9);
  }
  return 0;
}
