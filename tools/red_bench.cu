// red_bench: L2 reduction throughput (RED.ADD) fp32 vs fp64, contended vs spread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_bench tools/red_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
template <class T>
__global__ void red(T* p, int naddr, int per_thread) {
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; ++i) atomicAdd(p + ((gt * 7 + i * 131) % naddr), (T)1);
}
template <class T>
void run(const char* name, int naddr, int per_thread) {
  T* p;
  cudaMalloc(&p, naddr * sizeof(T));
  cudaMemset(p, 0, naddr * sizeof(T));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  red<T><<<148, 512>>>(p, naddr, per_thread);
  cudaEventRecord(a);
  red<T><<<148, 512>>>(p, naddr, per_thread);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double n = 148.0 * 512 * per_thread;
  printf("%s naddr %8d: %8.2f us  %6.2f G red/s\n", name, naddr, ms * 1e3, n / (ms * 1e-3) / 1e9);
  cudaFree(p);
}
int main() {
  for (int na : {1024, 8192, 65536, 1 << 20}) {
    run<float>("f32", na, 8);
    run<double>("f64", na, 8);
  }
  return 0;
}
