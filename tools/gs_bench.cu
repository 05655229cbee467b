// Cycle breakdown of the warp-level MGS (K2 small-matrix path) on this part.
#include "../paper_1905_13727_b200/csrc/psgd_b200.cu"

__global__ void gs_bench(const float* P, int n, int r, const double* repl, long long* cyc, float* out, int* status) {
  extern __shared__ double xs[];
  const int lane = threadIdx.x;
  long long t0 = clock64();
  for (int idx = lane; idx < n * r; idx += 32) {
    const int i = idx / r, j = idx - i * r;
    xs[j * n + i] = (double)P[idx];
  }
  __syncwarp();
  long long t1 = clock64();
  mgs_inplace(xs, n, r, repl, lane, 32, WarpReducer{}, status, 1, n);
  __syncwarp();
  long long t2 = clock64();
  for (int idx = lane; idx < n * r; idx += 32) {
    const int i = idx / r, j = idx - i * r;
    out[idx] = (float)xs[j * n + i];
  }
  long long t3 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}

__global__ void red_bench(long long* cyc) {
  double v = threadIdx.x;
  WarpReducer wr;
  long long t0 = clock64();
  for (int k = 0; k < 100; ++k) v = wr.sum(v) * 1e-3;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / 100;
  if (v == 12345.0) cyc[4] = 1;
}

int main() {
  for (int r : {2, 4}) {
    const int n = 512;
    float* P; double* repl; long long* cyc; float* out; int* st;
    cudaMalloc(&P, n * r * 4); cudaMalloc(&repl, n * r * 8); cudaMalloc(&cyc, 64); cudaMalloc(&out, n * r * 4);
    cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
    std::vector<float> h(n * r);
    for (int i = 0; i < n * r; ++i) h[i] = (float)((i * 7919) % 1000) / 1000.f - 0.5f;
    cudaMemcpy(P, h.data(), n * r * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) gs_bench<<<1, 32, n * r * 8>>>(P, n, r, repl, cyc, out, st);
    red_bench<<<1, 32>>>(cyc);
    long long c[4];
    cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
    printf("n=%d r=%d: load %lld  mgs %lld  store %lld cycles; warp fp64 reduction %lld cycles\n", n, r, c[0], c[1], c[2], c[3]);
  }
  return 0;
}
