#include "../paper_1905_13727_b200/csrc/psgd_b200.cu"
__global__ void parts(long long* cyc, double* sink) {
  __shared__ double x[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) x[i] = 1.0 + i * 1e-3;
  __syncwarp();
  WarpReducer wr;
  double acc = 0;
  long long t0 = clock64();
  acc += col_dot(x, x + 512, 512, 1, lane, 32);
  long long t1 = clock64();
  acc += wr.sum(acc);
  long long t2 = clock64();
  col_axpy(x + 512, acc * 1e-9, x, 512, 1, lane, 32);
  __syncwarp();
  long long t3 = clock64();
  double s = sqrt(acc + 2.0);
  long long t4 = clock64();
  double inv = 1.0 / (s + 1.0);
  long long t5 = clock64();
  col_scale(x, inv, 512, 1, lane, 32);
  __syncwarp();
  long long t6 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
  sink[lane] = x[lane] + s + inv;
}
int main() {
  long long* c; double* s; cudaMalloc(&c, 64); cudaMalloc(&s, 4096);
  for (int k = 0; k < 3; ++k) parts<<<1, 32>>>(c, s);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("col_dot %lld  warp_sum %lld  axpy %lld  sqrt %lld  div %lld  scale %lld cycles\n", h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
