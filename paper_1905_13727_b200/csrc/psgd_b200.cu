// psgd_b200.cu — B200 (sm_100a) kernels + C ABI for the PowerSGD compression hot path.
//
// Reference semantics: /root/reference/pkg/src/gradcomp
//   optimizer.py:98-129   EF add, per-matrix round trip, EF update, bias all-reduce
//   compressors.py:327-379 low_rank_iteration + PowerSGD.round_trip
//   linalg.py:54-90       modified Gram-Schmidt with seeded degenerate replacement
//   comm.py:51-98         tree-ordered all-reduce mean
//
// Design: every kernel is HBM-bound at small rank, so the work
// is organised around streaming each gradient element through the SM the
// minimum number of times:
//   K1 k1_ef_p      warp-per-row items: delta = g + e (one read of g and e, one
//                   write of delta), P = delta Q reduced in-warp (no atomics).
//   K2 k2_gs        one CTA per matrix, float64 MGS over the tiny P.
//   K3 k3_q_ef      one CTA per column slab holding ALL rows of the slab in
//                   registers: q_w = delta^T P-hat reduced in smem, then
//                   e = delta - P-hat q_w^T (and M-hat at W=1) written from the
//                   same registers — delta is read exactly once.  Tall matrices
//                   (n > 512) split rows into chunks, reduce chunk partials in
//                   fixed order by the last-arriving CTA, and take K4.
//   K4 k4_ef        row items: e = delta - P-hat q^T (+ M-hat at W=1), tall only.
//   K5 k5_decomp    row items: M-hat = P-hat (q_sum / W)^T, Q store (W > 1).
// All reductions are fixed-order, so results are bitwise run-to-run stable.

#include "../../include/psgd_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr int kThreads = 256;            // every kernel: 8 warps
constexpr int kRowItemElems = 4096;      // target elements per K1/K4/K5 warp item
constexpr int kGsThreads = 512;

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define PSGD_CUDA_CHECK(expr)                                                        \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(PSGD_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

struct MatDev {
  long long flat_off, p_off, q_off, repl_off;
  int n, m, r, tall;
};

// K1 / K4 / K5 work item: `nrows` rows of matrix `mat` starting at `row0`,
// processed by one warp with 2^lg lanes per row.  mat < 0: bias chunk
// [row0, row0 + nrows) of the bias vector (K1 only).
struct RowItem {
  int mat, row0, nrows, lg;
};

// K3 work item: rows [chunk * rows_per_chunk, ...) x columns [c0, c0 + C) of `mat`,
// C = vec << cq_log2.  nchunks > 1: tall matrix, partial written at ws_off.
struct SlabItem {
  long long ws_off;
  int mat, c0, chunk, nchunks, slab, vec, cq_log2, pad;
};

struct Group {       // a contiguous run of items sharing r_eff
  int r, beg, end;
  int smem;          // K3 only: dynamic shared memory bytes
};

__host__ __device__ constexpr int k3_dcap(int r) { return r <= 4 ? 64 : 32; }

// ----------------------------------------------------------------------------- helpers

__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }

__device__ __forceinline__ bool finite1(float x) {
  return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u;
}
__device__ __forceinline__ bool finite4(float4 v) {
  return finite1(v.x) & finite1(v.y) & finite1(v.z) & finite1(v.w);
}

// Q rows j0..j0+3 (4*r consecutive floats starting at q) -> qv[4][R].
template <int R, bool EXACT>
__device__ __forceinline__ void load_q4(const float* __restrict__ q, bool aligned, int r,
                                        float (&qv)[4][R]) {
  if (EXACT && aligned) {
#pragma unroll
    for (int t = 0; t < R; ++t) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(q) + t);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) qv[(4 * t + u) / R][(4 * t + u) % R] = vv[u];
    }
  } else {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
      for (int k = 0; k < R; ++k)
        qv[jj][k] = (EXACT || k < r) ? __ldg(q + jj * r + k) : 0.f;
  }
}

// ============================================================================= K1
// delta = g + e ; P[i,:] = sum_j delta[i,j] Q[j,:]   (optimizer.py:120, compressors.py:336)

template <int R, bool EXACT>
__device__ __forceinline__ void k1_rows(const MatDev& md, const RowItem& it, int lane,
                                        const float* __restrict__ g, const float* __restrict__ e,
                                        float* __restrict__ work, const float* __restrict__ Qall,
                                        float* __restrict__ Pall, bool& bad) {
  const int r = EXACT ? R : md.r;
  const int m = md.m;
  const int lg = it.lg;
  const int G = 1 << lg;
  const int gl = lane & (G - 1);
  const int sub = lane >> lg;
  const int rpp = 32 >> lg;
  const float* __restrict__ Q = Qall + md.q_off;
  for (int rb = 0; rb < it.nrows; rb += rpp) {
    const int li = rb + sub;
    const bool active = li < it.nrows;
    const int i = it.row0 + li;
    float acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.f;
    if (active) {
      const long long o = md.flat_off + (long long)i * m;
      const int head = min((int)((4 - (o & 3)) & 3), m);
      const int body4 = (m - head) >> 2;
      const int tail = m - head - 4 * body4;
      // scalar head / tail (rows whose start is not 16-B aligned, e.g. m = 27, 650)
      for (int s = gl; s < head + tail; s += G) {
        const int j = s < head ? s : head + 4 * body4 + (s - head);
        const float gv = ld_stream(g + o + j);
        const float d = e ? gv + ld_stream(e + o + j) : gv;
        bad |= !finite1(gv);
        work[o + j] = d;
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (EXACT || k < r) acc[k] = fmaf(d, __ldg(Q + (long long)j * r + k), acc[k]);
      }
      const float4* __restrict__ g4 = reinterpret_cast<const float4*>(g + o + head);
      const float4* __restrict__ e4 = e ? reinterpret_cast<const float4*>(e + o + head) : nullptr;
      float4* __restrict__ w4 = reinterpret_cast<float4*>(work + o + head);
      const float* __restrict__ qrow = Q + (long long)head * r;
      const bool qal = ((head * r) & 3) == 0;
      int c = gl;
      // 4 independent 16-B loads of g and of e in flight per lane
      for (; c + 3 * G < body4; c += 4 * G) {
        float4 gv[4], ev[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) gv[u] = ld_stream(g4 + c + u * G);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          ev[u] = e4 ? ld_stream(e4 + c + u * G) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4 d = make_float4(gv[u].x + ev[u].x, gv[u].y + ev[u].y, gv[u].z + ev[u].z,
                                       gv[u].w + ev[u].w);
          bad |= !finite4(gv[u]);
          w4[c + u * G] = d;
          float qv[4][R];
          load_q4<R, EXACT>(qrow + (long long)(4 * (c + u * G)) * r, qal, r, qv);
#pragma unroll
          for (int k = 0; k < R; ++k) {
            acc[k] = fmaf(d.x, qv[0][k], acc[k]);
            acc[k] = fmaf(d.y, qv[1][k], acc[k]);
            acc[k] = fmaf(d.z, qv[2][k], acc[k]);
            acc[k] = fmaf(d.w, qv[3][k], acc[k]);
          }
        }
      }
      for (; c < body4; c += G) {
        const float4 gv = ld_stream(g4 + c);
        const float4 ev = e4 ? ld_stream(e4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 d = make_float4(gv.x + ev.x, gv.y + ev.y, gv.z + ev.z, gv.w + ev.w);
        bad |= !finite4(gv);
        w4[c] = d;
        float qv[4][R];
        load_q4<R, EXACT>(qrow + (long long)(4 * c) * r, qal, r, qv);
#pragma unroll
        for (int k = 0; k < R; ++k) {
          acc[k] = fmaf(d.x, qv[0][k], acc[k]);
          acc[k] = fmaf(d.y, qv[1][k], acc[k]);
          acc[k] = fmaf(d.z, qv[2][k], acc[k]);
          acc[k] = fmaf(d.w, qv[3][k], acc[k]);
        }
      }
    }
    // fixed-order butterfly inside the 2^lg-lane group
    for (int off = G >> 1; off > 0; off >>= 1)
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
    if (active && gl == 0) {
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (EXACT || k < r) Pall[md.p_off + (long long)i * r + k] = acc[k];
    }
  }
}

template <int R, bool EXACT>
__global__ void __launch_bounds__(kThreads) k1_ef_p(const MatDev* __restrict__ mats,
                                                    const RowItem* __restrict__ items, int beg,
                                                    int end, const float* __restrict__ g,
                                                    const float* __restrict__ e,
                                                    float* __restrict__ work,
                                                    const float* __restrict__ Q,
                                                    float* __restrict__ P,
                                                    const float* __restrict__ bias_g,
                                                    long long bias_off, int* status) {
  const int lane = threadIdx.x & 31;
  const int wi = beg + blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  bool bad = false;
  if (wi < end) {
    const RowItem it = items[wi];
    if (it.mat < 0) {  // bias chunk -> P tail (packed into the P all-reduce, optimizer.py:111-113)
      for (int x = lane; x < it.nrows; x += 32) {
        const float v = bias_g[it.row0 + x];
        bad |= !finite1(v);
        P[bias_off + it.row0 + x] = v;
      }
    } else {
      const MatDev md = mats[it.mat];
      k1_rows<R, EXACT>(md, it, lane, g, e, work, Q, P, bad);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
}

// ============================================================================= K2
// P-hat = MGS(P / W)   (comm.py:97-98, linalg.py:61-90), float64 inside.

__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  const double out = red[32];
  __syncthreads();
  return out;
}

__global__ void __launch_bounds__(kGsThreads) k2_gs(const MatDev* __restrict__ mats, int nmat,
                                                    float* __restrict__ P, int divisor,
                                                    const double* __restrict__ repl,
                                                    double* __restrict__ ws,
                                                    float* __restrict__ bias_out,
                                                    long long bias_off, long long nbias,
                                                    int* status) {
  __shared__ double red[33];
  if (*status & PSGD_STATUS_NONFINITE_GRAD) return;
  const double div = (double)divisor;
  if ((int)blockIdx.x >= nmat) {  // bias mean: P tail / W
    const long long nb = gridDim.x - nmat;
    bool bad = false;
    for (long long x = (blockIdx.x - nmat) * (long long)blockDim.x + threadIdx.x; x < nbias;
         x += nb * blockDim.x) {
      const float v = P[bias_off + x];
      bad |= !finite1(v);
      bias_out[x] = divisor == 1 ? v : v / (float)divisor;
    }
    if (bad) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
    return;
  }
  const MatDev md = mats[blockIdx.x];
  const int n = md.n, r = md.r;
  double* __restrict__ x = ws + md.p_off;  // row-major n x r, same indexing as P
  float* __restrict__ p = P + md.p_off;
  int bad = 0;
  for (int idx = threadIdx.x; idx < n * r; idx += blockDim.x) {
    const float v = p[idx];
    bad |= !finite1(v);
    x[idx] = (double)v / div;
  }
  if (__syncthreads_or(bad)) {  // linalg.py:35-36 (ContractViolation)
    if (threadIdx.x == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
    return;
  }
  // Each thread owns rows i = tid + k * blockDim for the whole kernel, so the
  // elementwise updates need no barrier beyond the ones inside block_sum.
  for (int j = 0; j < r; ++j) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i * r + j] * x[i * r + j];
    double before = sqrt(block_sum(s, red));
    for (int i2 = 0; i2 < j; ++i2) {
      s = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i * r + i2] * x[i * r + j];
      const double c = block_sum(s, red);
      for (int i = threadIdx.x; i < n; i += blockDim.x) x[i * r + j] -= c * x[i * r + i2];
    }
    s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i * r + j] * x[i * r + j];
    double nrm = sqrt(block_sum(s, red));
    int attempt = 0;
    while (nrm < 1e-12 * (before + 1.0)) {  // DEGENERATE_EPS, linalg.py:15,82
      if (attempt > 0) {                     // table holds attempt 0 only
        if (threadIdx.x == 0) atomicOr(status, PSGD_STATUS_REPLACEMENT);
        break;
      }
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        x[i * r + j] = repl[md.repl_off + (long long)j * n + i];
      before = 1.0;
      for (int i2 = 0; i2 < j; ++i2) {
        s = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i * r + i2] * x[i * r + j];
        const double c = block_sum(s, red);
        for (int i = threadIdx.x; i < n; i += blockDim.x) x[i * r + j] -= c * x[i * r + i2];
      }
      s = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i * r + j] * x[i * r + j];
      nrm = sqrt(block_sum(s, red));
      ++attempt;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i * r + j] /= nrm;
  }
  __syncthreads();  // rows were owned per-thread above; the copy-out mapping differs
  for (int idx = threadIdx.x; idx < n * r; idx += blockDim.x) p[idx] = (float)x[idx];
}

// ============================================================================= K3
// q_w = delta^T P-hat over a column slab holding all (or a chunk of) rows;
// fused e = delta - P-hat q_w^T (+ M-hat when W == 1)   (compressors.py:339,375-378)

template <int R, bool EXACT>
__global__ void __launch_bounds__(kThreads, 2)
    k3_q_ef(const MatDev* __restrict__ mats, const SlabItem* __restrict__ items, int beg,
            float* __restrict__ work, const float* __restrict__ Phat, float* __restrict__ qout,
            float* __restrict__ e, float* __restrict__ wsq, int* __restrict__ counters,
            int write_mhat, const int* __restrict__ status) {
  constexpr int DCAP = k3_dcap(R);
  extern __shared__ float smem[];
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const SlabItem it = items[beg + blockIdx.x];
  const MatDev md = mats[it.mat];
  const int r = EXACT ? R : md.r;
  const int n = md.n, m = md.m;
  const int vec = it.vec;
  const int cql = it.cq_log2;
  const int CQ = 1 << cql;
  const int C = CQ * vec;
  const int RG = kThreads >> cql;
  const int smax = DCAP / vec;
  const int rows_chunk = RG * smax;
  const int t = threadIdx.x;
  const int cq = t & (CQ - 1);
  const int rg = t >> cql;
  const int col = it.c0 + cq * vec;
  const bool colok = col < m;
  const int rbeg = it.chunk * rows_chunk;
  const int nrows = min(n - rbeg, rows_chunk);
  const int ncols = min(C, m - it.c0);

  float* ps = smem;                           // nrows x r   (P-hat rows of this chunk)
  float* red = ps + rows_chunk * r;           // RG x C x r  (per-row-group partial q)
  float* qs = red + RG * C * r;               // C x r       (q of this slab)

  // 1. all loads of the slab in flight at once
  float d[DCAP];
  const long long base = md.flat_off + (long long)rbeg * m + col;
  if (vec == 4) {
#pragma unroll
    for (int s = 0; s < DCAP / 4; ++s) {
      const int li = rg + RG * s;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (colok && li < nrows) v = __ldcs(reinterpret_cast<const float4*>(work + base + (long long)li * m));
      d[4 * s + 0] = v.x; d[4 * s + 1] = v.y; d[4 * s + 2] = v.z; d[4 * s + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int s = 0; s < DCAP; ++s) {
      const int li = rg + RG * s;
      d[s] = (colok && li < nrows) ? __ldcs(work + base + (long long)li * m) : 0.f;
    }
  }
  // 2. P-hat rows of the chunk to smem (overlaps the loads above)
  {
    const float* src = Phat + md.p_off + (long long)rbeg * r;
    for (int x = t; x < nrows * r; x += kThreads) ps[x] = src[x];
  }
  __syncthreads();
  // 3. per-thread partial q over its rows
  float qp[4][R];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < R; ++k) qp[v][k] = 0.f;
  if (vec == 4) {
#pragma unroll
    for (int s = 0; s < DCAP / 4; ++s) {
      const int li = rg + RG * s;
      if (li < nrows) {
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (EXACT || k < r) {
            const float pk = ps[li * r + k];
#pragma unroll
            for (int v = 0; v < 4; ++v) qp[v][k] = fmaf(d[4 * s + v], pk, qp[v][k]);
          }
        }
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < DCAP; ++s) {
      const int li = rg + RG * s;
      if (li < nrows) {
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (EXACT || k < r) qp[0][k] = fmaf(d[s], ps[li * r + k], qp[0][k]);
      }
    }
  }
  // 4. fixed-order reduction over the row groups
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (v < vec && (EXACT || k < r)) red[(rg * C + cq * vec + v) * r + k] = qp[v][k];
  __syncthreads();
  for (int o = t; o < C * r; o += kThreads) {
    float s = 0.f;
    for (int gidx = 0; gidx < RG; ++gidx) s += red[gidx * C * r + o];
    qs[o] = s;
  }
  __syncthreads();

  float* __restrict__ qdst = qout + md.q_off + (long long)it.c0 * r;
  if (it.nchunks > 1) {
    // tall matrix: publish the chunk partial; the last CTA of the slab reduces
    // all partials in chunk order (deterministic) and writes q.
    float* part = wsq + it.ws_off;
    for (int o = t; o < ncols * r; o += kThreads) part[(long long)it.chunk * C * r + o] = qs[o];
    __threadfence();
    __syncthreads();
    __shared__ int is_last;
    if (t == 0) is_last = atomicAdd(counters + it.slab, 1) == it.nchunks - 1;
    __syncthreads();
    if (is_last) {
      __threadfence();
      for (int o = t; o < ncols * r; o += kThreads) {
        float s = 0.f;
        for (int ch = 0; ch < it.nchunks; ++ch) s += __ldcg(part + (long long)ch * C * r + o);
        qdst[o] = s;
      }
      if (t == 0) counters[it.slab] = 0;  // self-resetting for the next launch
    }
    return;
  }
  for (int o = t; o < ncols * r; o += kThreads) qdst[o] = qs[o];

  // 5. error feedback (and M-hat at W=1) from the registers
  float qv[4][R];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < R; ++k)
      qv[v][k] = (v < vec && (EXACT || k < r)) ? qs[(cq * vec + v) * r + k] : 0.f;
  if (!colok) return;
  if (vec == 4) {
#pragma unroll
    for (int s = 0; s < DCAP / 4; ++s) {
      const int li = rg + RG * s;
      if (li < nrows) {
        float mh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < R; ++k) {
          if (EXACT || k < r) {
            const float pk = ps[li * r + k];
#pragma unroll
            for (int v = 0; v < 4; ++v) mh[v] = fmaf(pk, qv[v][k], mh[v]);
          }
        }
        const long long a = base + (long long)li * m;
        st_stream(reinterpret_cast<float4*>(e + a),
                  make_float4(d[4 * s] - mh[0], d[4 * s + 1] - mh[1], d[4 * s + 2] - mh[2],
                              d[4 * s + 3] - mh[3]));
        if (write_mhat)
          st_stream(reinterpret_cast<float4*>(work + a), make_float4(mh[0], mh[1], mh[2], mh[3]));
      }
    }
  } else {
#pragma unroll
    for (int s = 0; s < DCAP; ++s) {
      const int li = rg + RG * s;
      if (li < nrows) {
        float mh = 0.f;
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (EXACT || k < r) mh = fmaf(ps[li * r + k], qv[0][k], mh);
        const long long a = base + (long long)li * m;
        st_stream(e + a, d[s] - mh);
        if (write_mhat) st_stream(work + a, mh);
      }
    }
  }
}

// ============================================================================= K4 / K5
// Row-streaming outer products.  mode 0 (K4): e = delta - P-hat q^T, and M-hat
// in place of delta when write_mhat.  mode 1 (K5): M-hat = P-hat (q / div)^T,
// items with row0 == 0 also store Q-bar = q / div.

template <int R, bool EXACT, int MODE>
__global__ void __launch_bounds__(kThreads) k45_rows(const MatDev* __restrict__ mats,
                                                     const RowItem* __restrict__ items, int beg,
                                                     int end, float* __restrict__ work,
                                                     float* __restrict__ e,
                                                     const float* __restrict__ Phat,
                                                     const float* __restrict__ qsrc, int divisor,
                                                     float* __restrict__ qstore, int write_mhat,
                                                     const int* __restrict__ status) {
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int lane = threadIdx.x & 31;
  const int wi = beg + blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (wi >= end) return;
  const RowItem it = items[wi];
  const MatDev md = mats[it.mat];
  const int r = EXACT ? R : md.r;
  const int m = md.m;
  const float inv = 1.0f / (float)divisor;
  const float* __restrict__ Q = qsrc + md.q_off;
  if (MODE == 1 && it.row0 == 0 && qstore != nullptr && qstore != qsrc) {
    for (int x = lane; x < m * r; x += 32) {
      const float v = Q[x];
      qstore[md.q_off + x] = divisor == 1 ? v : v / (float)divisor;
    }
  }
  const int lg = it.lg;
  const int G = 1 << lg;
  const int gl = lane & (G - 1);
  const int sub = lane >> lg;
  const int rpp = 32 >> lg;
  for (int rb = 0; rb < it.nrows; rb += rpp) {
    const int li = rb + sub;
    if (li >= it.nrows) break;
    const int i = it.row0 + li;
    float ph[R];
#pragma unroll
    for (int k = 0; k < R; ++k) ph[k] = (EXACT || k < r) ? __ldg(Phat + md.p_off + (long long)i * r + k) : 0.f;
    const long long o = md.flat_off + (long long)i * m;
    const int head = min((int)((4 - (o & 3)) & 3), m);
    const int body4 = (m - head) >> 2;
    const int tail = m - head - 4 * body4;
    for (int s = gl; s < head + tail; s += G) {
      const int j = s < head ? s : head + 4 * body4 + (s - head);
      float mh = 0.f;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (EXACT || k < r) {
          float qk = __ldg(Q + (long long)j * r + k);
          if (MODE == 1 && divisor != 1) qk = qk / (float)divisor;
          mh = fmaf(ph[k], qk, mh);
        }
      }
      if (MODE == 0) {
        const float d = work[o + j];
        st_stream(e + o + j, d - mh);
        if (write_mhat) st_stream(work + o + j, mh);
      } else {
        st_stream(work + o + j, mh);
      }
    }
    const float* __restrict__ qrow = Q + (long long)head * r;
    const bool qal = ((head * r) & 3) == 0;
    float4* __restrict__ w4 = reinterpret_cast<float4*>(work + o + head);
    float4* __restrict__ e4 = reinterpret_cast<float4*>(e + o + head);
    for (int c = gl; c < body4; c += G) {
      float qv[4][R];
      load_q4<R, EXACT>(qrow + (long long)(4 * c) * r, qal, r, qv);
      float mh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < R; ++k) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float qk = qv[u][k];
          if (MODE == 1 && divisor != 1) qk = qk / (float)divisor;
          mh[u] = fmaf(ph[k], qk, mh[u]);
        }
      }
      if (MODE == 0) {
        const float4 d = __ldcs(w4 + c);
        st_stream(e4 + c, make_float4(d.x - mh[0], d.y - mh[1], d.z - mh[2], d.w - mh[3]));
        if (write_mhat) st_stream(w4 + c, make_float4(mh[0], mh[1], mh[2], mh[3]));
      } else {
        st_stream(w4 + c, make_float4(mh[0], mh[1], mh[2], mh[3]));
      }
    }
  }
  (void)inv;
}

// ============================================================================= tree mean
struct TreeArgs {
  const float* p[PSGD_MAX_TREE];
};

__global__ void k_tree_mean(TreeArgs a, int nbuf, long long count, float* __restrict__ out) {
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < count;
       x += (long long)gridDim.x * blockDim.x) {
    float v[PSGD_MAX_TREE];
    for (int w = 0; w < nbuf; ++w) v[w] = a.p[w][x];
    int cnt = nbuf;
    while (cnt > 1) {  // comm.py:51-67 pairing: ((v0+v1)+(v2+v3))+..., odd carried
      const int h = cnt >> 1;
      for (int w = 0; w < h; ++w) v[w] = v[2 * w] + v[2 * w + 1];
      if (cnt & 1) v[h] = v[cnt - 1];
      cnt = h + (cnt & 1);
    }
    out[x] = nbuf == 1 ? v[0] : v[0] / (float)nbuf;
  }
}

// ============================================================================= dispatch helpers

template <template <int, bool> class F, typename... A>
int dispatch_r(int r, A... args) {
  switch (r) {
    case 1: return F<1, true>::run(args...);
    case 2: return F<2, true>::run(args...);
    case 3: return F<3, true>::run(args...);
    case 4: return F<4, true>::run(args...);
    case 5: return F<5, true>::run(args...);
    case 6: return F<6, true>::run(args...);
    case 7: return F<7, true>::run(args...);
    case 8: return F<8, true>::run(args...);
    default: return F<16, false>::run(args...);
  }
}

}  // namespace

// ============================================================================= plan

struct psgd_plan {
  int nmat = 0, rank = 0, world = 1, device = 0;
  long long nbias = 0, flat_elems = 0, p_elems = 0, p_bias_off = 0, q_elems = 0, repl_elems = 0;
  std::vector<MatDev> mats;
  std::vector<RowItem> k1, k4, k5;
  std::vector<SlabItem> k3;
  std::vector<Group> g1, g3, g4, g5;
  int n_tall = 0, n_tall_slabs = 0;
  long long wsq_elems = 0;
  // device
  void* dev_block = nullptr;
  MatDev* d_mats = nullptr;
  RowItem *d_k1 = nullptr, *d_k4 = nullptr, *d_k5 = nullptr;
  SlabItem* d_k3 = nullptr;
  double* d_gsws = nullptr;
  float* d_wsq = nullptr;
  int* d_counters = nullptr;
};

namespace {

long long align4(long long x) { return (x + 3) & ~3LL; }

int lanes_log2_for(int m) {
  // lanes per row: enough that each lane streams ~4 float4 per row, 4..32
  const long long per = (m + 15) / 16;
  int lg = 2;
  while ((1 << lg) < per && lg < 5) ++lg;
  return lg;
}

struct K3Cfg {
  int vec, cql, rows_chunk, nchunks;
};

// K3 geometry of one matrix: as many columns per CTA as possible while the CTA
// still holds all n rows (RG * smax >= n); at least 32 columns per row segment
// (one 128-B line); never wider than needed to cover m.
K3Cfg k3_config(int n, int m, int r) {
  const int vec = (m % 4 == 0) ? 4 : 1;
  const int smax = k3_dcap(r) / vec;
  int cql = vec == 4 ? 3 : 5;
  while (cql < 8) {
    const int cq2 = 1 << (cql + 1);
    const int rg2 = kThreads / cq2;
    if ((long long)rg2 * smax < n) break;
    if ((long long)(cq2 / 2) * vec >= m) break;
    if (r > 8 && cq2 * vec > 256) break;  // smem budget at high rank
    ++cql;
  }
  const int RG = kThreads >> cql;
  const int rows_chunk = RG * smax;
  return {vec, cql, rows_chunk, (n + rows_chunk - 1) / rows_chunk};
}

void build_row_items(const std::vector<MatDev>& mats, bool tall_only, std::vector<RowItem>& items,
                     std::vector<Group>& groups) {
  // group by r so each launch is one template instantiation
  std::vector<int> rs;
  for (auto& md : mats)
    if (!tall_only || md.tall)
      if (std::find(rs.begin(), rs.end(), md.r) == rs.end()) rs.push_back(md.r);
  for (int r : rs) {
    Group gp{r, (int)items.size(), 0, 0};
    for (int mi = 0; mi < (int)mats.size(); ++mi) {
      const MatDev& md = mats[mi];
      if (md.r != r || (tall_only && !md.tall)) continue;
      const int lg = lanes_log2_for(md.m);
      const int rpp = 32 >> lg;
      int rows = std::max(1, kRowItemElems / md.m);
      rows = ((rows + rpp - 1) / rpp) * rpp;
      for (int r0 = 0; r0 < md.n; r0 += rows) items.push_back({mi, r0, std::min(rows, md.n - r0), lg});
    }
    gp.end = (int)items.size();
    groups.push_back(gp);
  }
}

}  // namespace

extern "C" {

int32_t psgd_version(void) { return 1; }

const char* psgd_last_error(void) { return g_last_error.c_str(); }

int psgd_plan_create(int32_t nmat, const int64_t* n, const int64_t* m, int32_t rank, int32_t world,
                     int64_t nbias, psgd_plan** out) {
  if (!out) return fail(PSGD_EINVAL, "out is NULL");
  *out = nullptr;
  if (nmat < 0 || (nmat > 0 && (!n || !m))) return fail(PSGD_EINVAL, "bad matrix list");
  if (rank < 1) return fail(PSGD_EINVAL, "rank must be >= 1, got " + std::to_string(rank));
  if (world < 1) return fail(PSGD_EINVAL, "world_size must be >= 1, got " + std::to_string(world));
  if (nbias < 0) return fail(PSGD_EINVAL, "nbias must be >= 0");
  psgd_plan* pl = new psgd_plan();
  pl->nmat = nmat;
  pl->rank = rank;
  pl->world = world;
  pl->nbias = nbias;
  cudaGetDevice(&pl->device);
  long long fo = 0, po = 0, qo = 0, ro = 0;
  for (int i = 0; i < nmat; ++i) {
    if (n[i] < 1 || m[i] < 1 || n[i] > (1LL << 26) || m[i] > (1LL << 26)) {
      delete pl;
      return fail(PSGD_EINVAL, "matrix " + std::to_string(i) + " has an empty or oversized dimension");
    }
    MatDev md{};
    md.n = (int)n[i];
    md.m = (int)m[i];
    md.r = (int)std::min<long long>(std::min<long long>(n[i], m[i]), rank);
    if (md.r > PSGD_MAX_RANK) {
      delete pl;
      return fail(PSGD_EINVAL, "effective rank " + std::to_string(md.r) + " exceeds PSGD_MAX_RANK");
    }
    md.tall = k3_config(md.n, md.m, md.r).nchunks > 1;
    md.flat_off = fo;
    md.p_off = po;
    md.q_off = qo;
    md.repl_off = ro;
    fo = align4(fo + (long long)md.n * md.m);
    po = align4(po + (long long)md.n * md.r);
    qo = align4(qo + (long long)md.m * md.r);
    ro += (long long)md.n * md.r;
    pl->n_tall += md.tall;
    pl->mats.push_back(md);
  }
  pl->flat_elems = fo;
  pl->p_bias_off = po;
  pl->p_elems = std::max(1LL, po + nbias);
  pl->q_elems = std::max(1LL, qo);
  pl->repl_elems = std::max(1LL, ro);

  // K1 items (+ bias chunks in the first group)
  build_row_items(pl->mats, false, pl->k1, pl->g1);
  if (nbias > 0) {
    if (pl->g1.empty()) pl->g1.push_back({1, 0, 0, 0});
    Group& g0 = pl->g1.front();
    std::vector<RowItem> bias;
    for (long long b = 0; b < nbias; b += kRowItemElems)
      bias.push_back({-1, (int)b, (int)std::min<long long>(kRowItemElems, nbias - b), 0});
    pl->k1.insert(pl->k1.begin() + g0.end, bias.begin(), bias.end());
    const int add = (int)bias.size();
    g0.end += add;
    for (size_t gi = 1; gi < pl->g1.size(); ++gi) { pl->g1[gi].beg += add; pl->g1[gi].end += add; }
  }
  build_row_items(pl->mats, true, pl->k4, pl->g4);
  build_row_items(pl->mats, false, pl->k5, pl->g5);

  // K3 slab items
  {
    std::vector<int> rs;
    for (auto& md : pl->mats)
      if (std::find(rs.begin(), rs.end(), md.r) == rs.end()) rs.push_back(md.r);
    for (int r : rs) {
      Group gp{r, (int)pl->k3.size(), 0, 0};
      for (int mi = 0; mi < nmat; ++mi) {
        const MatDev& md = pl->mats[mi];
        if (md.r != r) continue;
        const K3Cfg cf = k3_config(md.n, md.m, r);
        const int vec = cf.vec, cql = cf.cql;
        const int CQ = 1 << cql, C = CQ * vec, RG = kThreads / CQ;
        const int rows_chunk = cf.rows_chunk;
        const int nchunks = cf.nchunks;
        const int nslab = (md.m + C - 1) / C;
        for (int s = 0; s < nslab; ++s) {
          const int slab_id = nchunks > 1 ? pl->n_tall_slabs++ : -1;
          const long long wo = nchunks > 1 ? pl->wsq_elems : 0;
          if (nchunks > 1) pl->wsq_elems += (long long)nchunks * C * r;
          for (int ch = 0; ch < nchunks; ++ch)
            pl->k3.push_back({wo, mi, s * C, ch, nchunks, slab_id, vec, cql, 0});
        }
        const int smem = (rows_chunk * r + RG * C * r + C * r) * (int)sizeof(float);
        gp.smem = std::max(gp.smem, smem);
      }
      gp.end = (int)pl->k3.size();
      pl->g3.push_back(gp);
    }
  }

  // device block: mats | k1 | k3 | k4 | k5 | gs ws (doubles) | wsq | counters
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  const size_t o_mats = off; off = al(off + pl->mats.size() * sizeof(MatDev));
  const size_t o_k1 = off; off = al(off + pl->k1.size() * sizeof(RowItem));
  const size_t o_k3 = off; off = al(off + pl->k3.size() * sizeof(SlabItem));
  const size_t o_k4 = off; off = al(off + pl->k4.size() * sizeof(RowItem));
  const size_t o_k5 = off; off = al(off + pl->k5.size() * sizeof(RowItem));
  const size_t o_gs = off; off = al(off + (size_t)pl->p_elems * sizeof(double));
  const size_t o_wsq = off; off = al(off + (size_t)std::max(1LL, pl->wsq_elems) * sizeof(float));
  const size_t o_cnt = off; off = al(off + (size_t)std::max(1, pl->n_tall_slabs) * sizeof(int));
  cudaError_t ce = cudaMalloc(&pl->dev_block, off);
  if (ce != cudaSuccess) {
    delete pl;
    return fail(PSGD_ENOMEM, std::string("cudaMalloc plan: ") + cudaGetErrorString(ce));
  }
  char* b = static_cast<char*>(pl->dev_block);
  pl->d_mats = reinterpret_cast<MatDev*>(b + o_mats);
  pl->d_k1 = reinterpret_cast<RowItem*>(b + o_k1);
  pl->d_k3 = reinterpret_cast<SlabItem*>(b + o_k3);
  pl->d_k4 = reinterpret_cast<RowItem*>(b + o_k4);
  pl->d_k5 = reinterpret_cast<RowItem*>(b + o_k5);
  pl->d_gsws = reinterpret_cast<double*>(b + o_gs);
  pl->d_wsq = reinterpret_cast<float*>(b + o_wsq);
  pl->d_counters = reinterpret_cast<int*>(b + o_cnt);
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
  };
  if ((ce = up(pl->d_mats, pl->mats.data(), pl->mats.size() * sizeof(MatDev))) != cudaSuccess ||
      (ce = up(pl->d_k1, pl->k1.data(), pl->k1.size() * sizeof(RowItem))) != cudaSuccess ||
      (ce = up(pl->d_k3, pl->k3.data(), pl->k3.size() * sizeof(SlabItem))) != cudaSuccess ||
      (ce = up(pl->d_k4, pl->k4.data(), pl->k4.size() * sizeof(RowItem))) != cudaSuccess ||
      (ce = up(pl->d_k5, pl->k5.data(), pl->k5.size() * sizeof(RowItem))) != cudaSuccess ||
      (ce = cudaMemset(pl->d_counters, 0, (size_t)std::max(1, pl->n_tall_slabs) * sizeof(int))) !=
          cudaSuccess) {
    cudaFree(pl->dev_block);
    delete pl;
    return fail(PSGD_ECUDA, std::string("plan upload: ") + cudaGetErrorString(ce));
  }
  *out = pl;
  return PSGD_OK;
}

int psgd_plan_destroy(psgd_plan* plan) {
  if (!plan) return PSGD_OK;
  if (plan->dev_block) cudaFree(plan->dev_block);
  delete plan;
  return PSGD_OK;
}

int psgd_plan_get_info(const psgd_plan* pl, psgd_plan_info* o) {
  if (!pl || !o) return fail(PSGD_EINVAL, "NULL plan or out");
  o->flat_elems = pl->flat_elems;
  o->p_elems = pl->p_elems;
  o->p_bias_off = pl->p_bias_off;
  o->q_elems = pl->q_elems;
  o->repl_elems = pl->repl_elems;
  o->nbias = pl->nbias;
  o->nmat = pl->nmat;
  o->rank = pl->rank;
  o->world = pl->world;
  o->n_tall = pl->n_tall;
  o->items_k1 = (int64_t)pl->k1.size();
  o->items_k3 = (int64_t)pl->k3.size();
  auto nonempty = [](const std::vector<Group>& gs) {
    int c = 0;
    for (const Group& g : gs) c += g.end > g.beg;
    return c;
  };
  o->launches_ef_p = nonempty(pl->g1);
  o->launches_orthogonalize = (pl->nmat + (pl->nbias > 0)) > 0 ? 1 : 0;
  o->launches_q_ef = nonempty(pl->g3) + nonempty(pl->g4);
  o->launches_decompress = nonempty(pl->g5);
  return PSGD_OK;
}

int psgd_plan_matrix(const psgd_plan* pl, int32_t i, psgd_matrix_info* o) {
  if (!pl || !o) return fail(PSGD_EINVAL, "NULL plan or out");
  if (i < 0 || i >= pl->nmat) return fail(PSGD_EINVAL, "matrix index out of range");
  const MatDev& md = pl->mats[i];
  o->flat_off = md.flat_off;
  o->p_off = md.p_off;
  o->q_off = md.q_off;
  o->repl_off = md.repl_off;
  o->n = md.n;
  o->m = md.m;
  o->r_eff = md.r;
  o->tall = md.tall;
  return PSGD_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------- launchers

namespace {

template <int R, bool EXACT>
struct RunK1 {
  static int run(const psgd_plan* pl, const Group& gp, const float* g, const float* e, float* work,
                 const float* q, float* p, const float* bias_g, int* status, cudaStream_t st) {
    const int nitems = gp.end - gp.beg;
    if (nitems <= 0) return PSGD_OK;
    const int blocks = (nitems + 7) / 8;
    k1_ef_p<R, EXACT><<<blocks, kThreads, 0, st>>>(pl->d_mats, pl->d_k1, gp.beg, gp.end, g, e,
                                                   work, q, p, bias_g, pl->p_bias_off, status);
    PSGD_CUDA_CHECK(cudaGetLastError());
    return PSGD_OK;
  }
};

template <int R, bool EXACT>
struct RunK3 {
  static int run(const psgd_plan* pl, const Group& gp, float* work, const float* phat, float* qout,
                 float* e, const int* status, cudaStream_t st) {
    const int nitems = gp.end - gp.beg;
    if (nitems <= 0) return PSGD_OK;
    auto kern = k3_q_ef<R, EXACT>;
    if (gp.smem > 48 * 1024)
      PSGD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, gp.smem));
    kern<<<nitems, kThreads, gp.smem, st>>>(pl->d_mats, pl->d_k3, gp.beg, work, phat, qout, e,
                                            pl->d_wsq, pl->d_counters, pl->world == 1 ? 1 : 0,
                                            status);
    PSGD_CUDA_CHECK(cudaGetLastError());
    return PSGD_OK;
  }
};

template <int MODE>
struct RunK45Mode {
  template <int R, bool EXACT>
  struct F {
    static int run(const psgd_plan* pl, const RowItem* items, const Group& gp, float* work, float* e,
                   const float* phat, const float* qsrc, int divisor, float* qstore, int write_mhat,
                   const int* status, cudaStream_t st) {
      const int nitems = gp.end - gp.beg;
      if (nitems <= 0) return PSGD_OK;
      const int blocks = (nitems + 7) / 8;
      k45_rows<R, EXACT, MODE><<<blocks, kThreads, 0, st>>>(pl->d_mats, items, gp.beg, gp.end, work,
                                                            e, phat, qsrc, divisor, qstore,
                                                            write_mhat, status);
      PSGD_CUDA_CHECK(cudaGetLastError());
      return PSGD_OK;
    }
  };
};

template <int R, bool EXACT>
using RunK4 = RunK45Mode<0>::F<R, EXACT>;
template <int R, bool EXACT>
using RunK5 = RunK45Mode<1>::F<R, EXACT>;

bool check_dev(const psgd_plan* pl) {
  int dev = -1;
  cudaGetDevice(&dev);
  return dev == pl->device;
}

}  // namespace

extern "C" {

int psgd_ef_p(const psgd_plan* pl, const float* g, const float* e, float* work, const float* q,
              float* p, const float* bias_g, int32_t* status, void* stream) {
  if (!pl || !status || !p || (pl->flat_elems > 0 && (!g || !work || !q)) ||
      (pl->nbias > 0 && !bias_g))
    return fail(PSGD_EINVAL, "psgd_ef_p: NULL argument");
  if (!check_dev(pl)) return fail(PSGD_EINVAL, "psgd_ef_p: plan belongs to another device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (const Group& gp : pl->g1) {
    int rc = dispatch_r<RunK1>(gp.r, pl, gp, g, e, work, q, p, bias_g, (int*)status, st);
    if (rc) return rc;
  }
  return PSGD_OK;
}

int psgd_orthogonalize(const psgd_plan* pl, float* p, int32_t divisor, const double* repl,
                       float* bias_out, int32_t* status, void* stream) {
  if (!pl || !p || !status || divisor < 1 || (pl->nmat > 0 && !repl) || (pl->nbias > 0 && !bias_out))
    return fail(PSGD_EINVAL, "psgd_orthogonalize: bad argument");
  const int bias_blocks = pl->nbias > 0 ? (int)std::min<long long>(64, (pl->nbias + kGsThreads * 4 - 1) / (kGsThreads * 4)) : 0;
  const int grid = pl->nmat + bias_blocks;
  if (grid == 0) return PSGD_OK;
  k2_gs<<<grid, kGsThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      pl->d_mats, pl->nmat, p, divisor, repl, pl->d_gsws, bias_out, pl->p_bias_off, pl->nbias,
      (int*)status);
  PSGD_CUDA_CHECK(cudaGetLastError());
  return PSGD_OK;
}

int psgd_q_ef(const psgd_plan* pl, float* work, const float* p_hat, float* q_out, float* e,
              const int32_t* status, void* stream) {
  if (!pl || !status || (pl->nmat > 0 && (!work || !p_hat || !q_out || !e)))
    return fail(PSGD_EINVAL, "psgd_q_ef: NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (const Group& gp : pl->g3) {
    int rc = dispatch_r<RunK3>(gp.r, pl, gp, work, p_hat, q_out, e, (const int*)status, st);
    if (rc) return rc;
  }
  for (const Group& gp : pl->g4) {
    int rc = dispatch_r<RunK4>(gp.r, pl, (const RowItem*)pl->d_k4, gp, work, e, p_hat,
                               (const float*)q_out, 1, (float*)nullptr, pl->world == 1 ? 1 : 0,
                               (const int*)status, st);
    if (rc) return rc;
  }
  return PSGD_OK;
}

int psgd_decompress(const psgd_plan* pl, const float* p_hat, const float* q_sum, int32_t divisor,
                    float* q_store, float* mhat, const int32_t* status, void* stream) {
  if (!pl || !status || divisor < 1 || (pl->nmat > 0 && (!p_hat || !q_sum || !mhat)))
    return fail(PSGD_EINVAL, "psgd_decompress: bad argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (const Group& gp : pl->g5) {
    int rc = dispatch_r<RunK5>(gp.r, pl, (const RowItem*)pl->d_k5, gp, mhat, (float*)nullptr, p_hat,
                               q_sum, divisor, q_store, 1, (const int*)status, st);
    if (rc) return rc;
  }
  return PSGD_OK;
}

int psgd_step_single(const psgd_plan* pl, const float* g, float* e, float* work, float* q, float* p,
                     const float* bias_g, const double* repl, float* bias_out, int32_t* status,
                     void* stream) {
  if (!pl) return fail(PSGD_EINVAL, "NULL plan");
  if (pl->world != 1) return fail(PSGD_EINVAL, "psgd_step_single needs a world-1 plan");
  if (!status) return fail(PSGD_EINVAL, "NULL status");
  PSGD_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int32_t), static_cast<cudaStream_t>(stream)));
  int rc = psgd_ef_p(pl, g, e, work, q, p, bias_g, status, stream);
  if (!rc) rc = psgd_orthogonalize(pl, p, 1, repl, bias_out, status, stream);
  if (!rc) rc = psgd_q_ef(pl, work, p, q, e, status, stream);
  return rc;
}

int psgd_tree_mean(const float* const* bufs, int32_t nbuf, int64_t count, float* out, void* stream) {
  if (!bufs || !out || nbuf < 1 || nbuf > PSGD_MAX_TREE || count < 0)
    return fail(PSGD_EINVAL, "psgd_tree_mean: bad argument");
  if (count == 0) return PSGD_OK;
  TreeArgs a{};
  for (int i = 0; i < nbuf; ++i) {
    if (!bufs[i]) return fail(PSGD_EINVAL, "psgd_tree_mean: NULL buffer");
    a.p[i] = bufs[i];
  }
  const int blocks = (int)std::min<long long>((count + 255) / 256, 148 * 8);
  k_tree_mean<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(a, nbuf, count, out);
  PSGD_CUDA_CHECK(cudaGetLastError());
  return PSGD_OK;
}

}  // extern "C"
