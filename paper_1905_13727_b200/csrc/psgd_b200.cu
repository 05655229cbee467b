// psgd_b200.cu — B200 (sm_100a) kernels + C ABI for the PowerSGD compression hot path.
//
// Reference semantics: /root/reference/pkg/src/gradcomp
//   optimizer.py:98-129    EF add, per-matrix round trip, EF update, bias all-reduce
//   compressors.py:327-379 low_rank_iteration + PowerSGD.round_trip
//   linalg.py:54-90        modified Gram-Schmidt with seeded degenerate replacement
//   comm.py:51-98          tree-ordered all-reduce mean
//
// Every kernel is HBM-bound at small rank, so the design is
// about streaming each gradient element through an SM the minimum number of
// times with enough bytes in flight.  The two heavy kernels are persistent,
// warp-specialised TMA pipelines (one CTA per SM, 8 consumer warps + 1
// producer warp, mbarrier full/empty rings):
//
//   K1 k1_ef_p   producer: cp.async.bulk of row-aligned chunks of g and e into
//                smem; consumers: delta = g + e (stored, L2 evict-last so K3
//                finds it in L2), P = delta Q reduced in-warp / in-CTA.  Each
//                CTA also publishes a non-finite flag into the P buffer so the
//                P all-reduce carries it to every rank (all-or-nothing step).
//   K3 k3_q_ef   producer: one cp.async.bulk per row segment of a column slab
//                holding ALL n rows of the slab; consumers: Gram-Schmidt of the
//                slab's matrix (float64, once per matrix per CTA, while the
//                slab's bytes are in flight), q_w = delta^T P-hat, then
//                e = delta - P-hat q_w^T (and M-hat at W=1) from the same smem
//                copy — delta is read from memory once.
//   Tall matrices (n > 512) take K2 (per-matrix GS) + a register-slab split-n
//   q kernel + a row-streaming EF kernel (K4).  K5 writes M-hat after the
//   q all-reduce when W > 1.
// All reductions are fixed-order: results are bitwise run-to-run stable.

#include "../../include/psgd_b200.h"
#include "common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

using namespace psgd;

constexpr int kThreads = 256;      // plain CTA size (8 warps)
constexpr int kCons = 512;         // consumer threads of the TMA kernels (16 warps)
constexpr int kConsWarps = kCons / 32;
constexpr int kTmaThreads = kCons + 32;  // + 1 producer warp
constexpr int kRowItemElems = 4096;
constexpr int kGsThreads = 1024;
constexpr int kFusedNMax = 512;    // K3 fused path holds all rows of a slab
constexpr int K1_STAGES = 8;       // max stages (the plan picks the ring depth and the stage size)
constexpr int K1_CHUNK = 4608;     // floats of g (and of e) per chunk at the smallest stage
constexpr int K1_QSLOT_CAP = 12288;  // floats of Q per smem slot (2 slots)
constexpr int K1_QBIG_CAP = 18432;   // one large slot up to this (ResNet-18 r = 4: 4 x 4608); beyond: column tiles
constexpr int K1_RED_ROWS = 16;
constexpr int K1_STAGE_FLOATS = K1_CHUNK + 8;  // + misalignment slack of a chunk
constexpr int K3_STAGES = 2;
constexpr int K3_QMAX = 512;       // C * r per slab

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
  int lg1, qs;  // lg1: log2 lanes per row in K1 (2..9); qs: Q staged in smem by K1
                // (tall == 2: a tall matrix whose EF pass is k4_rows)
  int nck, pipe;  // nck: K1 chunks of the matrix; pipe: q / EF / M-hat by k3_pipe (n <= 512, r <= 8)
  int qld, rcols;  // Q is column-major: element (j, k) at q_off + k * qld + j, qld = align4(m);
                  // rcols: columns per attempt of the replacement table at repl_off (shared by equal n)
};

struct SgdArgs {   // fused heavy-ball update (optimizer.py:131-134); x == nullptr: off
  float *x, *mom, *bx, *bm;
  const float* bu;   // bias mean (the bias update u)
  long long nbias;   // bias scalars this launch updates (0: none)
  float lr, mu;
  int keep;          // 1: M-hat is still stored
};

// m = mu m + u ; x -= lr (u + m)  (one rounding for mu m + u; the reference's numpy
// does buf *= mu; buf += u in float64 — within the fp32 tolerance)
__device__ __forceinline__ void sgd4(float4& x, float4& m, const float4& u, float lr, float mu) {
  m.x = fmaf(mu, m.x, u.x); m.y = fmaf(mu, m.y, u.y); m.z = fmaf(mu, m.z, u.z); m.w = fmaf(mu, m.w, u.w);
  x.x -= lr * (u.x + m.x); x.y -= lr * (u.y + m.y); x.z -= lr * (u.z + m.z); x.w -= lr * (u.w + m.w);
}
__device__ __forceinline__ void sgd1(float& x, float& m, float u, float lr, float mu) {
  m = fmaf(mu, m, u);
  x -= lr * (u + m);
}
__device__ __forceinline__ void sgd_bias(const SgdArgs& sg, long long t0, long long stride) {
  for (long long i = t0; i < sg.nbias; i += stride) {
    float x = sg.bx[i], m = sg.bm[i];
    sgd1(x, m, sg.bu[i], sg.lr, sg.mu);
    sg.bm[i] = m;
    sg.bx[i] = x;
  }
}

struct RowItem {   // K4 / K5 warp item: rows [row0, row0 + nrows) of `mat`, 2^lg lanes per row
  int mat, row0, nrows, lg;
};

struct Chunk1 {    // K1 chunk: rows [row0, row0+nrows) x cols [c0, c0+ncols) of `mat`
  long long off;   // flat element offset of the first element
  int mat, row0, nrows, c0, ncols;
  int split, part;  // split >= 0: a segment of an over-long row (partial P)
  int pad;
};

struct SplitRow {  // an over-long row whose P is combined from `parts` partials
  int mat, row, base, parts;
};

struct SlabItem {  // K3 item: column slab [c0, c0 + C) x row chunk `chunk` of `mat` (nchunks == 1: fused)
  long long ws_off;
  int mat, c0, chunk, nchunks, slab, vec, cq_log2, pad;
  int ksub, pad2;  // tall items: register-slab row chunks per CTA (q accumulated in registers)
};

struct Group {
  int r, beg, end, smem;
  int tall;  // K3 groups: items of tall matrices (k3_slab<..., TALL = true>)
};

__host__ __device__ constexpr int k3_dcap(int r) { return r <= 4 ? 64 : 32; }

// ----------------------------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> shared, completion counted on an mbarrier (TMA, SASS UBLKCP)
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}
// 2-D tiled tensor copy global -> shared (TMA, SASS UTMALDG): box at (x = column, y = row)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bar_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
#ifndef PSGD_STORE_HINT
#define PSGD_STORE_HINT 1
#endif
#ifndef PSGD_PDL
#define PSGD_PDL 1
#endif
__device__ __forceinline__ void st_hint(float4* p, float4 v, uint64_t pol) {
#if !PSGD_STORE_HINT
  *p = v;
  return;
#endif
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t pol) {
#if !PSGD_STORE_HINT
  *p = v;
  return;
#endif
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, 512;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }

__device__ __forceinline__ bool finite4(float4 v) {
  return finite1(v.x) & finite1(v.y) & finite1(v.z) & finite1(v.w);
}

// Q rows j0..j0+3 of every column k < r (Q column-major, column stride ld) -> qv[4][RM].
// Lanes handle consecutive j0, so each column read is a run of consecutive
// 16-B words across the warp (bank-conflict free in smem, coalesced in L1).
template <int RM, bool SMEM>
__device__ __forceinline__ void load_q4(const float* __restrict__ q, int ld, bool aligned, int r,
                                        float (&qv)[4][RM]) {
#pragma unroll
  for (int k = 0; k < RM; ++k) {
    if (k < r) {
      const float* qk = q + (long long)k * ld;
      if (aligned) {
        const float4 v = SMEM ? *reinterpret_cast<const float4*>(qk) : __ldg(reinterpret_cast<const float4*>(qk));
        qv[0][k] = v.x; qv[1][k] = v.y; qv[2][k] = v.z; qv[3][k] = v.w;
      } else if ((reinterpret_cast<uintptr_t>(qk) & 7) == 0) {  // rows at 8 B (m = 2 mod 4, odd rows)
        const float2 a = SMEM ? *reinterpret_cast<const float2*>(qk) : __ldg(reinterpret_cast<const float2*>(qk));
        const float2 b = SMEM ? *reinterpret_cast<const float2*>(qk + 2) : __ldg(reinterpret_cast<const float2*>(qk + 2));
        qv[0][k] = a.x; qv[1][k] = a.y; qv[2][k] = b.x; qv[3][k] = b.y;
      } else {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) qv[jj][k] = SMEM ? qk[jj] : __ldg(qk + jj);
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) qv[jj][k] = 0.f;
    }
  }
}

// ----------------------------------------------------------------------------- Gram-Schmidt
// linalg.py:61-90: in-order MODIFIED Gram-Schmidt on x (n x r, float64, smem
// or global); thread `tid` of `nth` owns rows tid + k*nth, so only the
// reductions need barriers.  A degenerate column (norm < 1e-12 (before + 1),
// linalg.py:15,82) is replaced by the seeded column of attempt 0, 1, ... from
// `repl` (column j of attempt a at repl[(a * rcols + j) * n], linalg.py:54-58),
// re-projected, and tested again, exactly as the reference's while loop; a
// column still degenerate after PSGD_REPL_ATTEMPTS draws raises
// PSGD_STATUS_REPLACEMENT (the host turns it into an error).

struct BlockReducer {  // all threads of the CTA, __syncthreads
  double* red;         // >= 32 doubles
  __device__ double sum(double v) const {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w];
    __syncthreads();
    return t;
  }
};

// strided column helpers: 4 independent accumulators / loads in flight, so
// the loops are throughput- rather than latency-bound
__device__ __forceinline__ double col_dot(const double* a, const double* b, int n, int rs, int tid, int nth) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = tid;
  for (; i + 3 * nth < n; i += 4 * nth) {
    const double a0 = a[i * rs], a1 = a[(i + nth) * rs], a2 = a[(i + 2 * nth) * rs], a3 = a[(i + 3 * nth) * rs];
    const double b0 = b[i * rs], b1 = b[(i + nth) * rs], b2 = b[(i + 2 * nth) * rs], b3 = b[(i + 3 * nth) * rs];
    s0 = fma(a0, b0, s0);
    s1 = fma(a1, b1, s1);
    s2 = fma(a2, b2, s2);
    s3 = fma(a3, b3, s3);
  }
  for (; i < n; i += nth) s0 = fma(a[i * rs], b[i * rs], s0);
  return (s0 + s1) + (s2 + s3);
}
__device__ __forceinline__ void col_axpy(double* y, double c, const double* x, int n, int rs, int tid, int nth) {
#pragma unroll 4
  for (int i = tid; i < n; i += nth) y[i * rs] -= c * x[i * rs];
}
__device__ __forceinline__ void col_scale(double* y, double c, int n, int rs, int tid, int nth) {
#pragma unroll 4
  for (int i = tid; i < n; i += nth) y[i * rs] *= c;
}

template <class Red>
__device__ void mgs_inplace(double* x, int n, int r, const double* __restrict__ repl, int rcols, int tid, int nth,
                            const Red& red, int* status, int rs, int cs) {
  // element (i, j) lives at x[i * rs + j * cs]
  for (int j = 0; j < r; ++j) {
    double* xj = x + j * cs;
    double before = sqrt(red.sum(col_dot(xj, xj, n, rs, tid, nth)));
    double nrm = before;
    if (j > 0) {
      for (int i2 = 0; i2 < j; ++i2) {
        const double* xi = x + i2 * cs;
        const double c = red.sum(col_dot(xi, xj, n, rs, tid, nth));
        col_axpy(xj, c, xi, n, rs, tid, nth);
      }
      nrm = sqrt(red.sum(col_dot(xj, xj, n, rs, tid, nth)));
    }
    for (int attempt = 0; nrm < 1e-12 * (before + 1.0); ++attempt) {  // linalg.py:82-88
      if (attempt >= PSGD_REPL_ATTEMPTS) {
        if (tid == 0) atomicOr(status, PSGD_STATUS_REPLACEMENT);
        break;
      }
      const double* rv = repl + ((long long)attempt * rcols + j) * n;
      for (int i = tid; i < n; i += nth) xj[i * rs] = rv[i];
      before = 1.0;
      for (int i2 = 0; i2 < j; ++i2) {
        const double* xi = x + i2 * cs;
        const double c = red.sum(col_dot(xi, xj, n, rs, tid, nth));
        col_axpy(xj, c, xi, n, rs, tid, nth);
      }
      nrm = sqrt(red.sum(col_dot(xj, xj, n, rs, tid, nth)));
    }
    col_scale(xj, 1.0 / nrm, n, rs, tid, nth);  // one fp64 divide; scale by the reciprocal
  }
}

struct WarpReducer {  // one warp, shuffles only
  __device__ double sum(double v) const {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
  }
};

// ============================================================================= K1
// delta = g + e ; P[i,:] = sum_j delta[i,j] Q[j,:]   (optimizer.py:120, compressors.py:336)

struct K1Layout {  // dynamic smem: g stages | e stages | Q slots (| Q slots shifted by 2) | red | barriers
  int qslot_floats, nq;  // nq = 2 (double-buffered Q) or 1 (one large slot: m r up to ~128 KB)
  int qshift;            // 1: each Q slot has a copy shifted by two floats (rows of m = 2 mod 4 at 8 B)
  int off_q, off_red, off_bar, total;
  int stages, stage_floats;  // chosen per plan: the largest stage that fits beside the Q slots
};

// One chunk: rows of the chunk to row groups of G = 2^lg consumer threads.
template <int RM, bool QS>
__device__ __forceinline__ void k1_chunk(const Chunk1& ch, const MatDev& md, const float* __restrict__ Qm,
                                         const float* __restrict__ Qm2,
                                         const float* __restrict__ sg, const float* __restrict__ se,
                                         bool has_e, float* __restrict__ work, float* __restrict__ P,
                                         const SplitRow* __restrict__ splits, float* __restrict__ psplit,
                                         int* __restrict__ split_cnt, float* __restrict__ red, uint64_t keep,
                                         bool& bad) {
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int r = md.r, m = md.m;
  const int lg = md.lg1;
  const int G = 1 << lg;
  const int gl = t & (G - 1);
  const int gid = t >> lg;
  const int rpp = kCons >> lg;
  const long long a4 = ch.off & ~3LL;
  for (int rb = 0; rb < ch.nrows; rb += rpp) {
    const int li = rb + gid;
    const bool active = li < ch.nrows;
    float acc[RM];
#pragma unroll
    for (int q = 0; q < RM; ++q) acc[q] = 0.f;
    if (active) {
      const long long og = ch.off + (long long)li * m;
      const int sm = (int)(og - a4);
      const int nc = ch.ncols;
      const int head = min((int)((4 - (og & 3)) & 3), nc);
      const int body4 = (nc - head) >> 2;
      const int tail = nc - head - 4 * body4;
      for (int x = gl; x < head + tail; x += G) {
        const int j = x < head ? x : head + 4 * body4 + (x - head);
        const float gv = sg[sm + j];
        const float d = has_e ? gv + se[sm + j] : gv;
        st_hint(work + og + j, d, keep);
        const float* qj = Qm + ch.c0 + j;
#pragma unroll
        for (int q = 0; q < RM; ++q)
          if (q < r) acc[q] = fmaf(d, QS ? qj[(long long)q * md.qld] : __ldg(qj + (long long)q * md.qld), acc[q]);
      }
      const float4* __restrict__ g4 = reinterpret_cast<const float4*>(sg + sm + head);
      const float4* __restrict__ e4 = reinterpret_cast<const float4*>(se + sm + head);
      float4* __restrict__ w4 = reinterpret_cast<float4*>(work + og + head);
      const float* __restrict__ qrow = Qm + ch.c0 + head;
      bool qal = ((ch.c0 + head) & 3) == 0;
      if (QS && Qm2 != nullptr && ((ch.c0 + head) & 3) == 2) {  // the shifted copy: 16-B aligned Q rows
        qrow = Qm2 + ch.c0 + head - 2;
        qal = true;
      }
#pragma unroll 2
      for (int c = gl; c < body4; c += G) {
        const float4 gv = g4[c];
        const float4 ev = has_e ? e4[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 d = make_float4(gv.x + ev.x, gv.y + ev.y, gv.z + ev.z, gv.w + ev.w);
#ifndef PSGD_K1_NOSTORE
        st_hint(w4 + c, d, keep);
#endif
        float qv[4][RM];
        load_q4<RM, QS>(qrow + 4 * c, md.qld, qal, r, qv);
#pragma unroll
        for (int q = 0; q < RM; ++q) {
          acc[q] = fmaf(d.x, qv[0][q], acc[q]);
          acc[q] = fmaf(d.y, qv[1][q], acc[q]);
          acc[q] = fmaf(d.z, qv[2][q], acc[q]);
          acc[q] = fmaf(d.w, qv[3][q], acc[q]);
        }
      }
    }
    if (G <= 32) {  // fixed-order butterfly inside the row group; no barrier
      for (int off = G >> 1; off > 0; off >>= 1)
#pragma unroll
        for (int q = 0; q < RM; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
      if (active && gl == 0) {
        float* dst = P + md.p_off + (long long)(ch.row0 + li) * r;
#pragma unroll
        for (int q = 0; q < RM; ++q)
          if (q < r) {
            dst[q] = acc[q];
            bad |= !finite1(acc[q]);  // a non-finite delta poisons its P row (inf*0 = NaN too)
          }
      }
    } else {  // multi-warp rows: per-warp partials, combined once per chunk below
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int q = 0; q < RM; ++q) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
      if (active && lane == 0) {
#pragma unroll
        for (int q = 0; q < RM; ++q) red[(li * kConsWarps + warp) * RM + q] = acc[q];
      }
    }
  }
#ifdef PSGD_K1_NORED
  if (false) {
#else
  if (G > 32) {
#endif
    bar_consumers();
    const int nw = G >> 5;
    for (int o = t; o < ch.nrows * r; o += kCons) {
      const int li = o / r, q = o - li * r;
      const int w0 = (li % rpp) * nw;
      float s = 0.f;
      for (int w = 0; w < nw; ++w) s += red[(li * kConsWarps + w0 + w) * RM + q];
      bad |= !finite1(s);
      if (ch.split < 0) {
        P[md.p_off + (long long)(ch.row0 + li) * r + q] = s;
      } else {
        red[(K1_RED_ROWS * kConsWarps) * RM + q] = s;  // staged for the split combine below
      }
    }
    if (ch.split >= 0) {
      bar_consumers();
      if (t == 0) {  // segment of an over-long row: the last-arriving segment combines in part order
        const SplitRow sp = splits[ch.split];
        for (int q = 0; q < r; ++q) psplit[(long long)(sp.base + ch.part) * r + q] = red[(K1_RED_ROWS * kConsWarps) * RM + q];
        __threadfence();
        if (atomicAdd(split_cnt + ch.split, 1) == sp.parts - 1) {
          __threadfence();
          for (int q = 0; q < r; ++q) {
            float s = 0.f;
            for (int p = 0; p < sp.parts; ++p) s += __ldcg(psplit + (long long)(sp.base + p) * r + q);
            P[md.p_off + (long long)sp.row * r + q] = s;
          }
          split_cnt[ch.split] = 0;
        }
      }
    }
  }
}

#ifdef PSGD_K1_TIMES
__device__ unsigned long long g_k1_times[3 * 1024];  // per CTA: start, end, chunks (diagnostic builds only)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

template <int RM>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k1_ef_p(const MatDev* __restrict__ mats, const Chunk1* __restrict__ chunks,
            const int* __restrict__ cta_beg, const SplitRow* __restrict__ splits, K1Layout L,
            const float* __restrict__ g, const float* __restrict__ e, float* __restrict__ work,
            const float* __restrict__ Q, float* __restrict__ P, float* __restrict__ psplit,
            int* __restrict__ split_cnt, const float* __restrict__ bias_g, long long nbias,
            long long bias_off, long long flag_off, int* status) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sgb = reinterpret_cast<float*>(smem_raw);
  float* seb = sgb + L.stages * L.stage_floats;
  float* qsl = reinterpret_cast<float*>(smem_raw + L.off_q);
  float* red = reinterpret_cast<float*>(smem_raw + L.off_red);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + L.off_bar);
  uint64_t* empty = full + L.stages;
  uint64_t* qfull = empty + L.stages;
  uint64_t* qempty = qfull + 2;
  int* sflag = reinterpret_cast<int*>(qempty + 2);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int cb = cta_beg[blockIdx.x], ce = cta_beg[blockIdx.x + 1];
#ifdef PSGD_K1_TIMES
  if (t == 0) {
    g_k1_times[3 * blockIdx.x] = gtimer();
    g_k1_times[3 * blockIdx.x + 2] = ce - cb;
  }
#endif
  if (t == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], kConsWarps);
    }
    *sflag = 0;
    fence_mbar_init();
    if (blockIdx.x == 0) *status = 0;  // the step's status word: nothing else writes it during K1
  }
  __syncthreads();
#if PSGD_PDL
  pdl_trigger();  // let the next kernel's CTAs stage in as ours retire
#endif

  if (warp == kConsWarps) {  // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = pol_evict_first();
      const uint64_t polq = pol_evict_last();
      int cur = -1, qseq = -1;  // qseq counts the matrices whose Q is staged
      Chunk1 nx = chunks[cb < ce ? cb : 0];
      MatDev md{};
      for (int k = cb; k < ce; ++k) {
        const int s = (k - cb) % L.stages;
        const uint32_t ph = ((k - cb) / L.stages) & 1;
        const Chunk1 ch = nx;
        if (k + 1 < ce) nx = chunks[k + 1];  // next descriptor in flight
        if (ch.mat != cur) {  // Q of the next matrix into a smem slot (double-buffered)
          md = mats[ch.mat];
          cur = ch.mat;
          if (md.qs) {
            ++qseq;
            const int qs = qseq % L.nq;
            mbar_wait(&qempty[qs], ((qseq / L.nq) & 1) ^ 1);
            const uint32_t qb = (uint32_t)((long long)md.r * md.qld * 4);
            mbar_expect_tx(&qfull[qs], qb);
            tma_load(qsl + qs * L.qslot_floats, Q + md.q_off, qb, &qfull[qs], polq);
          }
        }
        mbar_wait(&empty[s], ph ^ 1);
        const long long a4 = ch.off & ~3LL;
        const long long span = (long long)(ch.nrows - 1) * md.m + ch.ncols;
        const long long b4 = (ch.off + span + 3) & ~3LL;
        const uint32_t bytes = (uint32_t)((b4 - a4) * 4);
        mbar_expect_tx(&full[s], e ? 2 * bytes : bytes);
        tma_load(sgb + s * L.stage_floats, g + a4, bytes, &full[s], pol);
        if (e) tma_load(seb + s * L.stage_floats, e + a4, bytes, &full[s], pol);
      }
    }
    return;
  }

  // ---------------- consumers
  bool bad = false;
  for (long long x = (long long)blockIdx.x * kCons + t; x < nbias; x += (long long)gridDim.x * kCons) {
    const float v = bias_g[x];  // bias rides in the P all-reduce (optimizer.py:111-113)
    bad |= !finite1(v);
    P[bias_off + x] = v;
  }
  const uint64_t keep = pol_evict_last();
  int cur = -1, qseq = -1, rpar = 0;
  bool cur_qs = false;
  Chunk1 nx = chunks[cb < ce ? cb : 0];
  MatDev md{};
  for (int k = cb; k < ce; ++k) {
    const int s = (k - cb) % L.stages;
    const uint32_t ph = ((k - cb) / L.stages) & 1;
    const Chunk1 ch = nx;
    if (k + 1 < ce) nx = chunks[k + 1];  // next descriptor in flight
    if (ch.mat != cur) {
      if (cur >= 0 && cur_qs) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&qempty[qseq % L.nq]);
      }
      md = mats[ch.mat];
      cur = ch.mat;
      cur_qs = md.qs != 0;
      if (cur_qs) {
        ++qseq;
        mbar_wait(&qfull[qseq % L.nq], (qseq / L.nq) & 1);
        if (L.qshift && (md.m & 3) == 2) {  // Q shifted by two floats: odd rows read it as float4
          const float* src = qsl + (qseq % L.nq) * L.qslot_floats;
          float* dst = qsl + (L.nq + qseq % L.nq) * L.qslot_floats;
          const int nq = md.r * md.qld;
          for (int x = t; x < nq; x += kCons) dst[x] = x + 2 < nq ? src[x + 2] : 0.f;
          bar_consumers();  // every warp left the previous matrix (this slot's last user) before it
        }
      }
    }
    mbar_wait(&full[s], ph);
    const float* sg = sgb + s * L.stage_floats;
    const float* se = seb + s * L.stage_floats;
    float* rb = red + (rpar & 1) * (K1_RED_ROWS * kConsWarps * RM + RM);
    if ((1 << md.lg1) > 32) ++rpar;
#ifdef PSGD_K1_NOCOMPUTE
    if (false)
#else
    if (cur_qs)
#endif
      k1_chunk<RM, true>(ch, md, qsl + (qseq % L.nq) * L.qslot_floats,
                         (L.qshift && (md.m & 3) == 2) ? qsl + (L.nq + qseq % L.nq) * L.qslot_floats : nullptr,
                         sg, se, e != nullptr, work, P, splits,
                         psplit, split_cnt, rb, keep, bad);
#ifndef PSGD_K1_NOCOMPUTE
    else
#else
    else if (false)
#endif
      k1_chunk<RM, false>(ch, md, Q + md.q_off, nullptr, sg, se, e != nullptr, work, P, splits, psplit, split_cnt,
                          rb, keep, bad);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (bad) atomicOr(sflag, 1);
  bar_consumers();
  if (t == 0) P[flag_off + blockIdx.x] = *sflag ? 1.f : 0.f;  // rides in the P all-reduce (K2 reads it)
#ifdef PSGD_K1_TIMES
  if (t == 0) g_k1_times[3 * blockIdx.x + 1] = gtimer();
#endif
}

// ============================================================================= K2
// P-hat = MGS(P / W) for every listed matrix, one CTA each (comm.py:97-98,
// linalg.py:61-90), float64 in smem when it fits; plus the bias mean
// (optimizer.py:111-113) in the trailing CTAs.  Launched with programmatic
// dependent launch: it waits for K1 (or the all-reduce), then immediately lets
// K3 launch, so K3's CTAs stream their delta slabs in while this runs.

struct GroupReducer {  // one 256-thread group of a CTA (named barrier 2 + gi), double-buffered partials
  double* red;          // 2 x 8 doubles
  int* parity;
  int gi;
  __device__ double sum(double v) const {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 7;
    double* buf = red + 8 * (*parity & 1);
    ++*parity;
    if (lane == 0) buf[w] = v;
    asm volatile("bar.sync %0, 256;" ::"r"(2 + gi) : "memory");
    double t = lane < 8 ? buf[lane] : 0.0;
#pragma unroll
    for (int off = 4; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    return __shfl_sync(0xffffffffu, t, 0);
  }
};

struct SyncReducer {  // all threads of the CTA, one __syncthreads per reduction
  double* red;        // 2 x 32 doubles, double-buffered by call parity
  int* parity;
  __device__ double sum(double v) const {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* buf = red + 32 * (*parity & 1);
    ++*parity;
    if (lane == 0) buf[warp] = v;
    __syncthreads();
    double t = lane < nw ? buf[lane] : 0.0;  // every warp reduces the partials itself
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    return t;
  }
};

constexpr int K2_SMEM_DOUBLES = 12288;  // 96 KB: n * r up to this stays in smem (CTA item)
constexpr int K2_WARP_DOUBLES = 2048;   // n * r up to this: one warp per matrix (no barriers)
constexpr int K2_THREADS = 256;

// items: [warp blocks | CTA blocks | bias blocks].  A warp block orthogonalises
// up to 8 small matrices, one per warp, reductions by shuffles only; a CTA
// block one medium matrix with 8 warps and a __syncthreads per reduction.
__global__ void __launch_bounds__(K2_THREADS, 1)
    k2_gs(const MatDev* __restrict__ mats, const int* __restrict__ wlist, int nw_items, int nwblocks,
          const int* __restrict__ clist, int nc_items, int wregion, const float* __restrict__ P,
          float* __restrict__ Phat, int divisor, const double* __restrict__ repl, float* __restrict__ bias_out,
          long long bias_off, long long nbias, long long flag_off, int nflags, int* status) {
  extern __shared__ __align__(16) double k2smem[];
  __shared__ double red[64];
  pdl_wait();     // P (K1 output or the all-reduce result) is complete
  pdl_trigger();  // K3 may launch now: it only touches P-hat after its own wait
  {
    int bad = 0;  // a non-finite gradient anywhere (any rank) poisons the whole step
    for (int x = threadIdx.x; x < nflags; x += blockDim.x) bad |= P[flag_off + x] != 0.f;
    if (__syncthreads_or(bad)) {
      if (threadIdx.x == 0) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
      return;
    }
  }
  const int b = blockIdx.x;
  const double inv_div = 1.0 / (double)divisor;
  if (b >= nwblocks + nc_items) {  // bias mean: P tail / W
    const long long nb = gridDim.x - nwblocks - nc_items;
    bool bad = false;
    for (long long x = (b - nwblocks - nc_items) * (long long)blockDim.x + threadIdx.x; x < nbias;
         x += nb * blockDim.x) {
      const float v = P[bias_off + x];
      bad |= !finite1(v);
      bias_out[x] = divisor == 1 ? v : v / (float)divisor;
    }
    if (bad) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
    return;
  }
  if (b < nwblocks) {  // ---- one warp per small matrix
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int item = b * (K2_THREADS / 32) + warp;
    if (item >= nw_items) return;
    const MatDev md = mats[wlist[item]];
    const int n = md.n, r = md.r;
    if (warp_mgs(P + md.p_off, n, r, inv_div, repl + md.repl_off, md.rcols, Phat + md.p_off, status)) return;
    double* x = k2smem + warp * wregion;  // column-major: lanes hit consecutive banks
    int bad = 0;
#pragma unroll 8
    for (int idx = lane; idx < n * r; idx += 32) {  // (loads independent of the smem stores)
      const float v = P[md.p_off + idx];
      bad |= !finite1(v);
      const int i = idx / r, j = idx - i * r;
      x[j * n + i] = (double)v * inv_div;
    }
    if (__any_sync(0xffffffffu, bad)) {  // linalg.py:35-36 (ContractViolation)
      if (lane == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
      return;
    }
    __syncwarp();
    mgs_inplace(x, n, r, repl + md.repl_off, md.rcols, lane, 32, WarpReducer{}, status, 1, n);
    __syncwarp();
    for (int idx = lane; idx < n * r; idx += 32) {
      const int i = idx / r, j = idx - i * r;
      Phat[md.p_off + idx] = (float)x[j * n + i];
    }
    return;
  }
  // ---- one CTA per medium matrix
  const MatDev md = mats[clist[b - nwblocks]];
  const int n = md.n, r = md.r;
  double* x = k2smem;  // column-major
  int bad = 0;
  for (int idx = threadIdx.x; idx < n * r; idx += blockDim.x) {
    const float v = P[md.p_off + idx];
    bad |= !finite1(v);
    const int i = idx / r, j = idx - i * r;
    x[j * n + i] = (double)v * inv_div;
  }
  if (__syncthreads_or(bad)) {  // linalg.py:35-36 (ContractViolation)
    if (threadIdx.x == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
    return;
  }
  int par = 0;
  SyncReducer sr{red, &par};
  mgs_inplace(x, n, r, repl + md.repl_off, md.rcols, threadIdx.x, blockDim.x, sr, status, 1, n);
  __syncthreads();  // rows were thread-owned above; the copy-out mapping differs
  for (int idx = threadIdx.x; idx < n * r; idx += blockDim.x) {
    const int i = idx / r, j = idx - i * r;
    Phat[md.p_off + idx] = (float)x[j * n + i];
  }
}

// ---- K2 for very tall matrices (n * r beyond the smem budget: LSTM, stress).
// Modified Gram-Schmidt in Gram space, re-orthogonalised (CholeskyQR2 form),
// with the reference's direct MGS as the fallback for columns Gram space cannot
// resolve:
// pass 1 (k2_gram<1>, one CTA per 128-row block): float64 Gram partials of
//   X = P / W; the last-arriving block of a matrix sums them in block order and
//   warp 0 runs the reference's MGS sequence (linalg.py:61-90: same
//   projections, same order) on coefficient vectors, giving T1 (r x r, upper
//   triangular) with X T1 orthonormal in exact arithmetic.  The Gram matrix
//   squares the condition number, so any column whose residual after
//   projection is below kGramTrust x its norm before projection — this
//   includes every column the reference would call degenerate (linalg.py:82)
//   — makes the block run the reference's direct MGS on X itself (float64, the
//   seeded replacement loop of linalg.py:82-88, global scratch) and write
//   P-hat; the later passes skip that matrix.
// pass 2 (k2_gram<2>, only when pass 1 saw a residual ratio below kGramRefine):
//   Gram partials of Y = X T1 computed from the rows, T2 from MGS on them and
//   T = T1 T2 (orthogonality ~1e-16 instead of ~1e-16 kappa^2).
// apply (k2_apply): P-hat = X T.

struct GramItem {
  int mat, row0, nrows, blk, nblk, gidx;
  long long gbase;  // first partial slot of this matrix in the Gram workspace
};

constexpr int K2G_ROWS = 128;
constexpr int K2G_TS = PSGD_MAX_RANK * PSGD_MAX_RANK + 8;  // doubles per matrix in wsT: T, then flags
constexpr int K2G_DIRECT = PSGD_MAX_RANK * PSGD_MAX_RANK;  // flag: P-hat written by the direct fallback
constexpr int K2G_REFINE = K2G_DIRECT + 1;                 // flag: pass 2 needed
constexpr double kGramTrust = 1e-5;
constexpr double kGramRefine = 1e-2;

template <int PASS>
__global__ void __launch_bounds__(256)
    k2_gram(const MatDev* __restrict__ mats, const GramItem* __restrict__ items, const float* __restrict__ P,
            int divisor, const double* __restrict__ repl, double* __restrict__ wsg, double* __restrict__ wsT,
            int* __restrict__ counters, long long flag_off, int nflags, double* __restrict__ scratch,
            float* __restrict__ Phat, int* status) {
  __shared__ double X[K2G_ROWS][PSGD_MAX_RANK + 1];
  __shared__ double G[PSGD_MAX_RANK][PSGD_MAX_RANK + 1];
  __shared__ double T1s[PSGD_MAX_RANK * PSGD_MAX_RANK];
  __shared__ double cvec[PSGD_MAX_RANK];
  __shared__ double Tm[PSGD_MAX_RANK][PSGD_MAX_RANK];  // Tm[j]: coefficient vector of output column j
  __shared__ double gpart[256];
  __shared__ double red[64];
  __shared__ int s_last, s_direct, s_refine;
  const GramItem it = items[blockIdx.x];  // plan constants: read before the wait
  const MatDev md = mats[it.mat];
  pdl_wait();
  pdl_trigger();  // the next pass / k2_apply may stage in; it waits for this grid itself
  int fbad = 0;  // pass 1: a non-finite gradient on any worker (flags ride in P) — checked after the
                 // block's first loads are in flight; nothing global is written before the check
  if (PASS == 1) {
    for (int x = threadIdx.x; x < nflags; x += blockDim.x) fbad |= P[flag_off + x] != 0.f;
  } else if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) {
    return;
  }
  const int n = md.n, r = md.r;
  const int npairs = r * (r + 1) / 2;
  const double inv_div = 1.0 / (double)divisor;
  const int t = threadIdx.x;
  double* Tg = wsT + (long long)it.gidx * K2G_TS;
  if (PASS == 2) {
    if (Tg[K2G_DIRECT] != 0.0 || Tg[K2G_REFINE] == 0.0) return;  // same for every block of the matrix
    for (int x = t; x < r * r; x += 256) T1s[x] = Tg[x];
  }
  int pk = -1, pl = -1;  // pair index -> (k, l), k <= l (npairs <= 136 < 256)
  if (t < npairs) {
    int p = t, k = 0;
    while (p >= r - k) { p -= r - k; ++k; }
    pk = k;
    pl = k + p;
  }
  // the block's rows in one pass of loads (one memory round trip), then every thread sums its
  // pair over a stride of rows and the row groups are added in order (fixed order)
  double acc = 0.0;
  int bad = 0;
  const int NGp = npairs > 0 ? 256 / npairs : 1;
  for (int r0 = it.row0; r0 < it.row0 + it.nrows; r0 += K2G_ROWS) {
    const int nr = min(K2G_ROWS, it.row0 + it.nrows - r0);
    __syncthreads();  // X (and T1s on the first block) ready / free
    if (PASS == 1) {
      for (int idx = t; idx < nr * r; idx += 256) {
        const int i = idx / r, k = idx - i * r;
        const float f = P[md.p_off + (long long)(r0 + i) * r + k];
        bad |= !finite1(f);
        X[i][k] = (double)f * inv_div;
      }
    } else {  // Y = X T1, row by row
      for (int idx = t; idx < nr * r; idx += 256) {
        const int i = idx / r, k = idx - i * r;
        const float* pr = P + md.p_off + (long long)(r0 + i) * r;
        double v = 0.0;
        for (int l = 0; l <= k; ++l) v = fma((double)pr[l] * inv_div, T1s[l * r + k], v);
        X[i][k] = v;
      }
    }
    __syncthreads();
    const int p = t % npairs, q = t / npairs;
    if (npairs > 0 && q < NGp) {
      int kk = 0, pp = p;
      while (pp >= r - kk) { pp -= r - kk; ++kk; }
      const int ll = kk + pp;
      double a = 0.0;
      for (int i = q; i < nr; i += NGp) a = fma(X[i][kk], X[i][ll], a);
      gpart[q * npairs + p] = a;
    }
    __syncthreads();
    if (pk >= 0)
      for (int qq = 0; qq < NGp; ++qq) acc += gpart[qq * npairs + t];
  }
  if (PASS == 1 && __syncthreads_or(fbad)) {  // mutate nothing
    if (t == 0) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
    return;
  }
  if (PASS == 1 && __syncthreads_or(bad)) {  // linalg.py:35-36
    if (t == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
  }
  if (pk >= 0) wsg[it.gbase + (long long)it.blk * npairs + t] = acc;
  __threadfence();
  __syncthreads();
  if (t == 0) s_last = atomicAdd(counters + it.gidx, 1) == it.nblk - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (t == 0) counters[it.gidx] = 0;
  if (ld_acquire(status) & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;  // block-uniform
  {  // fixed order: thread groups take blocks q, q + NG, ...; then groups in order
    const int NG = 256 / npairs;
    const int p = t % npairs, q = t / npairs;
    double sacc = 0.0;
    if (q < NG) {
      for (int b0 = q; b0 < it.nblk; b0 += 8 * NG) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          x[u] = b0 + u * NG < it.nblk ? __ldcg(wsg + it.gbase + (long long)(b0 + u * NG) * npairs + p) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) sacc += x[u];
      }
      gpart[q * npairs + p] = sacc;
    }
    __syncthreads();
    if (t < npairs) {
      double s2 = 0.0;
      for (int qq = 0; qq < NG; ++qq) s2 += gpart[qq * npairs + t];
      G[pk][pl] = s2;
      G[pl][pk] = s2;
    }
    if (t == 0) {
      s_direct = 0;
      s_refine = 0;
    }
  }
  __syncthreads();
  if (t < 32) {  // ---- MGS on coefficient vectors: value(c) = X c ; <a, b> = a^T G b
    const int lane = t;
    auto gdot = [&](const double* a, const double* b) {  // warp-parallel a^T G b
      double s = 0.0;
      if (lane < r) {
        double gb = 0.0;
        for (int l = 0; l < r; ++l) gb = fma(G[lane][l], b[l], gb);
        s = a[lane] * gb;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      return s;
    };
    bool direct = false, refine = false;
    for (int j = 0; j < r && !direct; ++j) {
      if (lane < r) cvec[lane] = lane == j ? 1.0 : 0.0;
      __syncwarp();
      const double before = sqrt(fmax(G[j][j], 0.0));
      double nrm = before;
      for (int i2 = 0; i2 < j; ++i2) {
        const double c = gdot(Tm[i2], cvec);
        __syncwarp();
        if (lane < r) cvec[lane] -= c * Tm[i2][lane];
        __syncwarp();
      }
      if (j > 0) nrm = sqrt(fmax(gdot(cvec, cvec), 0.0));
      if (PASS == 1 && (nrm < 1e-12 * (before + 1.0) || nrm < kGramTrust * before)) {
        direct = true;  // degenerate (linalg.py:82) or beyond what Gram space resolves
        break;
      }
      refine |= nrm < kGramRefine * before;
      const double inv = 1.0 / nrm;
      if (lane < r) Tm[j][lane] = cvec[lane] * inv;
      __syncwarp();
    }
    if (lane == 0) {
      s_direct = direct;
      s_refine = refine;
    }
  }
  __syncthreads();
  if (PASS == 1 && s_direct) {  // the reference's direct MGS on X (column-major scratch)
    double* x = scratch + md.p_off;
    for (int idx = t; idx < n * r; idx += 256) {
      const int i = idx / r, j = idx - i * r;
      x[(long long)j * n + i] = (double)P[md.p_off + idx] * inv_div;
    }
    __syncthreads();
    int par = 0;
    SyncReducer sr{red, &par};
    mgs_inplace(x, n, r, repl + md.repl_off, md.rcols, t, 256, sr, status, 1, n);
    __syncthreads();
    for (int idx = t; idx < n * r; idx += 256) {
      const int i = idx / r, j = idx - i * r;
      Phat[md.p_off + idx] = (float)x[(long long)j * n + i];
    }
    if (t == 0) Tg[K2G_DIRECT] = 1.0;
    return;
  }
  for (int x = t; x < r * r; x += 256) {  // T row-major [k][j]: P-hat column j = sum_k X[:, k] T[k][j]
    const int k = x / r, j = x - k * r;
    double v;
    if (PASS == 1) {
      v = Tm[j][k];
    } else {  // T = T1 T2
      v = 0.0;
      for (int l = 0; l < r; ++l) v = fma(T1s[k * r + l], Tm[j][l], v);
    }
    Tg[x] = v;
  }
  if (PASS == 1 && t == 0) {
    Tg[K2G_DIRECT] = 0.0;
    Tg[K2G_REFINE] = s_refine ? 1.0 : 0.0;
  }
}

__global__ void __launch_bounds__(256)
    k2_apply(const MatDev* __restrict__ mats, const int* __restrict__ gram_list, const int* __restrict__ blk_mat,
             const int* __restrict__ blk_row0, const float* __restrict__ P, int divisor,
             const double* __restrict__ wsT, float* __restrict__ Phat, const int* status) {
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int gidx = blk_mat[blockIdx.x];
  const double* T = wsT + (long long)gidx * K2G_TS;
  if (T[K2G_DIRECT] != 0.0) return;  // orthogonalised directly by k2_gram<1>
  const MatDev md = mats[gram_list[gidx]];
  const int n = md.n, r = md.r;
  const int i = blk_row0[blockIdx.x] + threadIdx.x;
  if (i >= n) return;
  const double inv_div = 1.0 / (double)divisor;
  double x[PSGD_MAX_RANK];
  for (int k = 0; k < r; ++k) x[k] = (double)P[md.p_off + (long long)i * r + k] * inv_div;
  for (int j = 0; j < r; ++j) {
    double s = 0.0;
    for (int k = 0; k <= j; ++k) s = fma(x[k], T[k * r + j], s);  // T is upper triangular
    Phat[md.p_off + (long long)i * r + j] = (float)s;
  }
}

// linalg.orthogonalize on float64 input (linalg.py:61-90 as the reference runs
// it, no fp32 rounding): one CTA, the matrix column-major in float64 scratch,
// the reference's MGS with the seeded replacement loop.
__global__ void __launch_bounds__(1024)
    k2_gs_f64(const MatDev* __restrict__ mats, int mi, const double* __restrict__ P, const double* __restrict__ repl,
              double* __restrict__ scratch, double* __restrict__ Phat, int* status) {
  __shared__ double red[64];
  const MatDev md = mats[mi];
  const int n = md.n, r = md.r, t = threadIdx.x, nth = blockDim.x;
  double* x = scratch + md.p_off;
  int bad = 0;
  for (int idx = t; idx < n * r; idx += nth) {
    const double v = P[idx];
    bad |= !isfinite(v);
    const int i = idx / r, j = idx - i * r;
    x[(long long)j * n + i] = v;
  }
  if (__syncthreads_or(bad)) {  // linalg.py:35-36 (ContractViolation)
    if (t == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
    return;
  }
  int par = 0;
  SyncReducer sr{red, &par};
  mgs_inplace(x, n, r, repl + md.repl_off, md.rcols, t, nth, sr, status, 1, n);
  __syncthreads();
  for (int idx = t; idx < n * r; idx += nth) {
    const int i = idx / r, j = idx - i * r;
    Phat[idx] = x[(long long)j * n + i];
  }
}

// ============================================================================= K3
// One CTA per column slab (all n rows x C cols of one matrix, or a chunk of
// rows for tall matrices), the slab held in registers: every load is issued
// up front (64 KB in flight per CTA).  Fused matrices are orthogonalised by
// their first slab's CTA (the others wait on a flag); tall ones by K2.
//   fused (n <= rows per CTA): q_w = delta^T P-hat, e = delta - P-hat q_w^T and
//     M-hat at W = 1 from the same registers: delta is read once
//     (compressors.py:339,375-378, optimizer.py:124-127).
//   tall (n > rows per CTA): a chunk of rows contributes a partial q; the
//     last-arriving chunk of the slab sums the partials in chunk order; the EF
//     pass is K4.

template <int R, bool EXACT, bool TALL>
__global__ void __launch_bounds__(kThreads, 2)
    k3_slab(const MatDev* __restrict__ mats, const SlabItem* __restrict__ items, float* __restrict__ work,
            const float* __restrict__ P, int divisor, const double* __restrict__ repl, float* __restrict__ Phat,
            float* __restrict__ qout, float* __restrict__ e, float* __restrict__ wsq, int* __restrict__ counters,
            float* __restrict__ bias_out, long long nbias,
            long long bias_off, long long flag_off, int nflags, int write_mhat,
            int* status) {
  constexpr int DCAP = k3_dcap(R);
  extern __shared__ __align__(16) unsigned char k3smem[];
  __shared__ int s_flag;
  pdl_trigger();  // dependents only stage in; they wait for this grid before reading its output
  const SlabItem it = items[blockIdx.x];
  const int t = threadIdx.x;
  const bool fused = !TALL;  // fused: all n rows in this CTA; tall: split rows, q partials
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
  const int cq = t & (CQ - 1);
  const int rg = t >> cql;
  const int col = it.c0 + cq * vec;
  const bool colok = col < m;
  const int rbeg = it.chunk * it.ksub * rows_chunk;
  const int nrows = min(n - rbeg, rows_chunk);
  const int ncols = min(C, m - it.c0);
  float* ps = reinterpret_cast<float*>(k3smem);                      // nrows x r
  float* red = ps + rows_chunk * r;                                   // RG x C x r
  float* qs = red + RG * C * r;                                       // C x r

  // 1. every load of the slab in flight at once
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
  // K3 follows K2, which started only after K1 completed: delta was final when
  // the loads above were issued.  Now wait for K2's P-hat and status.
  pdl_wait();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;  // mutate nothing
  if (blockIdx.x < 64 && nbias > 0) {  // bias mean (optimizer.py:111-113), first CTAs of the launch
    bool bad = false;
    const long long nb = min(64, (int)gridDim.x);
    for (long long x = (long long)blockIdx.x * kThreads + t; x < nbias; x += nb * kThreads) {
      const float v = P[bias_off + x];
      bad |= !finite1(v);
      bias_out[x] = divisor == 1 ? v : v / (float)divisor;
    }
    if (bad) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
  }
  // 2. P-hat of the rows.  Fused: the matrix's first slab CTA orthogonalises
  //    P / W (linalg.py:61-90, float64) while its loads fly and publishes it;
  //    the other slabs of the matrix (dispatched after it) wait for the flag.
  //    Tall: from K2.
  {  // P-hat rows of this chunk (from K2)
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
  // 3b. tall items: the CTA's further row chunks, q accumulated in registers (one
  //     reduction and one partial per CTA instead of one per 32-64 KB chunk)
  for (int sub = 1; TALL && !fused && sub < it.ksub; ++sub) {
    const int rb = rbeg + sub * rows_chunk;
    const int nr = min(n - rb, rows_chunk);
    if (nr <= 0) break;
    __syncthreads();  // every thread is done with ps
    for (int x = t; x < nr * r; x += kThreads) ps[x] = Phat[md.p_off + (long long)rb * r + x];
    const long long bs = md.flat_off + (long long)rb * m + col;
    if (vec == 4) {
#pragma unroll
      for (int s2 = 0; s2 < DCAP / 4; ++s2) {
        const int li = rg + RG * s2;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (colok && li < nr) v = __ldcs(reinterpret_cast<const float4*>(work + bs + (long long)li * m));
        d[4 * s2 + 0] = v.x; d[4 * s2 + 1] = v.y; d[4 * s2 + 2] = v.z; d[4 * s2 + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < DCAP; ++s2) {
        const int li = rg + RG * s2;
        d[s2] = (colok && li < nr) ? __ldcs(work + bs + (long long)li * m) : 0.f;
      }
    }
    __syncthreads();
    if (vec == 4) {
#pragma unroll
      for (int s2 = 0; s2 < DCAP / 4; ++s2) {
        const int li = rg + RG * s2;
        if (li < nr) {
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if (EXACT || k < r) {
              const float pk = ps[li * r + k];
#pragma unroll
              for (int v = 0; v < 4; ++v) qp[v][k] = fmaf(d[4 * s2 + v], pk, qp[v][k]);
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int s2 = 0; s2 < DCAP; ++s2) {
        const int li = rg + RG * s2;
        if (li < nr) {
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (EXACT || k < r) qp[0][k] = fmaf(d[s2], ps[li * r + k], qp[0][k]);
        }
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
  float* __restrict__ qdst = qout + md.q_off + it.c0;  // column-major: (c, k) at k * qld + c
  if constexpr (TALL) {  // partial of a tall slab; the last chunk combines in chunk order
    float* part = wsq + it.ws_off;
    for (int o = t; o < ncols * r; o += kThreads) part[(long long)it.chunk * C * r + o] = qs[o];
    __threadfence();
    __syncthreads();
    if (t == 0) s_flag = atomicAdd(counters + it.slab, 1) == it.nchunks - 1;
    __syncthreads();
    if (s_flag) {
      __threadfence();
      for (int o = t; o < ncols * r; o += kThreads) {
        const int k = o / ncols, cc = o - k * ncols;
        float s = 0.f;
        const float* pc = part + cc * r + k;
        int ch = 0;
        for (; ch + 8 <= it.nchunks; ch += 8) {  // 8 loads in flight, summed in chunk order
          float y[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) y[u] = __ldcg(pc + (long long)(ch + u) * C * r);
#pragma unroll
          for (int u = 0; u < 8; ++u) s += y[u];
        }
        for (; ch < it.nchunks; ++ch) s += __ldcg(pc + (long long)ch * C * r);
        qdst[(long long)k * md.qld + cc] = s;
      }
      if (t == 0) counters[it.slab] = 0;
    }
    return;
  } else {
  for (int o = t; o < ncols * r; o += kThreads) {
    const int k = o / ncols, cc = o - k * ncols;
    qdst[(long long)k * md.qld + cc] = qs[cc * r + k];
  }
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
                  make_float4(d[4 * s] - mh[0], d[4 * s + 1] - mh[1], d[4 * s + 2] - mh[2], d[4 * s + 3] - mh[3]));
        if (write_mhat) st_stream(reinterpret_cast<float4*>(work + a), make_float4(mh[0], mh[1], mh[2], mh[3]));
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
  }  // !TALL
}

// ============================================================================= K3 pipeline
// k3_pipe: q_w = delta^T P-hat, e = delta - P-hat q_w^T and (W = 1) M-hat for
// every matrix with n <= 512 (compressors.py:339, 375-378; optimizer.py:124-127),
// as one persistent warp-specialised kernel (1 CTA per SM):
//   producer warp: takes the next column slab (all n rows x C columns of one
//     matrix, <= 64 KB) from a global counter (dynamic balance), stages it into
//     shared memory with 2-D tensor TMA (one box per 256 rows) plus P-hat's n x r
//     rows with a 1-D bulk copy, on a 2-3 stage mbarrier ring;
//   8 consumer warps: q from the staged slab (fixed-order warp-shuffle + smem
//     reduction), then e (and M-hat) from the same staged bytes, float4
//     streaming stores.  delta is read from HBM once.
// Slabs of matrices without a tensor map (m % 4 != 0, or beyond K3P_MAXMAPS)
// are loaded by the consumers themselves (scalar, "direct").  Launched with
// programmatic dependent launch after K2: delta is final when it starts (K2
// began after K1 completed), so the slab loads overlap K2; P-hat is fetched
// after griddepcontrol.wait.

constexpr int K3P_CW = 16;                     // consumer warps
constexpr int K3P_CT = 32 * K3P_CW;            // consumer threads
#ifndef PSGD_K3P_GROUPS
#define PSGD_K3P_GROUPS 2
#endif
constexpr int K3P_GROUPS = PSGD_K3P_GROUPS;    // consumer groups taking alternate stages
constexpr int K3P_GW = K3P_CW / K3P_GROUPS;    // warps per group
constexpr int K3P_GT = 32 * K3P_GW;            // threads per group
constexpr int K3P_SLAB = 16384;                // floats of delta per stage (all rows x C columns)
constexpr int K3P_MAXMAPS = 48;

struct PipeItem {
  int mat, c0, C, map;  // map < 0: direct (consumer) loads
};
struct K3Maps {
  CUtensorMap m[K3P_MAXMAPS];
};
struct K3PLayout {
  int stages, phat_floats, stage_floats, slab_floats;  // stage: slab (slab_floats) | P-hat rows
  int off_red, off_qs, off_bar, total;
  int red_floats;  // per consumer group: K3P_GW x C x r
  int qs_floats;   // per consumer group: C x r (largest slab of the plan)
};
struct K3GS {  // Gram-Schmidt of the pipeline's matrices inside k3_pipe (no K2 launch for them)
  const int* list;     // matrices orthogonalised here; CTA b owns list[b], list[b + grid], ...
  int n;               // 0: P-hat comes from K2 (the previous launch)
  int* ready;          // per matrix: 1 once its P-hat is published (reset by the last CTA out)
  const float* P;      // summed P: flag tail at flag_off, bias tail at bias_off
  const double* repl;
  float* bias_out;     // non-null: this launch writes the bias mean
  long long flag_off, bias_off, nbias;
  int nflags, divisor;
};
struct K3PHdr {  // what the consumers need of a staged slab (written by the producer)
  long long base, q_off;  // base: flat offset of (row 0, column c0)
  int n, m, r, C, c0, direct, qld, live;  // live = 0: no more slabs
};

// linalg.py:61-90 for one matrix (n <= 512, r <= R) by one consumer group of k3_pipe:
// thread gt owns rows gt and gt + 256 in registers (float64), reductions over the
// group's named barrier; the same MGS sequence, threshold and seeded replacement loop
// (linalg.py:82-88, draws from repl) as mgs_inplace.
struct GroupReducer256 {
  double* red;  // 2 x K3P_GW doubles
  int* parity;
  int bar_id;
  __device__ double sum(double v) const {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, gw = (threadIdx.x >> 5) % K3P_GW;
    double* buf = red + K3P_GW * (*parity & 1);
    ++*parity;
    if (lane == 0) buf[gw] = v;
    bar_named(bar_id, K3P_GT);
    double t2 = 0.0;
#pragma unroll
    for (int w = 0; w < K3P_GW; ++w) t2 += buf[w];
    return t2;
  }
};

template <int R>
__device__ void group_mgs(const MatDev& md, const float* __restrict__ P, int divisor, const double* __restrict__ repl,
                          float* __restrict__ Phat, int* status, const GroupReducer256& red, int gt) {
  const int n = md.n, r = md.r;
  const double inv_div = 1.0 / (double)divisor;
  double x[2][R];
  bool bad = false;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = gt + K3P_GT * h;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const float v = (i < n && j < r) ? __ldcg(P + md.p_off + (long long)i * r + j) : 0.f;
      bad |= !finite1(v);
      x[h][j] = (double)v * inv_div;
    }
  }
  if (red.sum(bad ? 1.0 : 0.0) != 0.0) {  // linalg.py:35-36 (ContractViolation)
    if (gt == 0) atomicOr(status, PSGD_STATUS_NONFINITE_P);
    return;
  }
  auto dot = [&](int a, int b) {
    double s2 = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) s2 = fma(x[h][a], x[h][b], s2);
    return red.sum(s2);
  };
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (j >= r) break;
    double before = sqrt(dot(j, j));
    double nrm = before;
    for (int attempt = 0;; ++attempt) {  // attempt a > 0: after the a-th replacement draw
      if (attempt > 0 || j > 0) {
#pragma unroll
        for (int i2 = 0; i2 < R; ++i2) {
          if (i2 >= j) break;
          const double c = dot(i2, j);
#pragma unroll
          for (int h = 0; h < 2; ++h) x[h][j] -= c * x[h][i2];
        }
        nrm = sqrt(dot(j, j));
      }
      if (!(nrm < 1e-12 * (before + 1.0))) break;  // linalg.py:82-88
      if (attempt == PSGD_REPL_ATTEMPTS) {
        if (gt == 0) atomicOr(status, PSGD_STATUS_REPLACEMENT);
        break;
      }
      const double* rv = repl + md.repl_off + ((long long)attempt * md.rcols + j) * n;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = gt + K3P_GT * h;
        x[h][j] = i < n ? rv[i] : 0.0;
      }
      before = 1.0;
    }
    const double inv = 1.0 / nrm;
#pragma unroll
    for (int h = 0; h < 2; ++h) x[h][j] *= inv;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = gt + K3P_GT * h;
    if (i < n)
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (j < r) Phat[md.p_off + (long long)i * r + j] = (float)x[h][j];
  }
}

template <int R>
__global__ void __launch_bounds__(K3P_CT + 32, 1)
    k3_pipe(const __grid_constant__ K3Maps maps, const MatDev* __restrict__ mats, const PipeItem* __restrict__ items,
            int nitems, K3PLayout L, float* __restrict__ work, const float* __restrict__ Phat,
            float* __restrict__ qout, float* __restrict__ e, int write_mhat, int* __restrict__ ctr, int* status,
            SgdArgs sg, K3GS gs) {
  extern __shared__ __align__(1024) unsigned char k3p_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(k3p_smem + L.off_bar);
  uint64_t* empty = full + L.stages;
  K3PHdr* hdr = reinterpret_cast<K3PHdr*>(empty + L.stages);
  __shared__ int s_next, s_claim[K3P_GROUPS];  // stage claiming: the next ring position, per-group broadcast
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], K3P_GW);  // a stage is consumed by one group
    }
    s_next = 0;
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == K3P_CW) {  // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = pol_evict_first();
      bool waited = false;
      if (gs.n > 0) {  // no K2 in front: delta (K1's output) is final only after this
        pdl_wait();
        waited = true;
      }
      // one item of lookahead: the next slab's index (global atomic) and descriptors
      // are fetched while the current slab's copies fly, so the dependent
      // atomic -> item -> matrix loads are off the issue path
      int it = atomicAdd(ctr, 1);
      PipeItem pi{};
      MatDev md{};
      if (it < nitems) {
        pi = items[it];
        md = mats[pi.mat];
      }
      for (int k = 0, ends = 0; ends < K3P_GROUPS; ++k) {
        const int s = k % L.stages;
        mbar_wait(&empty[s], ((k / L.stages) & 1) ^ 1);
        if (it >= nitems) {  // one end marker per consumer group (groups take alternate stages)
          hdr[s].live = 0;
          mbar_arrive(&full[s]);
          ++ends;
          continue;
        }
        float* dst = reinterpret_cast<float*>(k3p_smem) + (long long)s * L.stage_floats;
        const int br = md.n < 256 ? md.n : 256;
        const int nbox = (md.n + br - 1) / br;
        const uint32_t pb = (uint32_t)(((md.n * md.r + 3) & ~3) * 4);
        hdr[s] = K3PHdr{md.flat_off + pi.c0, md.q_off, md.n, md.m, md.r, pi.C, pi.c0, pi.map < 0, md.qld, 1};
        mbar_expect_tx(&full[s], (pi.map >= 0 ? (uint32_t)(nbox * br * pi.C * 4) : 0u) + pb);
        if (pi.map >= 0)
          for (int b = 0; b < nbox; ++b) tma_load_2d(dst + b * br * pi.C, &maps.m[pi.map], pi.c0, b * br, &full[s], pol);
        if (!waited) {  // P-hat is K2's output
          pdl_wait();
          waited = true;
        }
        if (gs.n > 0)  // P-hat of this matrix published by its owner CTA
          while (ld_acquire(gs.ready + pi.mat) == 0) __nanosleep(32);
        tma_load(dst + L.slab_floats, Phat + md.p_off, pb, &full[s], pol);
        it = atomicAdd(ctr, 1);
        if (it < nitems) {
          pi = items[it];
          md = mats[pi.mat];
        }
      }
    }
    return;
  }

  // ---------------- consumers: K3P_GROUPS groups of K3P_GW warps, each claiming the next
  // filled stage when free (ping-pong), so one group's q reduction overlaps the other's stores
  const int grp = warp / K3P_GW, gw = warp - grp * K3P_GW, gt = t - grp * K3P_GT;
  float* red = reinterpret_cast<float*>(k3p_smem + L.off_red) + grp * L.red_floats;  // K3P_GW x C x r
  float* qs = reinterpret_cast<float*>(k3p_smem + L.off_qs) + grp * L.qs_floats;     // C x r
  const int bar_id = 1 + grp;
  pdl_wait();  // K2 / K1 / the P all-reduce complete: P (or P-hat) and the status word are final
  bool skip = (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) != 0;  // mutate nothing
  if (gs.n > 0) {
    // no K2 in front: the non-finite flags of every K1 CTA (optimizer.py:72-76, carried in P)
    bool fl = false;
    for (int x = lane; x < gs.nflags; x += 32) fl |= gs.P[gs.flag_off + x] != 0.f;
    fl = __any_sync(0xffffffffu, fl);
    skip |= fl;
    if (blockIdx.x == 0 && t == 0 && fl) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
    if (gs.bias_out && !skip)  // bias mean (optimizer.py:111-113)
      for (long long x = (long long)blockIdx.x * K3P_CT + t; x < gs.nbias; x += (long long)gridDim.x * K3P_CT) {
        const float v = gs.P[gs.bias_off + x];
        gs.bias_out[x] = gs.divisor == 1 ? v : v / (float)gs.divisor;
      }
    if (grp == 0) {  // this CTA's matrices: P-hat = MGS(P / W) (linalg.py:61-90), then publish
      __shared__ double gsred[2 * K3P_GW];
      int par = 0;
      GroupReducer256 gr{gsred, &par, bar_id};
      for (int k = blockIdx.x; k < gs.n; k += gridDim.x) {
        const int mi = gs.list[k];
        if (!skip) group_mgs<R>(mats[mi], gs.P, gs.divisor, gs.repl, const_cast<float*>(Phat), status, gr, gt);
        __threadfence();
        bar_named(bar_id, K3P_GT);
        if (gt == 0) st_release(gs.ready + mi, 1);
      }
    }
  }
  if (sg.x && !skip) sgd_bias(sg, (long long)blockIdx.x * K3P_CT + t, (long long)gridDim.x * K3P_CT);
  const bool fuse = sg.x != nullptr;
  const bool store_mhat = write_mhat && (!fuse || sg.keep);
  for (;;) {
    // a free group claims the next ring position (the producer fills them in order), so a
    // group busy with an owner GS or a long slab never holds up the other one
    if (gt == 0) s_claim[grp] = atomicAdd(&s_next, 1);
    bar_named(bar_id, K3P_GT);
    const int k = s_claim[grp];
    bar_named(bar_id, K3P_GT);
    const int s = k % L.stages;
    mbar_wait(&full[s], (k / L.stages) & 1);
    const K3PHdr hd = hdr[s];
    if (!hd.live) break;
    const int n = hd.n, m = hd.m, r = hd.r, C = hd.C, c0 = hd.c0;
    const float* slab = reinterpret_cast<const float*>(k3p_smem) + (long long)s * L.stage_floats;
    const float* ph = slab + L.slab_floats;
    const long long base = hd.base;
#ifdef PSGD_K3P_NOCONSUME
    if (false) {
#else
    if (!skip) {
#endif
      if (hd.direct) {  // direct: the consumers stage the slab themselves
        float* ds = const_cast<float*>(slab);
        for (int idx = gt; idx < n * C; idx += K3P_GT) {
          const int i = idx / C, c = idx - i * C;
          ds[idx] = c0 + c < m ? __ldcs(work + base + (long long)i * m + c) : 0.f;
        }
        bar_named(bar_id, K3P_GT);
      }
      const int CQ = C >> 2, RG = K3P_GT / CQ;
      const int cq = gt & (CQ - 1), rg = gt / CQ;
      // 1. per-thread partial q over rows rg, rg + RG, ...
      float qp[4][R];
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int kk = 0; kk < R; ++kk) qp[v][kk] = 0.f;
#pragma unroll 4
      for (int i = rg; i < n; i += RG) {
        const float4 d = *reinterpret_cast<const float4*>(slab + i * C + 4 * cq);
#pragma unroll
        for (int kk = 0; kk < R; ++kk) {
          if (kk < r) {
            const float p = ph[i * r + kk];
            qp[0][kk] = fmaf(d.x, p, qp[0][kk]);
            qp[1][kk] = fmaf(d.y, p, qp[1][kk]);
            qp[2][kk] = fmaf(d.z, p, qp[2][kk]);
            qp[3][kk] = fmaf(d.w, p, qp[3][kk]);
          }
        }
      }
      // 2. fixed-order reduction: lanes of a warp that share cq (butterfly), then warps in order
      for (int off = CQ; off < 32; off <<= 1)
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int kk = 0; kk < R; ++kk) qp[v][kk] += __shfl_xor_sync(0xffffffffu, qp[v][kk], off);
      bar_named(bar_id, K3P_GT);  // every thread of the group is done with the previous slab's qs
      if (lane < CQ)
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int kk = 0; kk < R; ++kk)
            if (kk < r) red[(gw * C + 4 * cq + v) * r + kk] = qp[v][kk];
      bar_named(bar_id, K3P_GT);
      for (int o = gt; o < C * r; o += K3P_GT) {
        float sacc = 0.f;
        for (int w = 0; w < K3P_GW; ++w) sacc += red[w * C * r + o];
        qs[o] = sacc;
        const int c = o / r, kk = o - c * r;
        if (c0 + c < m) qout[hd.q_off + (long long)kk * hd.qld + c0 + c] = sacc;  // column-major Q
      }
      bar_named(bar_id, K3P_GT);
      // 3. e = delta - P-hat q^T (and M-hat) from the staged slab
      float qv[4][R];
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int kk = 0; kk < R; ++kk) qv[v][kk] = kk < r ? qs[(4 * cq + v) * r + kk] : 0.f;
      const int col = c0 + 4 * cq;
#ifdef PSGD_K3P_NOSTORE
      if (col < 0) {
#else
      if (col < m) {
#endif
        const bool vec = !hd.direct;  // tensor-mapped matrices have m % 4 == 0: whole float4 in range
        if (fuse && vec) {
          // fused optimizer (optimizer.py:131-134): x and m of 4 rows are loaded together,
          // M-hat is consumed from the registers (a software-pipelined prefetch of the
          // next 4 rows measured slower: it needs registers the 17-warp CTA does not have)
          for (int i0 = rg; i0 < n; i0 += 4 * RG) {
            float4 xv[4], mv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + u * RG;
              if (i < n) {
                const long long a = base + (long long)i * m + 4 * cq;
                xv[u] = __ldcs(reinterpret_cast<const float4*>(sg.x + a));
                mv[u] = __ldcs(reinterpret_cast<const float4*>(sg.mom + a));
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = i0 + u * RG;
              if (i < n) {
                const float4 d = *reinterpret_cast<const float4*>(slab + i * C + 4 * cq);
                float mh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int kk = 0; kk < R; ++kk) {
                  if (kk < r) {
                    const float p = ph[i * r + kk];
#pragma unroll
                    for (int v = 0; v < 4; ++v) mh[v] = fmaf(p, qv[v][kk], mh[v]);
                  }
                }
                const long long a = base + (long long)i * m + 4 * cq;
                const float4 u4 = make_float4(mh[0], mh[1], mh[2], mh[3]);
                st_stream(reinterpret_cast<float4*>(e + a), make_float4(d.x - mh[0], d.y - mh[1], d.z - mh[2], d.w - mh[3]));
                if (store_mhat) st_stream(reinterpret_cast<float4*>(work + a), u4);
                sgd4(xv[u], mv[u], u4, sg.lr, sg.mu);
                st_stream(reinterpret_cast<float4*>(sg.mom + a), mv[u]);
                st_stream(reinterpret_cast<float4*>(sg.x + a), xv[u]);
              }
            }
          }
        } else {
#pragma unroll 4
        for (int i = rg; i < n; i += RG) {
          const float4 d = *reinterpret_cast<const float4*>(slab + i * C + 4 * cq);
          float mh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int kk = 0; kk < R; ++kk) {
            if (kk < r) {
              const float p = ph[i * r + kk];
#pragma unroll
              for (int v = 0; v < 4; ++v) mh[v] = fmaf(p, qv[v][kk], mh[v]);
            }
          }
          const long long a = base + (long long)i * m + 4 * cq;
          if (vec) {
            st_stream(reinterpret_cast<float4*>(e + a), make_float4(d.x - mh[0], d.y - mh[1], d.z - mh[2], d.w - mh[3]));
            if (store_mhat) st_stream(reinterpret_cast<float4*>(work + a), make_float4(mh[0], mh[1], mh[2], mh[3]));
          } else {
            const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
            for (int v = 0; v < 4; ++v)
              if (col + v < m) {
                st_stream(e + a + v, dv[v] - mh[v]);
                if (store_mhat) st_stream(work + a + v, mh[v]);
                if (fuse) {
                  float xx = sg.x[a + v], mm = sg.mom[a + v];
                  sgd1(xx, mm, mh[v], sg.lr, sg.mu);
                  sg.mom[a + v] = mm;
                  sg.x[a + v] = xx;
                }
              }
          }
        }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (t == 0) {  // last CTA out resets the counters
    // (group 0's thread 0; group 1 may still be draining, but the producer's atomics are done:
    //  it sent both end markers only after its final atomicAdd)
    if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      for (int k = 0; k < gs.n; ++k) gs.ready[gs.list[k]] = 0;  // every producer is done with them
    }
  }
}

// ============================================================================= tall, row-oriented
// k4_rows — the EF pass of tall matrices with m = 2 (mod 4), m <= 1024 and r <= 4
// (LSTM: 28869 x 650, 2600 x 650): e = delta - P-hat q^T (and M-hat at W = 1) of a
// 32-row block (compressors.py:376-378, optimizer.py:124-127).  A CTA streams whole
// rows (contiguous memory, 8-byte pieces — even m keeps every row 8-byte aligned),
// thread t owning the column pairs t and t + 256, so its q values stay in registers.
// (A row-oriented q pass with an ordered two-level partial reduction measured slower
// than k3_slab — 65-70 + 10 us vs 51 us on LSTM — and is not kept.)
constexpr int KR_THREADS = 256;
constexpr int KR_EROWS = 32;  // measured: 32 rows per EF item (LSTM 226 -> 220 us vs 64; sweeps/swer*.txt)
struct RowsItem {
  int mat, r0, nrows, pad;
};

template <int R>
__device__ __forceinline__ void kr_prow(const float* __restrict__ Phat, const MatDev& md, int row, float (&p)[R]) {
  const float* pr = Phat + md.p_off + (long long)row * md.r;
  if constexpr (R == 4) {
    if (md.r == 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(pr));
      p[0] = v.x; p[1] = v.y; p[2] = v.z; p[3] = v.w;
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) p[k] = k < md.r ? __ldg(pr + k) : 0.f;
}

template <int R>
__global__ void __launch_bounds__(KR_THREADS)
    k4_rows(const MatDev* __restrict__ mats, const RowsItem* __restrict__ items, float* __restrict__ work,
            float* __restrict__ e, const float* __restrict__ Phat, const float* __restrict__ qsrc, int write_mhat,
            const int* __restrict__ status) {
  const RowsItem it = items[blockIdx.x];  // plan constants: read before the wait
  const MatDev md = mats[it.mat];
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int m = md.m, r = md.r, np = m >> 1, t = threadIdx.x;
  const bool ok0 = t < np, ok1 = t + KR_THREADS < np;
  float qv[2][2][R];  // q of the thread's four columns
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * (t + h * KR_THREADS);
    const bool okh = h == 0 ? ok0 : ok1;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const float* qk = qsrc + md.q_off + (long long)k * md.qld + c;
      qv[h][0][k] = (okh && k < r) ? __ldg(qk) : 0.f;
      qv[h][1][k] = (okh && k < r) ? __ldg(qk + 1) : 0.f;
    }
  }
  const long long o0 = md.flat_off + (long long)it.r0 * m;
  for (int i0 = 0; i0 < it.nrows; i0 += 8) {
    float2 d0[8], d1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const bool in = i0 + u < it.nrows;
      const float2* row = reinterpret_cast<const float2*>(work + o0 + (long long)(i0 + u) * m);
      d0[u] = (in && ok0) ? __ldcs(row + t) : make_float2(0.f, 0.f);
      d1[u] = (in && ok1) ? __ldcs(row + t + KR_THREADS) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u >= it.nrows) break;
      float p[R];
      kr_prow<R>(Phat, md, it.r0 + i0 + u, p);
      const long long a = o0 + (long long)(i0 + u) * m;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!(h == 0 ? ok0 : ok1)) continue;
        float m0 = 0.f, m1 = 0.f;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          m0 = fmaf(p[k], qv[h][0][k], m0);
          m1 = fmaf(p[k], qv[h][1][k], m1);
        }
        const float2 d = h == 0 ? d0[u] : d1[u];
        const long long ad = a + 2 * (t + h * KR_THREADS);
        __stcs(reinterpret_cast<float2*>(e + ad), make_float2(d.x - m0, d.y - m1));
        if (write_mhat) __stcs(reinterpret_cast<float2*>(work + ad), make_float2(m0, m1));
      }
    }
  }
}

// ============================================================================= tall q pass, row blocks
// k3_rq — q_w = delta^T P-hat (compressors.py:339) of the k4_rows matrices (tall,
// m = 2 mod 4, m <= 1024).  A block of whole rows is one contiguous span of delta,
// so a persistent CTA (1 per SM, 16 consumer warps + 1 producer warp) streams its
// static, contiguous range of row blocks with 1-D bulk TMA (cp.async.bulk) into a
// 4-stage smem ring, the P-hat rows of each block beside it.  Thread (rg, tp) owns
// the column pair tp of the rows rg, rg + RGn, ... and keeps its 2 x r partial q in
// registers; after its last block of a matrix the CTA writes one partial (fixed
// order over the row groups) into the matrix's slot list.  k3_rq_reduce then sums
// the slots in row order (deterministic).  Delta is final when the kernel starts
// (K2 ran after K1), so the ring is filled before griddepcontrol.wait; P-hat is
// fetched after it.  The range is walked backwards: the last rows K1 wrote (still
// in L2) are read first.  For matrices orthogonalised in Gram space the kernel
// stages the rows of P instead, and one warp makes k2_apply's P-hat = (P / W) T
// (float64, stored for K4) a stage ahead of the 15 streaming warps, so q_ef has no
// k2_apply launch.  3 stages (~172 KB): the CTA fits on an SM beside K2's CTAs and
// starts streaming while they run (4 stages: 214 vs 206 us on LSTM, sweeps).
constexpr int RQ_STAGES = 4;      // ring capacity; the plan uses PSGD_RQ_STAGES (default 3: the CTA then fits beside K2's, measured)
constexpr int RQ_STAGE_FLOATS = 12288;  // 48 KB of delta per stage
constexpr int RQ_PST = 512;             // P-hat floats per stage
struct RqChunk {
  long long off;   // flat offset of the block's first element
  long long slot;  // float offset of this CTA's partial of `mat` in the slot workspace
  int mat, row0, nrows, flush;  // flush: the CTA's last block of `mat` in traversal order
  int gidx, pad;  // gidx >= 0: P-hat = (P / W) T from the Gram-space T (k2_apply folded in); -1: staged P-hat
};
struct RqLayout {
  int stages, off_p, off_ph, off_red, off_bar, off_ck, total;
};
constexpr int RQ_MAXCK = 64;  // block descriptors of a CTA staged in smem (more: read from global)

template <int R>
__global__ void __launch_bounds__(kTmaThreads, 1)
    k3_rq(const MatDev* __restrict__ mats, const RqChunk* __restrict__ chunks, const int* __restrict__ cta_beg,
          RqLayout L, const float* __restrict__ work, float* __restrict__ Phat, float* __restrict__ wsq,
          const float* __restrict__ P, const double* __restrict__ wsT, float* __restrict__ bias_out, long long nbias,
          long long bias_off, int divisor, int rev, int dpol, int* status) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* sdb = reinterpret_cast<float*>(smem_raw);
  float* spb = reinterpret_cast<float*>(smem_raw + L.off_p);
  float* phb = reinterpret_cast<float*>(smem_raw + L.off_ph);  // stages x RQ_PST: P-hat rows made from P
  float* red = reinterpret_cast<float*>(smem_raw + L.off_red);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + L.off_bar);
  uint64_t* empty = full + L.stages;
  uint64_t* pready = empty + L.stages;  // the P-hat rows of a stage are ready (transform warp)
  RqChunk* cks = reinterpret_cast<RqChunk*>(smem_raw + L.off_ck);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int cb = cta_beg[blockIdx.x], ce = cta_beg[blockIdx.x + 1], nck = ce - cb;
  // the P-hat rows of a block: (P / W) T when the matrix went through Gram space (and the direct
  // fallback did not write P-hat itself), else K2's P-hat (read after griddepcontrol.wait only)
  auto from_p = [&](const RqChunk& ch) {
    return ch.gidx >= 0 && wsT[(long long)ch.gidx * K2G_TS + K2G_DIRECT] == 0.0;
  };
  if (t == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsWarps);
      mbar_init(&pready[s], 1);
    }
    fence_mbar_init();
  }
  auto chunk_g = [&](int j) { return chunks[rev ? ce - 1 - j : cb + j]; };
  if (nck <= RQ_MAXCK && t < nck) cks[t] = chunk_g(t);  // no dependent global loads per block later
  __syncthreads();
  pdl_trigger();  // the slot reduction may stage in; it waits for this grid
  auto chunk_at = [&](int j) { return nck <= RQ_MAXCK ? cks[j] : chunk_g(j); };

  if (warp == kConsWarps) {  // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = dpol == 0 ? pol_evict_first() : pol_evict_last();
      const uint64_t polp = pol_evict_last();
      auto p_span = [&](const RqChunk& ch, const MatDev& md, long long& a4) {
        const long long pa = md.p_off + (long long)ch.row0 * md.r;
        a4 = pa & ~3LL;
        return (uint32_t)((((pa + (long long)ch.nrows * md.r + 3) & ~3LL) - a4) * 4);
      };
      const int pre = min(nck, L.stages);
      int cur = -1, fcur = -1;
      bool fpc = false;
      MatDev md{};
      auto fp_of = [&](const RqChunk& c) {  // after griddepcontrol.wait only
        if (c.mat != fcur) {
          fcur = c.mat;
          fpc = from_p(c);
        }
        return fpc;
      };
      for (int j = 0; j < nck; ++j) {
        const int s = j % L.stages;
        const uint32_t ph = (j / L.stages) & 1;
        const RqChunk ch = chunk_at(j);
        if (ch.mat != cur) {
          cur = ch.mat;
          md = mats[ch.mat];
        }
        mbar_wait(&empty[s], ph ^ 1);
        const long long a4 = ch.off & ~3LL;
        const long long b4 = (ch.off + (long long)ch.nrows * md.m + 3) & ~3LL;
        const uint32_t bytes = (uint32_t)((b4 - a4) * 4);
        long long pa4;
        const uint32_t pbytes = p_span(ch, md, pa4);
        mbar_expect_tx(&full[s], bytes + pbytes);
        tma_load(sdb + s * RQ_STAGE_FLOATS, work + a4, bytes, &full[s], pol);
        if (j >= pre) tma_load(spb + s * RQ_PST, (fp_of(ch) ? P : Phat) + pa4, pbytes, &full[s], polp);
        if (j == pre - 1) {  // the ring is full of delta: wait for K2's P-hat, then its copies
          pdl_wait();
          for (int j2 = 0; j2 < pre; ++j2) {
            const RqChunk c2 = chunk_at(j2);
            const MatDev m2 = mats[c2.mat];
            long long q4;
            const uint32_t qb = p_span(c2, m2, q4);
            tma_load(spb + j2 * RQ_PST, (fp_of(c2) ? P : Phat) + q4, qb, &full[j2], polp);
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers
  pdl_wait();
  const bool bad = (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) != 0;  // mutate nothing
  if (!bad && nbias > 0) {  // bias mean (optimizer.py:111-113), when this launch is the one to write it
    bool bb = false;
    for (long long x = (long long)blockIdx.x * kCons + t; x < nbias; x += (long long)gridDim.x * kCons) {
      const float v = P[bias_off + x];
      bb |= !finite1(v);
      bias_out[x] = divisor == 1 ? v : v / (float)divisor;
    }
    if (bb) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);
  }
  // warps 0..14 stream the column pairs; warp 15 makes the P-hat rows of each stage (k2_apply's
  // (P / W) T, float64) ahead of them and publishes them on pready
  constexpr int XW = kConsWarps - 1, NCT = kCons - 32;
  float acc[2][R];
#pragma unroll
  for (int k = 0; k < R; ++k) acc[0][k] = acc[1][k] = 0.f;
  int cur = -1;
  bool fpm = false;
  MatDev md{};
  for (int j = 0; j < nck; ++j) {
    const int s = j % L.stages;
    const uint32_t ph = (j / L.stages) & 1;
    const RqChunk ch = chunk_at(j);
    if (ch.mat != cur) {
      cur = ch.mat;
      md = mats[ch.mat];
      fpm = !bad && from_p(ch);
    }
    const int m = md.m, r = md.r, np = m >> 1;
    const int TPR = min(NCT, (np + 31) & ~31), RGn = NCT / TPR;
    const int rg = t / TPR, tp = t - rg * TPR;
    const bool act = warp < XW && rg < RGn && tp < np;
    const long long pa = md.p_off + (long long)ch.row0 * r;
    const float* sp = spb + s * RQ_PST + (int)(pa - (pa & ~3LL));
    const bool fp = fpm;
    mbar_wait(&full[s], ph);
    if (warp == XW) {
      if (fp) {
        const double* T = wsT + (long long)ch.gidx * K2G_TS;
        const double inv_div = 1.0 / (double)divisor;
        for (int li = lane; li < ch.nrows; li += 32) {
          double x[R];
#pragma unroll
          for (int k = 0; k < R; ++k) x[k] = k < r ? (double)sp[li * r + k] * inv_div : 0.0;
          float* dst = Phat + pa + (long long)li * r;
#pragma unroll
          for (int jj = 0; jj < R; ++jj) {
            if (jj < r) {
              double v = 0.0;
#pragma unroll
              for (int k = 0; k <= jj; ++k) v = fma(x[k], T[k * r + jj], v);
              phb[s * RQ_PST + li * r + jj] = (float)v;
              dst[jj] = (float)v;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pready[s]);
    } else {
      mbar_wait(&pready[s], ph);
      if (!bad && act) {
        const float* sd = sdb + s * RQ_STAGE_FLOATS + (int)(ch.off - (ch.off & ~3LL));
        const float* pp = fp ? phb + s * RQ_PST : sp;
        const float2* d2 = reinterpret_cast<const float2*>(sd) + tp;
        int li = rg;
#pragma unroll 2
        for (; li < ch.nrows; li += RGn) {
          const float2 d = d2[(li * m) >> 1];
          const float* pr = pp + li * r;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const float pk = k < r ? pr[k] : 0.f;
            acc[0][k] = fmaf(d.x, pk, acc[0][k]);
            acc[1][k] = fmaf(d.y, pk, acc[1][k]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (ch.flush) {  // the CTA's partial of this matrix: slot (k, c) at slot + k * m + c
      if (!bad) {
        float* slot = wsq + ch.slot;
        if (RGn == 1) {
          if (act)
#pragma unroll
            for (int k = 0; k < R; ++k)
              if (k < r) *reinterpret_cast<float2*>(slot + (long long)k * m + 2 * tp) = make_float2(acc[0][k], acc[1][k]);
        } else {  // fixed order over the row groups
          if (act)
#pragma unroll
            for (int k = 0; k < R; ++k) {
              red[((rg * R + k) * np + tp) * 2] = acc[0][k];
              red[((rg * R + k) * np + tp) * 2 + 1] = acc[1][k];
            }
          bar_consumers();
          for (int o = t; o < np * r; o += kCons) {
            const int k = o / np, c2 = o - k * np;
            float sx = 0.f, sy = 0.f;
            for (int g2 = 0; g2 < RGn; ++g2) {
              sx += red[((g2 * R + k) * np + c2) * 2];
              sy += red[((g2 * R + k) * np + c2) * 2 + 1];
            }
            *reinterpret_cast<float2*>(slot + (long long)k * m + 2 * c2) = make_float2(sx, sy);
          }
          bar_consumers();
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) acc[0][k] = acc[1][k] = 0.f;
    }
  }
}

struct RqMat {
  long long slot0;  // float offset of slot 0 in the workspace (slots of m x r floats, row order)
  int mat, nslots;
};

// q_w of the k3_rq matrices: a CTA owns 32 consecutive outputs; its 8 warps sum the
// slots g, g + 8, g + 16, ... (all loads in flight), then the 8 group sums are added
// in group order (fixed order: deterministic)
constexpr int RQR_GROUPS = 8;
__global__ void __launch_bounds__(32 * RQR_GROUPS)
    k3_rq_reduce(const MatDev* __restrict__ mats, const RqMat* __restrict__ rqm, const int2* __restrict__ blocks,
                 const float* __restrict__ wsq, float* __restrict__ qout, const int* __restrict__ status) {
  __shared__ float part[RQR_GROUPS][32];
  const int2 b = blocks[blockIdx.x];  // plan constants: read before the wait
  const RqMat rm = rqm[b.x];
  const MatDev md = mats[rm.mat];
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int o = b.y + lane;
  const long long mr = (long long)md.m * md.r;
  float s = 0.f;
  if (o < mr) {
    const float* src = wsq + rm.slot0 + o;
    for (int j0 = g; j0 < rm.nslots; j0 += 16 * RQR_GROUPS) {
      float y[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int j = j0 + u * RQR_GROUPS;
        y[u] = j < rm.nslots ? __ldcg(src + (long long)j * mr) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s += y[u];
    }
  }
  part[g][lane] = s;
  __syncthreads();
  if (g == 0 && o < mr) {
    float t = 0.f;
#pragma unroll
    for (int g2 = 0; g2 < RQR_GROUPS; ++g2) t += part[g2][lane];
    const int k = o / md.m, c = o - k * md.m;
    qout[md.q_off + (long long)k * md.qld + c] = t;
  }
}

// K4 / K5 row streaming.  MODE 0 (K4): e = delta - P-hat q^T (+ M-hat in place
// when write_mhat).  MODE 1 (K5): M-hat = P-hat (q / div)^T; items with
// row0 == 0 store Q-bar = q / div.

template <int R, bool EXACT, int MODE>
__global__ void __launch_bounds__(kThreads) k45_rows(const MatDev* __restrict__ mats,
                                                     const RowItem* __restrict__ items, int beg,
                                                     int end, float* __restrict__ work,
                                                     float* __restrict__ e,
                                                     const float* __restrict__ Phat,
                                                     const float* __restrict__ qsrc, int divisor,
                                                     float* __restrict__ qstore, int write_mhat,
                                                     const int* __restrict__ status, SgdArgs sg) {
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const bool fuse = MODE == 1 && sg.x != nullptr;  // K5 with the optimizer update (optimizer.py:131-134)
  if (fuse) sgd_bias(sg, (long long)blockIdx.x * kThreads + threadIdx.x, (long long)gridDim.x * kThreads);
  const bool store = MODE == 0 || !fuse || sg.keep;
  const int lane = threadIdx.x & 31;
  const int wi = beg + blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (wi >= end) return;
  const RowItem it = items[wi];
  const MatDev md = mats[it.mat];
  const int r = EXACT ? R : md.r;
  const int m = md.m;
  const float* __restrict__ Q = qsrc + md.q_off;
  if (MODE == 1 && it.row0 == 0 && qstore != nullptr && qstore != qsrc) {
    for (int x = lane; x < md.qld * r; x += 32) {
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
    for (int k = 0; k < R; ++k)
      ph[k] = (EXACT || k < r) ? __ldg(Phat + md.p_off + (long long)i * r + k) : 0.f;
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
          float qk = __ldg(Q + (long long)k * md.qld + j);
          if (MODE == 1 && divisor != 1) qk = qk / (float)divisor;
          mh = fmaf(ph[k], qk, mh);
        }
      }
      if (MODE == 0) {
        const float d = work[o + j];
        st_stream(e + o + j, d - mh);
        if (write_mhat) st_stream(work + o + j, mh);
      } else {
        if (store) st_stream(work + o + j, mh);
        if (fuse) {
          float xx = sg.x[o + j], mm = sg.mom[o + j];
          sgd1(xx, mm, mh, sg.lr, sg.mu);
          sg.mom[o + j] = mm;
          sg.x[o + j] = xx;
        }
      }
    }
    const float* __restrict__ qrow = Q + head;
    const bool qal = (head & 3) == 0;
    float4* __restrict__ w4 = reinterpret_cast<float4*>(work + o + head);
    float4* __restrict__ e4 = reinterpret_cast<float4*>(e + o + head);
    // 4 float4 per lane per pass: the delta loads are issued together (memory-level parallelism)
    for (int c0 = gl; c0 < body4; c0 += 4 * G) {
      float4 d[4];
      if (MODE == 0) {
#pragma unroll
        for (int v = 0; v < 4; ++v)
          d[v] = c0 + v * G < body4 ? __ldcs(w4 + c0 + v * G) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float4 xs[4], ms[4];
      if (fuse) {
        const float4* x4 = reinterpret_cast<const float4*>(sg.x + o + head);
        const float4* m4 = reinterpret_cast<const float4*>(sg.mom + o + head);
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (c0 + v * G < body4) {
            xs[v] = __ldcs(x4 + c0 + v * G);
            ms[v] = __ldcs(m4 + c0 + v * G);
          }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int c = c0 + v * G;
        if (c >= body4) break;
        float qv[4][R];
        load_q4<R, false>(qrow + 4 * c, md.qld, qal, r, qv);
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
          st_stream(e4 + c, make_float4(d[v].x - mh[0], d[v].y - mh[1], d[v].z - mh[2], d[v].w - mh[3]));
          if (write_mhat) st_stream(w4 + c, make_float4(mh[0], mh[1], mh[2], mh[3]));
        } else {
          const float4 u4 = make_float4(mh[0], mh[1], mh[2], mh[3]);
          if (store) st_stream(w4 + c, u4);
          if (fuse) {
            sgd4(xs[v], ms[v], u4, sg.lr, sg.mu);
            st_stream(reinterpret_cast<float4*>(sg.mom + o + head) + c, ms[v]);
            st_stream(reinterpret_cast<float4*>(sg.x + o + head) + c, xs[v]);
          }
        }
      }
    }
  }
}

// K4 column tiles (tall matrices with m % 4 == 0): a warp owns 128 columns x
// K4T_ROWS rows; its Q block (4 columns x r) sits in registers for the whole
// tile, so per float4 of delta the warp loads only delta and a broadcast P-hat
// row (the row pass above re-reads r float4 of Q per float4 of delta).
constexpr int K4T_ROWS = 64;
struct TileItem {
  int mat, row0, nrows, c0;
};

template <int R, bool EXACT>
__global__ void __launch_bounds__(kThreads) k4_tile(const MatDev* __restrict__ mats, const TileItem* __restrict__ items,
                                                    int beg, int end, float* __restrict__ work, float* __restrict__ e,
                                                    const float* __restrict__ Phat, const float* __restrict__ qsrc,
                                                    int write_mhat, const int* __restrict__ status) {
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int lane = threadIdx.x & 31;
  const int wi = beg + blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (wi >= end) return;
  const TileItem it = items[wi];
  const MatDev md = mats[it.mat];
  const int r = EXACT ? R : md.r;
  const int m = md.m;
  const int col = it.c0 + 4 * lane;
  const bool ok = col < m;
  float qv[4][R];
  if (ok) {
    load_q4<R, false>(qsrc + md.q_off + col, md.qld, true, r, qv);
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int k = 0; k < R; ++k) qv[v][k] = 0.f;
  }
  const float* __restrict__ pr = Phat + md.p_off + (long long)it.row0 * r;
  const long long base = md.flat_off + (long long)it.row0 * m + col;
  for (int i0 = 0; i0 < it.nrows; i0 += 8) {
    float4 d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      d[u] = (ok && i0 + u < it.nrows) ? __ldcs(reinterpret_cast<const float4*>(work + base + (long long)(i0 + u) * m))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (!ok || i0 + u >= it.nrows) break;
      float mh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (EXACT || k < r) {
          const float p = __ldg(pr + (long long)(i0 + u) * r + k);  // one address per warp: broadcast
#pragma unroll
          for (int v = 0; v < 4; ++v) mh[v] = fmaf(p, qv[v][k], mh[v]);
        }
      }
      const long long a = base + (long long)(i0 + u) * m;
      st_stream(reinterpret_cast<float4*>(e + a),
                make_float4(d[u].x - mh[0], d[u].y - mh[1], d[u].z - mh[2], d[u].w - mh[3]));
      if (write_mhat) st_stream(reinterpret_cast<float4*>(work + a), make_float4(mh[0], mh[1], mh[2], mh[3]));
    }
  }
}

// K1 column tiles for matrices whose Q block cannot be staged in shared memory
// (m r > the Q slot, e.g. the 4096 x 4096 rank-8 stress set): a warp owns 128
// columns x K1T_ROWS rows with its Q block (4 columns x r) in registers; per
// batch of 8 rows it loads g and e (16 float4 in flight per lane), stores delta,
// and reduce-scatters the 8 x r row partials across the warp (each lane ends up
// owning V / 32 sums) into a per-column-tile partial buffer; k1_tile_reduce
// sums the tiles in order into P (optimizer.py:120, compressors.py:336).
constexpr int K1T_ROWS = 64;

template <int RM>
__global__ void __launch_bounds__(kThreads) k1_tile(const MatDev* __restrict__ mats, const TileItem* __restrict__ items,
                                                    int nitems, const long long* __restrict__ part_off,
                                                    const float* __restrict__ g, const float* __restrict__ e,
                                                    float* __restrict__ work, const float* __restrict__ Q,
                                                    float* __restrict__ part) {
  constexpr int V = 8 * RM;
  const int lane = threadIdx.x & 31;
  const int wi = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (wi >= nitems) return;
  const TileItem it = items[wi];
  const MatDev md = mats[it.mat];
  const int r = md.r, m = md.m, n = md.n;
  const int col = it.c0 + 4 * lane;
  const bool ok = col < m;
  float qv[4][RM];
  if (ok) {
    load_q4<RM, false>(Q + md.q_off + col, md.qld, true, r, qv);
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int k = 0; k < RM; ++k) qv[v][k] = 0.f;
  }
  const long long base = md.flat_off + (long long)it.row0 * m + col;
  float* __restrict__ pt = part + part_off[it.mat] + (long long)(it.c0 >> 7) * n * r;
  for (int i0 = 0; i0 < it.nrows; i0 += 8) {
    float4 d[8];
    {
      float4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = b[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok && i0 + u < it.nrows) {
          a[u] = __ldcs(reinterpret_cast<const float4*>(g + base + (long long)(i0 + u) * m));
          if (e) b[u] = __ldcs(reinterpret_cast<const float4*>(e + base + (long long)(i0 + u) * m));
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) d[u] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (ok && i0 + u < it.nrows) reinterpret_cast<float4*>(work + base + (long long)(i0 + u) * m)[0] = d[u];
    float v[V];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < RM; ++k) {
        float s2 = d[u].x * qv[0][k];
        s2 = fmaf(d[u].y, qv[1][k], s2);
        s2 = fmaf(d[u].z, qv[2][k], s2);
        v[u * RM + k] = fmaf(d[u].w, qv[3][k], s2);
      }
    int vbase = 0, h = V;  // reduce-scatter over the 32 lanes (fixed order => deterministic)
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int o = 16 >> l;
      if (h > 1) {
        h >>= 1;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < V / 2; ++i)
          if (i < h) {
            const float send = up ? v[i] : v[i + h];
            const float keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        if (up) vbase += h;
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      }
    }
    const bool owner = V >= 32 || (lane & ((32 / V) - 1)) == 0;
#pragma unroll
    for (int i = 0; i < (V >= 32 ? V / 32 : 1); ++i) {
      const int oi = vbase + i, u = oi / RM, k = oi - u * RM;
      if (owner && k < r && i0 + u < it.nrows) pt[(long long)(it.row0 + i0 + u) * r + k] = v[i];
    }
  }
}

// P = sum over the column tiles (in tile order) of the k1_tile partials; a
// non-finite sum (a non-finite g or e poisons its row) raises the plan's last flag
__global__ void __launch_bounds__(256) k1_tile_reduce(const MatDev* __restrict__ mats, const int* __restrict__ list,
                                                      const long long* __restrict__ part_off,
                                                      const float* __restrict__ part, float* __restrict__ P,
                                                      long long flag_slot) {
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  const int mi = list[blockIdx.y];
  const MatDev md = mats[mi];
  const long long nr = (long long)md.n * md.r;
  const int ntiles = (md.m + 127) >> 7;
  const float* src = part + part_off[mi];
  bool bad = false;
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < nr; x += (long long)gridDim.x * blockDim.x) {
    float s2 = 0.f;
    for (int t0 = 0; t0 < ntiles; t0 += 8) {
      float y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) y[u] = t0 + u < ntiles ? __ldcs(src + (long long)(t0 + u) * nr + x) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) s2 += y[u];
    }
    bad |= !finite1(s2);
    P[md.p_off + x] = s2;
  }
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x == 0 && s_bad) P[flag_slot] = 1.f;
}

// K3 column tiles for tall matrices with m % 4 == 0: a warp owns 128 columns x
// K3T_ROWS rows, accumulates q_w = delta^T P-hat for its 4 columns x r in
// registers (P-hat rows are warp-broadcast loads), and writes one partial per
// (row block, column); k3_tile_reduce sums the row blocks in order into q
// (column-major Q layout; compressors.py:339).
constexpr int K3T_ROWS = 256;

template <int RM>
__global__ void __launch_bounds__(kThreads) k3_tile(const MatDev* __restrict__ mats, const TileItem* __restrict__ items,
                                                    int nitems, const long long* __restrict__ part_off,
                                                    const float* __restrict__ work, const float* __restrict__ Phat,
                                                    float* __restrict__ part, const int* __restrict__ status) {
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int lane = threadIdx.x & 31;
  const int wi = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (wi >= nitems) return;
  const TileItem it = items[wi];
  const MatDev md = mats[it.mat];
  const int r = md.r, m = md.m;
  const int col = it.c0 + 4 * lane;
  const bool ok = col < m;
  float qp[4][RM];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < RM; ++k) qp[v][k] = 0.f;
  const float* __restrict__ pr = Phat + md.p_off + (long long)it.row0 * r;
  const long long base = md.flat_off + (long long)it.row0 * m + col;
  for (int i0 = 0; i0 < it.nrows; i0 += 8) {
    float4 d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      d[u] = (ok && i0 + u < it.nrows) ? __ldcs(reinterpret_cast<const float4*>(work + base + (long long)(i0 + u) * m))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u >= it.nrows) break;
      float p[RM];  // the P-hat row: one address per warp (broadcast), float4 when r == RM % 4 == 0
      if (RM % 4 == 0 && r == RM) {
#pragma unroll
        for (int k4 = 0; k4 < RM / 4; ++k4) {
          const float4 pv = __ldg(reinterpret_cast<const float4*>(pr + (long long)(i0 + u) * r) + k4);
          p[4 * k4] = pv.x; p[4 * k4 + 1] = pv.y; p[4 * k4 + 2] = pv.z; p[4 * k4 + 3] = pv.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < RM; ++k) p[k] = k < r ? __ldg(pr + (long long)(i0 + u) * r + k) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < RM; ++k) {
        qp[0][k] = fmaf(d[u].x, p[k], qp[0][k]);
        qp[1][k] = fmaf(d[u].y, p[k], qp[1][k]);
        qp[2][k] = fmaf(d[u].z, p[k], qp[2][k]);
        qp[3][k] = fmaf(d[u].w, p[k], qp[3][k]);
      }
    }
  }
  if (!ok) return;
  // partial layout [row block][k][column] (column-major like Q, ld = m)
  float* pt = part + part_off[it.mat] + (long long)(it.row0 / K3T_ROWS) * r * m;
#pragma unroll
  for (int k = 0; k < RM; ++k)
    if (k < r) *reinterpret_cast<float4*>(pt + (long long)k * m + col) = make_float4(qp[0][k], qp[1][k], qp[2][k], qp[3][k]);
}

__global__ void __launch_bounds__(256) k3_tile_reduce(const MatDev* __restrict__ mats, const int* __restrict__ list,
                                                      const long long* __restrict__ part_off,
                                                      const float* __restrict__ part, float* __restrict__ qout,
                                                      const int* __restrict__ status) {
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int mi = list[blockIdx.y];
  const MatDev md = mats[mi];
  const long long mr = (long long)md.m * md.r;
  const int nblk = (md.n + K3T_ROWS - 1) / K3T_ROWS;
  const float* src = part + part_off[mi];
  for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < mr; x += (long long)gridDim.x * blockDim.x) {
    float s2 = 0.f;
    for (int b0 = 0; b0 < nblk; b0 += 8) {
      float y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) y[u] = b0 + u < nblk ? __ldcs(src + (long long)(b0 + u) * mr + x) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) s2 += y[u];
    }
    const long long k = x / md.m, c = x - k * md.m;
    qout[md.q_off + k * md.qld + c] = s2;
  }
}

// K4 column tiles for m % 4 == 2 (LSTM, m = 650): consecutive rows alternate
// between two 16-byte alignment classes, so even-aligned rows use float4 columns
// c0 + 4l.. and odd-aligned rows c0 + 2 + 4l..; each lane keeps both Q blocks in
// registers.  Columns 0, 1 of odd-aligned rows (tile 0, lane 0) and the last two
// columns of even-aligned rows (last tile) are scalar.
template <int R, bool EXACT>
__global__ void __launch_bounds__(kThreads) k4_tile2(const MatDev* __restrict__ mats, const TileItem* __restrict__ items,
                                                     int beg, int end, float* __restrict__ work, float* __restrict__ e,
                                                     const float* __restrict__ Phat, const float* __restrict__ qsrc,
                                                     int write_mhat, const int* __restrict__ status) {
  pdl_wait();
  pdl_trigger();
  if (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P)) return;
  const int lane = threadIdx.x & 31;
  const int wi = beg + blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (wi >= end) return;
  const TileItem it = items[wi];
  const MatDev md = mats[it.mat];
  const int r = EXACT ? R : md.r;
  const int m = md.m;
  const float* Qm = qsrc + md.q_off;
  auto qcol = [&](int c, int k) { return (c < m && (EXACT || k < r)) ? __ldg(Qm + (long long)k * md.qld + c) : 0.f; };
  const int ce = it.c0 + 4 * lane, co = it.c0 + 2 + 4 * lane;  // first column of the lane's float4, per class
  float qe[4][R], qo[4][R], qx[2][R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      qe[v][k] = qcol(ce + v, k);
      qo[v][k] = qcol(co + v, k);
    }
    qx[0][k] = qcol(0, k);
    qx[1][k] = qcol(1, k);
  }
  const bool lead = it.c0 == 0 && lane == 0;  // scalar columns 0, 1 of odd-aligned rows
  const float* __restrict__ pr = Phat + md.p_off + (long long)it.row0 * r;
  for (int i0 = 0; i0 < it.nrows; i0 += 8) {
    float4 d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      d[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (i0 + u < it.nrows) {
        const long long o = md.flat_off + (long long)(it.row0 + i0 + u) * m;
        const int c = (o & 3) ? co : ce;
        if (c + 3 < m) d[u] = __ldcs(reinterpret_cast<const float4*>(work + o + c));
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u >= it.nrows) break;
      const long long o = md.flat_off + (long long)(it.row0 + i0 + u) * m;
      const bool odd = (o & 3) != 0;
      const int c = odd ? co : ce;
      float p[R];
#pragma unroll
      for (int k = 0; k < R; ++k) p[k] = (EXACT || k < r) ? __ldg(pr + (long long)(i0 + u) * r + k) : 0.f;
      if (c + 3 < m) {
        float mh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int v = 0; v < 4; ++v) mh[v] = fmaf(p[k], odd ? qo[v][k] : qe[v][k], mh[v]);
        st_stream(reinterpret_cast<float4*>(e + o + c),
                  make_float4(d[u].x - mh[0], d[u].y - mh[1], d[u].z - mh[2], d[u].w - mh[3]));
        if (write_mhat) st_stream(reinterpret_cast<float4*>(work + o + c), make_float4(mh[0], mh[1], mh[2], mh[3]));
      } else if (!odd && c < m) {  // last two columns of an even-aligned row
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          float mh = 0.f;
#pragma unroll
          for (int k = 0; k < R; ++k) mh = fmaf(p[k], qe[v][k], mh);
          const float dv = work[o + c + v];
          st_stream(e + o + c + v, dv - mh);
          if (write_mhat) st_stream(work + o + c + v, mh);
        }
      }
      if (odd && lead) {  // columns 0, 1 of an odd-aligned row
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          float mh = 0.f;
#pragma unroll
          for (int k = 0; k < R; ++k) mh = fmaf(p[k], qx[v][k], mh);
          const float dv = work[o + v];
          st_stream(e + o + v, dv - mh);
          if (write_mhat) st_stream(work + o + v, mh);
        }
      }
    }
  }
}

template <int R, bool EXACT>
struct RunK4T2 {
  static int run(const psgd_plan* pl, const Group& gp, float* work, float* e, const float* phat, const float* q,
                 int write_mhat, const int* status, cudaStream_t st);
};

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

// ============================================================================= optimizer
// optimizer.py:131-134 for every parameter in one pass over the packed buffers:
// m = momentum * m + u ; x -= lr * (u + m).  u is M-hat (work) / the bias mean.
// 20 B per element (read u, m, x; write m, x), HBM-bound, float4 streaming.
__global__ void __launch_bounds__(256) k_momentum(float* __restrict__ x, float* __restrict__ mom,
                                                  const float* __restrict__ u, long long n4, float lr,
                                                  float momentum, float* __restrict__ bx, float* __restrict__ bm,
                                                  const float* __restrict__ bu, long long nb,
                                                  const int* __restrict__ status) {
  // a failed step (non-finite gradient / P) leaves x and m untouched, like the
  // reference, which raises before optimizer.py:131-134 runs
  if (status && (*status & (PSGD_STATUS_NONFINITE_GRAD | PSGD_STATUS_NONFINITE_P))) return;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 uu = __ldcs(reinterpret_cast<const float4*>(u) + i);
    float4 mm = __ldcs(reinterpret_cast<const float4*>(mom) + i);
    float4 xx = __ldcs(reinterpret_cast<const float4*>(x) + i);
    mm.x = fmaf(momentum, mm.x, uu.x); mm.y = fmaf(momentum, mm.y, uu.y);
    mm.z = fmaf(momentum, mm.z, uu.z); mm.w = fmaf(momentum, mm.w, uu.w);
    xx.x -= lr * (uu.x + mm.x); xx.y -= lr * (uu.y + mm.y);
    xx.z -= lr * (uu.z + mm.z); xx.w -= lr * (uu.w + mm.w);
    __stcs(reinterpret_cast<float4*>(mom) + i, mm);
    __stcs(reinterpret_cast<float4*>(x) + i, xx);
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += stride) {
    const float m2 = fmaf(momentum, bm[i], bu[i]);
    bm[i] = m2;
    bx[i] -= lr * (bu[i] + m2);
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

int rmax_of(int r) { return r <= 1 ? 1 : r <= 2 ? 2 : r <= 4 ? 4 : r <= 8 ? 8 : 16; }

}  // namespace

// ============================================================================= plan

struct psgd_plan {
  int nmat = 0, rank = 0, world = 1, device = 0, nsm = 148;
  long long nbias = 0, flat_elems = 0, p_elems = 0, p_bias_off = 0, flag_off = 0, q_elems = 0,
            repl_elems = 0;
  int nflags = 0;
  int rmax = 1;
  std::vector<MatDev> mats;
  // K1
  std::vector<Chunk1> k1;
  std::vector<int> k1_beg;
  K1Layout k1l{};
  std::vector<SplitRow> splits;
  long long psplit_elems = 0;
  // K3 fused
  int k2_smem = 0;
  std::vector<int> small_list, gram_list;   // K2 in smem / in Gram space
  std::vector<int> wlist, clist;             // K2 small: warp items / CTA items
  std::vector<int> wlist3, clist3;           // the same without the matrices k3_pipe orthogonalises
  std::vector<int> gs3_list;                 // matrices orthogonalised inside k3_pipe (psgd_q_ef)
  int *d_small_list3 = nullptr, *d_gs3_list = nullptr, *d_gs3_ready = nullptr;
  int k2_wregion = 0, k2_wblocks = 0;
  std::vector<GramItem> gram_items;
  std::vector<int> apply_mat, apply_row0;   // k2_apply blocks
  std::vector<int> apply_mat_q, apply_row0_q;  // the same without k3_rq's matrices (psgd_q_ef)
  int *d_apply_mat_q = nullptr, *d_apply_row0_q = nullptr;
  long long wsg_elems = 0;
  std::vector<SlabItem> k3;          // fused and tall slabs, grouped by r
  std::vector<Group> g3;
  // K3 pipeline (k3_pipe): slab items, the matrices with a tensor map (map order), layout
  std::vector<PipeItem> pipe_items;
  std::vector<int> pipe_maps, pipe_mapC;
  K3PLayout k3pl{}, k3pl_f{};  // k3pl_f: the layout of the fused-optimizer launch
  int pipe_rmax = 1;
  PipeItem* d_pipe_items = nullptr;
  int* d_pipe_ctr = nullptr;
  mutable std::mutex map_mu;               // tensor maps encode the work buffer's address:
  mutable const float* maps_for = nullptr;  // re-encoded when a call passes another buffer
  mutable K3Maps maps{};

  // tall path
  struct RowsGroup {  // one k4_rows launch per R
    int R, ebeg, eend;
  };
  std::vector<RowsItem> kr_e;
  std::vector<RowsGroup> gkr;
  RowsItem* d_kr_e = nullptr;
  // k3_rq (q pass of the k4_rows matrices): row blocks, CTA ranges, slot lists, reduce blocks
  std::vector<RqChunk> rq;
  std::vector<int> rq_beg;
  std::vector<RqMat> rq_mats;
  std::vector<int2> rq_blocks;
  RqLayout rql{};
  int rq_rmax = 1, rq_rev = 1;
  std::vector<char> rq_on;  // per matrix: q pass by k3_rq
  long long rq_ws_elems = 0;
  RqChunk* d_rq = nullptr;
  int* d_rq_beg = nullptr;
  RqMat* d_rq_mats = nullptr;
  int2* d_rq_blocks = nullptr;
  float* d_rq_ws = nullptr;
  std::vector<int> tall_list, all_list;
  std::vector<RowItem> k4, k5;
  std::vector<Group> g4, g5;
  std::vector<TileItem> k4t;   // K4 column tiles (tall, m % 4 == 0)
  std::vector<Group> g4t, g4t2;
  TileItem* d_k4t = nullptr;
  // K1 column tiles (matrices whose Q block is not staged): items, matrix list, partials
  std::vector<TileItem> k1t;
  std::vector<int> k1t_list;
  std::vector<long long> k1t_off;  // per matrix (all matrices, -1 unused)
  long long k1t_part_elems = 0;
  TileItem* d_k1t = nullptr;
  int* d_k1t_list = nullptr;
  long long* d_k1t_off = nullptr;
  float* d_k1t_part = nullptr;
  // K3 column tiles (tall, m % 4 == 0): q partials per 256-row block
  std::vector<TileItem> k3t;
  std::vector<int> k3t_list;
  std::vector<long long> k3t_off;
  long long k3t_part_elems = 0;
  TileItem* d_k3t = nullptr;
  int* d_k3t_list = nullptr;
  long long* d_k3t_off = nullptr;
  float* d_k3t_part = nullptr;
  int n_tall = 0, n_tall_slabs = 0;
  long long wsq_elems = 0;
  // device
  void* dev_block = nullptr;
  MatDev* d_mats = nullptr;
  Chunk1* d_k1 = nullptr;
  int* d_k1_beg = nullptr;
  SplitRow* d_splits = nullptr;
  float* d_psplit = nullptr;
  int* d_split_cnt = nullptr;
  SlabItem* d_k3 = nullptr;
  int *d_tall_list = nullptr, *d_all_list = nullptr, *d_small_list = nullptr, *d_gram_list = nullptr;
  GramItem* d_gram_items = nullptr;
  int *d_apply_mat = nullptr, *d_apply_row0 = nullptr;
  double *d_wsg = nullptr, *d_wsT = nullptr;
  int *d_gs_flag = nullptr, *d_gs_done = nullptr, *d_gs_cnt = nullptr, *d_k1_done = nullptr;
  int* d_gram_cnt = nullptr;
  RowItem *d_k4 = nullptr, *d_k5 = nullptr;
  double* d_gsws = nullptr;  // float64 scratch in the P layout (direct MGS fallback of k2_gram)
  float* d_wsq = nullptr;
  int* d_counters = nullptr;
};

namespace {

long long align4(long long x) { return (x + 3) & ~3LL; }

int lanes_log2_for(int m, int max_lg) {
  const long long per = (m + 15) / 16;  // ~4 float4 per lane per row
  int lg = 2;
  while ((1LL << lg) < per && lg < max_lg) ++lg;
  return lg;
}

bool k3_tileable(const MatDev& md) {
  static const bool off = getenv("PSGD_K3_TILE") && getenv("PSGD_K3_TILE")[0] == '0';
  return !off && md.tall && md.m % 4 == 0 && md.flat_off % 4 == 0 && md.m >= 128;
}

bool k4_tileable(const MatDev& md) {
  static const bool off = getenv("PSGD_K4_TILE") && getenv("PSGD_K4_TILE")[0] == '0';
  return !off && md.tall && md.m % 4 == 0 && md.flat_off % 4 == 0 && md.m >= 128;
}

bool k4_tileable2(const MatDev& md) {  // two alignment classes (k4_tile2)
  static const bool off = getenv("PSGD_K4_TILE2") && getenv("PSGD_K4_TILE2")[0] == '0';
  return !off && md.tall == 1 && md.m % 4 == 2 && md.flat_off % 4 == 0 && md.m >= 128;
}

void build_tile_items(const std::vector<MatDev>& mats, std::vector<TileItem>& items, std::vector<Group>& groups) {
  std::vector<int> rs;
  for (auto& md : mats)
    if (k4_tileable(md) && std::find(rs.begin(), rs.end(), md.r) == rs.end()) rs.push_back(md.r);
  for (int r : rs) {
    Group gp{r, (int)items.size(), 0, 0, 0};
    for (int mi = 0; mi < (int)mats.size(); ++mi) {
      const MatDev& md = mats[mi];
      if (md.r != r || !k4_tileable(md)) continue;
      for (int r0 = 0; r0 < md.n; r0 += K4T_ROWS)
        for (int c0 = 0; c0 < md.m; c0 += 128) items.push_back({mi, r0, std::min(K4T_ROWS, md.n - r0), c0});
    }
    gp.end = (int)items.size();
    groups.push_back(gp);
  }
}

void build_row_items(const std::vector<MatDev>& mats, bool tall_only, std::vector<RowItem>& items,
                     std::vector<Group>& groups) {
  std::vector<int> rs;
  for (auto& md : mats)
    if (!tall_only || md.tall)
      if (std::find(rs.begin(), rs.end(), md.r) == rs.end()) rs.push_back(md.r);
  for (int r : rs) {
    Group gp{r, (int)items.size(), 0, 0};
    for (int mi = 0; mi < (int)mats.size(); ++mi) {
      const MatDev& md = mats[mi];
      if (md.r != r || (tall_only && md.tall != 1)) continue;
      if (tall_only && (k4_tileable(md) || k4_tileable2(md))) continue;  // K4 column tiles instead
      const int lg = lanes_log2_for(md.m, 5);
      const int rpp = 32 >> lg;
      int rows = std::max(1, kRowItemElems / md.m);
      rows = ((rows + rpp - 1) / rpp) * rpp;
      for (int r0 = 0; r0 < md.n; r0 += rows) items.push_back({mi, r0, std::min(rows, md.n - r0), lg});
    }
    gp.end = (int)items.size();
    groups.push_back(gp);
  }
}

// contiguous ranges of items with ~equal weight, one per CTA
std::vector<int> balance(const std::vector<double>& w, int ctas) {
  const int n = (int)w.size();
  std::vector<int> beg(1, 0);
  if (n == 0) {
    beg.push_back(0);
    return beg;
  }
  ctas = std::max(1, std::min(ctas, n));
  double total = 0;
  for (double x : w) total += x;
  double acc = 0;
  int b = 1;
  for (int i = 0; i < n && b < ctas; ++i) {
    acc += w[i];
    if (acc >= total * b / ctas && i + 1 < n) {
      beg.push_back(i + 1);
      ++b;
    }
  }
  beg.push_back(n);
  return beg;
}

struct K3Cfg {
  int vec, cql, rows_chunk, nchunks;
};

// tall-path geometry (register slab): RG * smax rows per chunk
K3Cfg k3_tall_config(int n, int m, int r) {
  const int vec = (m % 4 == 0) ? 4 : 1;
  const int smax = k3_dcap(r) / vec;
  int cql = vec == 4 ? 3 : 5;
  while (cql < 8) {
    const int cq2 = 1 << (cql + 1);
    const int rg2 = kThreads / cq2;
    if ((long long)rg2 * smax < n) break;
    if ((long long)(cq2 / 2) * vec >= m) break;
    if (r > 8 && cq2 * vec > 256) break;
    ++cql;
  }
  const int RG = kThreads >> cql;
  const int rows_chunk = RG * smax;
  return {vec, cql, rows_chunk, (n + rows_chunk - 1) / rows_chunk};
}

}  // namespace

namespace {
bool opt_fusable(const psgd_plan* pl);
}

extern "C" {

int32_t psgd_version(void) { return 3; }

#ifdef PSGD_K1_TIMES
int psgd_debug_k1_times(unsigned long long* out, int n) {  // diagnostic builds (tools/k1_tail.py) only
  return cudaMemcpyFromSymbol(out, g_k1_times, sizeof(unsigned long long) * 3 * std::min(n, 1024)) == cudaSuccess
             ? 0 : -2;
}
#endif

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
  if (cudaDeviceGetAttribute(&pl->nsm, cudaDevAttrMultiProcessorCount, pl->device) != cudaSuccess || pl->nsm <= 0)
    pl->nsm = 148;
  cudaGetLastError();
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
    md.pipe = (md.n <= kFusedNMax && md.r <= 8) ? 1 : 0;  // k3_pipe: q, EF and M-hat from one staged slab
    md.tall = !md.pipe && k3_tall_config(md.n, md.m, md.r).nchunks > 1;
    md.lg1 = 5;  // set with the K1 chunk geometry below
    md.qs = 0;  // decided below, once the K1 smem budget is known
    md.flat_off = fo;
    md.p_off = po;
    md.q_off = qo;
    md.qld = (int)align4(md.m);
    fo = align4(fo + (long long)md.n * md.m);
    po = align4(po + (long long)md.n * md.r);
    qo += (long long)md.r * md.qld;
    pl->n_tall += md.tall;
    pl->rmax = std::max(pl->rmax, rmax_of(md.r));
    pl->all_list.push_back(i);
    if (md.tall) pl->tall_list.push_back(i);
    pl->mats.push_back(md);
  }
  pl->flat_elems = std::max(4LL, fo);
  {  // the row-oriented EF pass (k4_rows) for tall matrices with m = 2 (mod 4), m <= 1024, r <= 4 (LSTM)
    static const bool off = getenv("PSGD_ROWS2") && getenv("PSGD_ROWS2")[0] == '0';
    for (auto& md : pl->mats)
      if (!off && md.tall && md.m % 4 == 2 && md.m <= 4 * KR_THREADS && md.r <= 4) md.tall = 2;
    for (int R : {1, 2, 4}) {
      psgd_plan::RowsGroup gp{R, (int)pl->kr_e.size(), 0};
      for (int mi = 0; mi < nmat; ++mi) {
        const MatDev& md = pl->mats[mi];
        if (md.tall != 2 || rmax_of(md.r) != R) continue;
        for (int r0 = 0; r0 < md.n; r0 += KR_EROWS) pl->kr_e.push_back({mi, r0, std::min(KR_EROWS, md.n - r0), 0});
      }
      gp.eend = (int)pl->kr_e.size();
      if (gp.eend > gp.ebeg) pl->gkr.push_back(gp);
    }
  }
  {  // k3_rq: the q pass of the k4_rows matrices, row blocks by bulk TMA (PSGD_K3RQ=0: k3_slab instead)
    static const bool off = getenv("PSGD_K3RQ") && getenv("PSGD_K3RQ")[0] == '0';
    static const bool rev = !(getenv("PSGD_RQ_REV") && getenv("PSGD_RQ_REV")[0] == '0');
    pl->rq_rev = rev ? 1 : 0;
    pl->rq_on.assign(std::max(1, nmat), 0);
    std::vector<double> w;
    for (int mi = 0; mi < nmat && !off; ++mi) {
      const MatDev& md = pl->mats[mi];
      if (md.tall != 2 || md.flat_off % 4 != 0 || md.m % 2 != 0 || md.m > 2 * (kCons - 32)) continue;
      const int rows = std::max(1, std::min((RQ_STAGE_FLOATS - 8) / md.m, (RQ_PST - 8) / md.r));
      for (int r0 = 0; r0 < md.n; r0 += rows) {
        const int nr = std::min(rows, md.n - r0);
        pl->rq.push_back({md.flat_off + (long long)r0 * md.m, 0, mi, r0, nr, 0, -1, 0});
        w.push_back((double)nr * md.m);
      }
      pl->rq_on[mi] = 1;
      pl->rq_rmax = std::max(pl->rq_rmax, rmax_of(md.r));
    }
    if (!pl->rq.empty()) {
      pl->rq_beg = balance(w, pl->nsm);
      const int nct = (int)pl->rq_beg.size() - 1;
      std::vector<int> nslots(nmat, 0), sidx(pl->rq.size(), 0);
      for (int b = 0; b < nct; ++b)
        for (int k = pl->rq_beg[b]; k < pl->rq_beg[b + 1]; ++k) {
          const bool first = k == pl->rq_beg[b] || pl->rq[k - 1].mat != pl->rq[k].mat;
          const bool last = k + 1 == pl->rq_beg[b + 1] || pl->rq[k + 1].mat != pl->rq[k].mat;
          sidx[k] = first ? nslots[pl->rq[k].mat]++ : sidx[k - 1];
          pl->rq[k].flush = rev ? first : last;  // the run's last block in traversal order
        }
      std::vector<long long> slot0(nmat, 0);
      for (int mi = 0; mi < nmat; ++mi) {
        if (!nslots[mi]) continue;
        const MatDev& md = pl->mats[mi];
        slot0[mi] = pl->rq_ws_elems;
        pl->rq_ws_elems += (long long)nslots[mi] * md.m * md.r;
        const int ri = (int)pl->rq_mats.size();
        pl->rq_mats.push_back({slot0[mi], mi, nslots[mi]});
        for (int e0 = 0; e0 < md.m * md.r; e0 += 32) pl->rq_blocks.push_back(make_int2(ri, e0));
      }
      for (size_t k = 0; k < pl->rq.size(); ++k) {
        const MatDev& md = pl->mats[pl->rq[k].mat];
        pl->rq[k].slot = slot0[pl->rq[k].mat] + (long long)sidx[k] * md.m * md.r;
      }
      {  // K4 (k4_rows) items in the order the q pass left delta in L2: k3_rq walked every CTA range
         // backwards, so the starts of the ranges were read last — interleave the ranges, starts first
        static const bool k4o_off = getenv("PSGD_K4_ORDER") && getenv("PSGD_K4_ORDER")[0] == '0';
        std::vector<int> rng_of(pl->rq.size());
        std::vector<long long> pos_of(pl->rq.size());
        for (int b2 = 0; b2 < nct; ++b2) {
          long long acc = 0;
          for (int k = pl->rq_beg[b2]; k < pl->rq_beg[b2 + 1]; ++k) {
            rng_of[k] = b2;
            pos_of[k] = acc;
            acc += pl->rq[k].nrows;
          }
        }
        std::map<std::pair<int, int>, int> chunk_at_row;  // (mat, row0) of each block
        for (size_t k = 0; k < pl->rq.size(); ++k) chunk_at_row[{pl->rq[k].mat, pl->rq[k].row0}] = (int)k;
        for (auto& gp : pl->gkr) {
          if (k4o_off || !rev) break;
          std::vector<std::pair<std::pair<long long, int>, RowsItem>> keyed;
          bool all = true;
          for (int x = gp.ebeg; x < gp.eend; ++x) {
            const RowsItem& it = pl->kr_e[x];
            auto f = chunk_at_row.upper_bound({it.mat, it.r0});
            if (f == chunk_at_row.begin() || (--f)->first.first != it.mat) { all = false; break; }
            const int k = f->second;
            keyed.push_back({{pos_of[k] + (it.r0 - pl->rq[k].row0), rng_of[k]}, it});
          }
          if (!all) continue;
          std::stable_sort(keyed.begin(), keyed.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
          for (int x = gp.ebeg; x < gp.eend; ++x) pl->kr_e[x] = keyed[x - gp.ebeg].second;
        }
      }
      RqLayout& L = pl->rql;
      static const int nst = getenv("PSGD_RQ_STAGES") ? atoi(getenv("PSGD_RQ_STAGES")) : 3;
      for (L.stages = std::max(2, std::min(RQ_STAGES, nst));; --L.stages) {
        L.off_p = L.stages * RQ_STAGE_FLOATS * 4;
        L.off_ph = L.off_p + L.stages * RQ_PST * 4;
        L.off_red = L.off_ph + L.stages * RQ_PST * 4;
        L.off_bar = (L.off_red + kCons * 2 * pl->rq_rmax * 4 + 15) & ~15;
        L.off_ck = (L.off_bar + 3 * L.stages * 8 + 15) & ~15;
        L.total = L.off_ck + RQ_MAXCK * (int)sizeof(RqChunk) + 16;
        if (L.total <= 232448 - 1024 || L.stages == 2) break;  // 227 KB - static smem
      }
    }
  }
  {  // replacement columns depend on (n, j, attempt) only (linalg.py:54-58): one table per distinct n
    std::map<int, int> cols;
    for (auto& md : pl->mats) cols[md.n] = std::max(cols[md.n], md.r);
    std::map<int, long long> off;
    for (auto& kv : cols) {
      off[kv.first] = ro;
      ro += (long long)PSGD_REPL_ATTEMPTS * kv.second * kv.first;
    }
    for (auto& md : pl->mats) {
      md.repl_off = off[md.n];
      md.rcols = cols[md.n];
    }
  }

  // ---- K1 smem layout: Q slots for the matrices whose r x q_ld block fits, then
  // the largest 2-stage ring of g / e chunks that fits beside them (227 KB)
  {
    K1Layout& L = pl->k1l;
    const long long red_b = 2LL * (K1_RED_ROWS * kConsWarps * pl->rmax + pl->rmax) * 4;
    const long long bar_b = (2 * K1_STAGES + 4) * 8 + 16;
    const long long min_stage = 2LL * 2 * (K1_CHUNK + 8) * 4;  // 2 stages of the smallest chunk
    static const long long qcap = getenv("PSGD_K1_QCAP") ? atoll(getenv("PSGD_K1_QCAP")) : K1_QSLOT_CAP;
    const long long cap = std::min<long long>(qcap, ((227LL * 1024 - min_stage - red_b - bar_b - 512) / 8) & ~3LL);
    // one large slot (up to 128 KB) when some Q does not fit a double-buffered slot:
    // Q read from smem beats Q read through L1/L2 per element (stress: 4096 x 8)
    const long long cap1 = std::min<long long>(K1_QBIG_CAP, ((227LL * 1024 - min_stage - red_b - bar_b - 512) / 4) & ~3LL);
    // one large Q slot when a Q block exceeds the double-buffered slot but not 18432
    // floats (ResNet-18 r = 4: 90 vs 95 us); larger blocks (stress) go to the K1 column
    // tiles, which beat a single 128 KB slot there (9.9 vs 22 ms).  PSGD_K1_BIGQ=0/1 forces.
    const char* bq = getenv("PSGD_K1_BIGQ");
    bool big = false;
    for (auto& md : pl->mats) {
      const long long qb = (long long)md.r * md.qld;
      big |= qb > cap && qb <= K1_QBIG_CAP;
    }
    if (bq) big = bq[0] == '1';
    L.nq = big ? 1 : 2;
    long long qslot = 4;
    for (auto& md : pl->mats) {
      md.qs = (long long)md.r * md.qld <= (big ? cap1 : cap) ? 1 : 0;
      if (md.qs) qslot = std::max(qslot, (long long)md.r * md.qld);
    }
    L.qslot_floats = (int)qslot;
    static const bool qsh_off = getenv("PSGD_K1_QSHIFT") && getenv("PSGD_K1_QSHIFT")[0] == '0';
    L.qshift = 0;
    for (auto& md : pl->mats) L.qshift |= (!qsh_off && md.qs && (md.m & 3) == 2 && md.m >= 64) ? 1 : 0;
    if (qslot > 4096) L.qshift = 0;  // the copies must stay small beside the ring (LSTM: 4 x 652 floats)
    const int qcopies = L.qshift ? 2 : 1;
    static const int nst = getenv("PSGD_K1_NST") ? atoi(getenv("PSGD_K1_NST")) : 2;
    L.stages = std::max(2, std::min(K1_STAGES, nst));
    const long long room = 227LL * 1024 - qcopies * L.nq * qslot * 4 - red_b - bar_b - 512;
    L.stage_floats = (int)std::min<long long>(16384 + 8, (room / (2LL * L.stages * 4)) & ~3LL);
    int off = 2 * L.stages * L.stage_floats * 4;
    L.off_q = off;   off += qcopies * L.nq * L.qslot_floats * 4;
    L.off_red = off; off += (int)red_b;
    off = (off + 15) & ~15;
    L.off_bar = off; off += (int)bar_b;
    L.total = off;
  }
  // ---- K1 chunks: whole rows, <= stage_floats - 8 floats; 2^lg1 lanes per row so
  // that a pass keeps all 16 consumer warps busy (rows <= 32 lanes need no barrier)
  const int seg = pl->k1l.stage_floats - 8;
  pl->k1t_off.assign(std::max(1, nmat), 0);
  for (int mi = 0; mi < nmat; ++mi) {
    MatDev& md = pl->mats[mi];
    static const bool k1t_off_env = getenv("PSGD_K1_TILE") && getenv("PSGD_K1_TILE")[0] == '0';
    if (!k1t_off_env && !md.qs && md.m % 4 == 0 && md.flat_off % 4 == 0 && md.m >= 128) {
      // K1 column tiles: Q stays in registers per warp tile (k1_tile + k1_tile_reduce)
      pl->k1t_list.push_back(mi);
      pl->k1t_off[mi] = pl->k1t_part_elems;
      pl->k1t_part_elems += (long long)((md.m + 127) / 128) * md.n * md.r;
      for (int r0 = 0; r0 < md.n; r0 += K1T_ROWS)
        for (int c0 = 0; c0 < md.m; c0 += 128) pl->k1t.push_back({mi, r0, std::min(K1T_ROWS, md.n - r0), c0});
      md.nck = 0;
      continue;
    }
    if (md.m <= seg) {
      const int rows_fit = seg / md.m;
      int lg = 2;  // ~4 float4 per lane per row, 4..32 lanes
      while ((1 << lg) < (md.m + 15) / 16 && lg < 5) ++lg;
      int rows;
      static const bool partial = getenv("PSGD_K1_PARTIAL") && getenv("PSGD_K1_PARTIAL")[0] == '1';
      if (partial && rows_fit < (kCons >> lg)) {  // experiment: a partial pass (idle warps), no multi-warp rows
        rows = rows_fit;
      } else if (rows_fit >= (kCons >> lg)) {
        rows = (rows_fit / (kCons >> lg)) * (kCons >> lg);
      } else {  // fewer rows than a pass: multi-warp rows, one reduction barrier per chunk
        int p2 = 1;
        while (p2 * 2 <= rows_fit) p2 *= 2;
        lg = 0;
        while ((1 << lg) < kCons / p2) ++lg;
        rows = p2;
      }
      md.lg1 = lg;
      for (int r0 = 0; r0 < md.n; r0 += rows) {
        const int nr = std::min(rows, md.n - r0);
        pl->k1.push_back({md.flat_off + (long long)r0 * md.m, mi, r0, nr, 0, md.m, -1, 0, 0});
      }
    } else {
      md.lg1 = 9;
      const int parts = (md.m + seg - 1) / seg;
      const int slen = (int)align4((md.m + parts - 1) / parts);  // equal segments
      for (int row = 0; row < md.n; ++row) {
        const int sid = (int)pl->splits.size();
        pl->splits.push_back({mi, row, (int)(pl->psplit_elems / md.r), parts});
        pl->psplit_elems += (long long)parts * md.r;
        for (int p = 0; p < parts; ++p) {
          const int c0 = p * slen;
          const int nc = std::min(slen, md.m - c0);
          pl->k1.push_back({md.flat_off + (long long)row * md.m + c0, mi, row, 1, c0, nc, sid, p, 0});
        }
      }
    }
  }
  for (auto& c : pl->k1) pl->mats[c.mat].nck++;
  {
    std::vector<double> w;
    for (auto& c : pl->k1) w.push_back((double)c.nrows * c.ncols + 2048.0);  // + per-chunk overhead
    pl->k1_beg = balance(w, pl->nsm);
  }
  pl->nflags = std::max(1, (int)pl->k1_beg.size() - 1) + (pl->k1t.empty() ? 0 : 1);  // + k1_tile_reduce's slot
  pl->p_bias_off = po;
  pl->flag_off = align4(po + nbias);
  pl->p_elems = pl->flag_off + align4(pl->nflags);
  pl->q_elems = std::max(4LL, qo);
  pl->repl_elems = std::max(1LL, ro);

  for (int mi = 0; mi < nmat; ++mi) {
    const MatDev& md = pl->mats[mi];
    if ((long long)md.n * md.r <= K2_WARP_DOUBLES) {
      pl->wlist.push_back(mi);
      pl->small_list.push_back(mi);
      pl->k2_wregion = std::max(pl->k2_wregion, (int)align4((long long)md.n * md.r));
    } else if ((long long)md.n * md.r <= K2_SMEM_DOUBLES && md.n <= 1024) {  // taller: Gram space
      pl->clist.push_back(mi);
      pl->small_list.push_back(mi);
      pl->k2_smem = std::max(pl->k2_smem, md.n * md.r * 8);
    } else {
      const int gidx = (int)pl->gram_list.size();
      pl->gram_list.push_back(mi);
      static const int grows = getenv("PSGD_K2G_ROWS") ? std::max(64, atoi(getenv("PSGD_K2G_ROWS"))) : K2G_ROWS;
      const int nblk = (md.n + grows - 1) / grows;
      const int npairs = md.r * (md.r + 1) / 2;
      for (int b2 = 0; b2 < nblk; ++b2)
        pl->gram_items.push_back({mi, b2 * grows, std::min(grows, md.n - b2 * grows), b2, nblk, gidx,
                                  pl->wsg_elems});
      pl->wsg_elems += (long long)nblk * npairs;
      for (int r0 = 0; r0 < md.n; r0 += 256) {
        pl->apply_mat.push_back(gidx);
        pl->apply_row0.push_back(r0);
      }
    }
  }
  {  // k3_rq makes the P-hat of its Gram-space matrices itself: q_ef's k2_apply skips them
    static const bool off = getenv("PSGD_RQ_APPLY") && getenv("PSGD_RQ_APPLY")[0] == '0';
    for (auto& ch : pl->rq) {
      const auto it = std::find(pl->gram_list.begin(), pl->gram_list.end(), ch.mat);
      ch.gidx = (off || it == pl->gram_list.end()) ? -1 : (int)(it - pl->gram_list.begin());
    }
    for (size_t b2 = 0; b2 < pl->apply_mat.size(); ++b2) {
      const int mi = pl->gram_list[pl->apply_mat[b2]];
      if (!off && mi < (int)pl->rq_on.size() && pl->rq_on[mi]) continue;
      pl->apply_mat_q.push_back(pl->apply_mat[b2]);
      pl->apply_row0_q.push_back(pl->apply_row0[b2]);
    }
  }
  pl->k2_wblocks = ((int)pl->wlist.size() + K2_THREADS / 32 - 1) / (K2_THREADS / 32);
  {  // the warp items need smem only when one is beyond the register MGS (n > 512 or r > 4): with no
     // dynamic smem K2's CTAs fit beside K1's on an SM and wait there (PDL) instead of launching late
    bool smem_warp = false;
    for (int mi : pl->wlist) smem_warp |= pl->mats[mi].n > 512 || pl->mats[mi].r > 4;
    if (smem_warp) pl->k2_smem = std::max(pl->k2_smem, pl->k2_wregion * (K2_THREADS / 32) * 8);
  }
  // ---- K3 slabs, grouped by r (one launch per group): fused slabs hold all rows
  {
    std::vector<int> rs;
    for (auto& md : pl->mats)
      if (std::find(rs.begin(), rs.end(), md.r) == rs.end()) rs.push_back(md.r);
    for (int r : rs) for (int tall = 0; tall < 2; ++tall) {
      Group gp{r, (int)pl->k3.size(), 0, 0, tall};
      for (int mi = 0; mi < nmat; ++mi) {
        const MatDev& md = pl->mats[mi];
        if (md.r != r || md.pipe) continue;
        const K3Cfg cf = k3_tall_config(md.n, md.m, r);
        if ((cf.nchunks > 1) != (tall == 1)) continue;
        if (tall && k3_tileable(md)) continue;  // K3 column tiles instead
        if (tall && pl->rq_on[mi]) continue;    // k3_rq row blocks instead
        const int CQ = 1 << cf.cql, C = CQ * cf.vec, RG = kThreads / CQ;
        const int nslab = (md.m + C - 1) / C;
        for (int s = 0; s < nslab; ++s) {
          int slab_id = -1;
          long long wo = 0;
          // tall: ~PSGD_K3_SUBROWS rows per CTA, q accumulated in registers
          // (measured: 2048 rows for float4 slabs (stress 4096 x 4096), one register slab for
          // scalar-column slabs (LSTM, m % 4 != 0) where the extra loop only adds latency)
          static const int sub_rows = getenv("PSGD_K3_SUBROWS") ? atoi(getenv("PSGD_K3_SUBROWS")) : 2048;
          const int ksub = (cf.nchunks > 1 && cf.vec == 4)
                               ? std::max(1, std::min(cf.nchunks, sub_rows / cf.rows_chunk)) : 1;
          const int nitems = (cf.nchunks + ksub - 1) / ksub;
          if (cf.nchunks > 1) {
            slab_id = pl->n_tall_slabs++;
            wo = pl->wsq_elems;
            pl->wsq_elems += (long long)nitems * C * r;
          }
          for (int ch = 0; ch < nitems; ++ch)
            pl->k3.push_back({wo, mi, s * C, ch, cf.nchunks > 1 ? nitems : 1, slab_id, cf.vec, cf.cql, nslab,
                              ksub, 0});
        }
        const int smem = (cf.rows_chunk * r + RG * C * r + C * r) * (int)sizeof(float);
        gp.smem = std::max(gp.smem, smem);
      }
      gp.end = (int)pl->k3.size();
      if (gp.end > gp.beg) pl->g3.push_back(gp);
    }
  }
  // ---- K3 pipeline slabs: all n rows x C columns, C a power of two with the slab <= 64 KB
  {
    long long phf = 4, redf = 4, qsmax = 4;
    static const int slabf = getenv("PSGD_K3P_SLAB") ? atoi(getenv("PSGD_K3P_SLAB")) : K3P_SLAB;
    static const int maxst = getenv("PSGD_K3P_STAGES") ? atoi(getenv("PSGD_K3P_STAGES")) : 3;
    pl->k3pl.slab_floats = slabf;
    for (int mi = 0; mi < nmat; ++mi) {
      const MatDev& md = pl->mats[mi];
      if (!md.pipe) continue;
      const int rows_pad = md.n <= 256 ? md.n : (md.n + 255) / 256 * 256;
      int C = 4;
      while (C < 128 && C < md.m && (long long)(2 * C) * rows_pad <= slabf) C *= 2;
      int map = -1;
      if (md.m % 4 == 0 && md.flat_off % 4 == 0 && (int)pl->pipe_maps.size() < K3P_MAXMAPS) {
        map = (int)pl->pipe_maps.size();
        pl->pipe_maps.push_back(mi);
        pl->pipe_mapC.push_back(C);
      }
      for (int c0 = 0; c0 < md.m; c0 += C) pl->pipe_items.push_back({mi, c0, C, map});
      phf = std::max(phf, align4((long long)md.n * md.r));
      redf = std::max(redf, (long long)K3P_GW * C * md.r);
      qsmax = std::max(qsmax, (long long)C * md.r);
      pl->pipe_rmax = std::max(pl->pipe_rmax, rmax_of(md.r));
    }
    // largest slabs first: the dynamic schedule then ends on small ones
    std::stable_sort(pl->pipe_items.begin(), pl->pipe_items.end(), [&](const PipeItem& a, const PipeItem& b) {
      const long long wa = (long long)pl->mats[a.mat].n * std::min(a.C, pl->mats[a.mat].m - a.c0);
      const long long wb = (long long)pl->mats[b.mat].n * std::min(b.C, pl->mats[b.mat].m - b.c0);
      return wa > wb;
    });
    K3PLayout& L = pl->k3pl;
    L.phat_floats = (int)phf;
    L.stage_floats = (int)((L.slab_floats + phf + 255) / 256 * 256);
    L.red_floats = (int)align4(redf);
    redf = (long long)K3P_GROUPS * L.red_floats;
    // The q buffer is sized to the plan (r = 4 then keeps 3 stages).  The fused-optimizer launch
    // uses the same layout with the q buffer padded to 1024 floats per group: measured faster there
    // (ResNet-18 r=2 step + update 105 -> 92 us), while the plain step is faster with the tight
    // layout (59.7 -> 58.2 us) — profiles/r2/sweeps/opt_ab5.txt.
    static const int qs_pad = getenv("PSGD_K3P_QSPAD") ? atoi(getenv("PSGD_K3P_QSPAD")) : 0;
    const long long redf_all = redf;
    auto finish = [&](K3PLayout& X, long long qsf_group) {
      X = L;
      X.qs_floats = (int)align4(qsf_group);
      const long long qsf = (long long)K3P_GROUPS * X.qs_floats;
      auto total_for = [&](int stages) {
        long long off = (long long)stages * X.stage_floats * 4;
        off += (redf_all + qsf) * 4;
        off = (off + 15) & ~15LL;
        return off + 2LL * stages * 8 + (long long)stages * sizeof(K3PHdr) + 16;
      };
      X.stages = 2;
      while (X.stages < maxst && total_for(X.stages + 1) <= 232448 - 512) ++X.stages;  // 227 KB - static smem
      X.off_red = X.stages * X.stage_floats * 4;
      X.off_qs = X.off_red + (int)redf_all * 4;
      X.off_bar = (X.off_qs + (int)qsf * 4 + 15) & ~15;
      X.total = (int)total_for(X.stages);
    };
    K3PLayout tight{}, padded{};
    finish(tight, std::max<long long>(qsmax, qs_pad));
    finish(padded, std::max<long long>(qsmax, 1024));
    L = tight;
    pl->k3pl_f = padded;
  }
  {  // Gram-Schmidt of the pipeline's matrices inside k3_pipe (owner CTAs), not in K2
    static const bool off = getenv("PSGD_K3_GS") && getenv("PSGD_K3_GS")[0] == '0';
    for (int mi = 0; mi < nmat && !off; ++mi)
      if (pl->mats[mi].pipe) pl->gs3_list.push_back(mi);
    for (int mi : pl->wlist)
      if (std::find(pl->gs3_list.begin(), pl->gs3_list.end(), mi) == pl->gs3_list.end()) pl->wlist3.push_back(mi);
    for (int mi : pl->clist)
      if (std::find(pl->gs3_list.begin(), pl->gs3_list.end(), mi) == pl->gs3_list.end()) pl->clist3.push_back(mi);
  }
  build_row_items(pl->mats, true, pl->k4, pl->g4);
  build_tile_items(pl->mats, pl->k4t, pl->g4t);
  {  // k4_tile2 items go after the k4_tile items in the same array, in their own groups
    std::vector<int> rs;
    for (auto& md : pl->mats)
      if (k4_tileable2(md) && std::find(rs.begin(), rs.end(), md.r) == rs.end()) rs.push_back(md.r);
    for (int r : rs) {
      Group gp{r, (int)pl->k4t.size(), 0, 0, 0};
      for (int mi = 0; mi < nmat; ++mi) {
        const MatDev& md = pl->mats[mi];
        if (md.r != r || !k4_tileable2(md)) continue;
        for (int r0 = 0; r0 < md.n; r0 += K4T_ROWS)
          for (int c0 = 0; c0 < md.m; c0 += 128) pl->k4t.push_back({mi, r0, std::min(K4T_ROWS, md.n - r0), c0});
      }
      gp.end = (int)pl->k4t.size();
      pl->g4t2.push_back(gp);
    }
  }
  pl->k3t_off.assign(std::max(1, nmat), 0);
  for (int mi = 0; mi < nmat; ++mi) {
    const MatDev& md = pl->mats[mi];
    if (!k3_tileable(md)) continue;
    pl->k3t_list.push_back(mi);
    pl->k3t_off[mi] = pl->k3t_part_elems;
    pl->k3t_part_elems += (long long)((md.n + K3T_ROWS - 1) / K3T_ROWS) * md.m * md.r;
    for (int r0 = 0; r0 < md.n; r0 += K3T_ROWS)
      for (int c0 = 0; c0 < md.m; c0 += 128) pl->k3t.push_back({mi, r0, std::min(K3T_ROWS, md.n - r0), c0});
  }
  build_row_items(pl->mats, false, pl->k5, pl->g5);

  // ---- device block
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = al(off + std::max<size_t>(bytes, 16));
    return o;
  };
  const size_t o_mats = take(pl->mats.size() * sizeof(MatDev));
  const size_t o_k1 = take(pl->k1.size() * sizeof(Chunk1));
  const size_t o_k1b = take(pl->k1_beg.size() * sizeof(int));
  const size_t o_spl = take(pl->splits.size() * sizeof(SplitRow));
  const size_t o_psp = take((size_t)pl->psplit_elems * sizeof(float));
  const size_t o_spc = take(pl->splits.size() * sizeof(int));
  const size_t o_k3 = take(pl->k3.size() * sizeof(SlabItem));
  const size_t o_tl = take(pl->tall_list.size() * sizeof(int));
  const size_t o_al = take(pl->all_list.size() * sizeof(int));
  const size_t o_sl = take((pl->wlist.size() + pl->clist.size() + pl->wlist3.size() + pl->clist3.size()) * sizeof(int));
  const size_t o_g3l = take(pl->gs3_list.size() * sizeof(int));
  const size_t o_g3r = take((size_t)std::max(1, nmat) * sizeof(int));
  const size_t o_gl = take(pl->gram_list.size() * sizeof(int));
  const size_t o_gi = take(pl->gram_items.size() * sizeof(GramItem));
  const size_t o_am = take(pl->apply_mat.size() * sizeof(int));
  const size_t o_ar = take(pl->apply_row0.size() * sizeof(int));
  const size_t o_amq = take(pl->apply_mat_q.size() * sizeof(int));
  const size_t o_arq = take(pl->apply_row0_q.size() * sizeof(int));
  const size_t o_wg = take((size_t)std::max(1LL, pl->wsg_elems) * sizeof(double));
  const size_t o_wt = take(std::max<size_t>(1, pl->gram_list.size()) * K2G_TS * sizeof(double));
  const size_t o_gc = take(std::max<size_t>(1, pl->gram_list.size()) * sizeof(int));
  const size_t o_gf = take((size_t)std::max(1, nmat) * 3 * sizeof(int) + 16);
  const size_t o_k4 = take(pl->k4.size() * sizeof(RowItem));
  const size_t o_k4t = take(pl->k4t.size() * sizeof(TileItem));
  const size_t o_k1t = take(pl->k1t.size() * sizeof(TileItem));
  const size_t o_k1tl = take(pl->k1t_list.size() * sizeof(int));
  const size_t o_k1to = take(pl->k1t_off.size() * sizeof(long long));
  const size_t o_k1tp = take((size_t)std::max(1LL, pl->k1t_part_elems) * sizeof(float));
  const size_t o_k3t = take(pl->k3t.size() * sizeof(TileItem));
  const size_t o_k3tl = take(pl->k3t_list.size() * sizeof(int));
  const size_t o_k3to = take(pl->k3t_off.size() * sizeof(long long));
  const size_t o_k3tp = take((size_t)std::max(1LL, pl->k3t_part_elems) * sizeof(float));
  const size_t o_k5 = take(pl->k5.size() * sizeof(RowItem));
  const size_t o_pipe = take(pl->pipe_items.size() * sizeof(PipeItem));
  const size_t o_kre = take(pl->kr_e.size() * sizeof(RowsItem));
  const size_t o_pctr = take(2 * sizeof(int));
  const size_t o_gs = take((size_t)pl->p_elems * sizeof(double));
  const size_t o_wsq = take((size_t)std::max(1LL, pl->wsq_elems) * sizeof(float));
  const size_t o_cnt = take((size_t)std::max(1, pl->n_tall_slabs) * sizeof(int));
  const size_t o_rq = take(pl->rq.size() * sizeof(RqChunk));
  const size_t o_rqb = take(pl->rq_beg.size() * sizeof(int));
  const size_t o_rqm = take(pl->rq_mats.size() * sizeof(RqMat));
  const size_t o_rqk = take(pl->rq_blocks.size() * sizeof(int2));
  const size_t o_rqw = take((size_t)std::max(1LL, pl->rq_ws_elems) * sizeof(float));
  cudaError_t ce = cudaMalloc(&pl->dev_block, off);
  if (ce != cudaSuccess) {
    delete pl;
    return fail(PSGD_ENOMEM, std::string("cudaMalloc plan: ") + cudaGetErrorString(ce));
  }
  char* b = static_cast<char*>(pl->dev_block);
  pl->d_mats = reinterpret_cast<MatDev*>(b + o_mats);
  pl->d_k1 = reinterpret_cast<Chunk1*>(b + o_k1);
  pl->d_k1_beg = reinterpret_cast<int*>(b + o_k1b);
  pl->d_splits = reinterpret_cast<SplitRow*>(b + o_spl);
  pl->d_psplit = reinterpret_cast<float*>(b + o_psp);
  pl->d_split_cnt = reinterpret_cast<int*>(b + o_spc);
  pl->d_k3 = reinterpret_cast<SlabItem*>(b + o_k3);
  pl->d_tall_list = reinterpret_cast<int*>(b + o_tl);
  pl->d_all_list = reinterpret_cast<int*>(b + o_al);
  pl->d_small_list = reinterpret_cast<int*>(b + o_sl);
  pl->d_small_list3 = pl->d_small_list + pl->wlist.size() + pl->clist.size();
  pl->d_gs3_list = reinterpret_cast<int*>(b + o_g3l);
  pl->d_gs3_ready = reinterpret_cast<int*>(b + o_g3r);
  pl->d_gram_list = reinterpret_cast<int*>(b + o_gl);
  pl->d_gram_items = reinterpret_cast<GramItem*>(b + o_gi);
  pl->d_apply_mat = reinterpret_cast<int*>(b + o_am);
  pl->d_apply_row0 = reinterpret_cast<int*>(b + o_ar);
  pl->d_apply_mat_q = reinterpret_cast<int*>(b + o_amq);
  pl->d_apply_row0_q = reinterpret_cast<int*>(b + o_arq);
  pl->d_wsg = reinterpret_cast<double*>(b + o_wg);
  pl->d_wsT = reinterpret_cast<double*>(b + o_wt);
  pl->d_gram_cnt = reinterpret_cast<int*>(b + o_gc);
  pl->d_gs_flag = reinterpret_cast<int*>(b + o_gf);
  pl->d_gs_done = pl->d_gs_flag + std::max(1, nmat);
  pl->d_gs_cnt = pl->d_gs_done + std::max(1, nmat);
  pl->d_k1_done = pl->d_gs_cnt + std::max(1, nmat);
  pl->d_k4 = reinterpret_cast<RowItem*>(b + o_k4);
  pl->d_k4t = reinterpret_cast<TileItem*>(b + o_k4t);
  pl->d_k1t = reinterpret_cast<TileItem*>(b + o_k1t);
  pl->d_k1t_list = reinterpret_cast<int*>(b + o_k1tl);
  pl->d_k1t_off = reinterpret_cast<long long*>(b + o_k1to);
  pl->d_k1t_part = reinterpret_cast<float*>(b + o_k1tp);
  pl->d_k3t = reinterpret_cast<TileItem*>(b + o_k3t);
  pl->d_k3t_list = reinterpret_cast<int*>(b + o_k3tl);
  pl->d_k3t_off = reinterpret_cast<long long*>(b + o_k3to);
  pl->d_k3t_part = reinterpret_cast<float*>(b + o_k3tp);
  pl->d_k5 = reinterpret_cast<RowItem*>(b + o_k5);
  pl->d_pipe_items = reinterpret_cast<PipeItem*>(b + o_pipe);
  pl->d_kr_e = reinterpret_cast<RowsItem*>(b + o_kre);
  pl->d_pipe_ctr = reinterpret_cast<int*>(b + o_pctr);
  pl->d_gsws = reinterpret_cast<double*>(b + o_gs);
  pl->d_wsq = reinterpret_cast<float*>(b + o_wsq);
  pl->d_counters = reinterpret_cast<int*>(b + o_cnt);
  pl->d_rq = reinterpret_cast<RqChunk*>(b + o_rq);
  pl->d_rq_beg = reinterpret_cast<int*>(b + o_rqb);
  pl->d_rq_mats = reinterpret_cast<RqMat*>(b + o_rqm);
  pl->d_rq_blocks = reinterpret_cast<int2*>(b + o_rqk);
  pl->d_rq_ws = reinterpret_cast<float*>(b + o_rqw);
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
  };
  ce = up(pl->d_mats, pl->mats.data(), pl->mats.size() * sizeof(MatDev));
  if (ce == cudaSuccess) ce = up(pl->d_k1, pl->k1.data(), pl->k1.size() * sizeof(Chunk1));
  if (ce == cudaSuccess) ce = up(pl->d_k1_beg, pl->k1_beg.data(), pl->k1_beg.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_splits, pl->splits.data(), pl->splits.size() * sizeof(SplitRow));
  if (ce == cudaSuccess) ce = up(pl->d_k3, pl->k3.data(), pl->k3.size() * sizeof(SlabItem));
  if (ce == cudaSuccess) ce = up(pl->d_tall_list, pl->tall_list.data(), pl->tall_list.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_all_list, pl->all_list.data(), pl->all_list.size() * sizeof(int));
  {
    std::vector<int> wc(pl->wlist);
    wc.insert(wc.end(), pl->clist.begin(), pl->clist.end());
    wc.insert(wc.end(), pl->wlist3.begin(), pl->wlist3.end());
    wc.insert(wc.end(), pl->clist3.begin(), pl->clist3.end());
    if (ce == cudaSuccess) ce = up(pl->d_small_list, wc.data(), wc.size() * sizeof(int));
  }
  if (ce == cudaSuccess) ce = up(pl->d_gram_list, pl->gram_list.data(), pl->gram_list.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_gs3_list, pl->gs3_list.data(), pl->gs3_list.size() * sizeof(int));
  if (ce == cudaSuccess) ce = cudaMemset(pl->d_gs3_ready, 0, (size_t)std::max(1, nmat) * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_gram_items, pl->gram_items.data(), pl->gram_items.size() * sizeof(GramItem));
  if (ce == cudaSuccess) ce = up(pl->d_apply_mat, pl->apply_mat.data(), pl->apply_mat.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_apply_row0, pl->apply_row0.data(), pl->apply_row0.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_apply_mat_q, pl->apply_mat_q.data(), pl->apply_mat_q.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_apply_row0_q, pl->apply_row0_q.data(), pl->apply_row0_q.size() * sizeof(int));
  if (ce == cudaSuccess) ce = cudaMemset(pl->d_gram_cnt, 0, std::max<size_t>(1, pl->gram_list.size()) * sizeof(int));
  if (ce == cudaSuccess) ce = cudaMemset(pl->d_gs_flag, 0, (size_t)std::max(1, nmat) * 3 * sizeof(int) + 16);
  if (ce == cudaSuccess) ce = up(pl->d_k4, pl->k4.data(), pl->k4.size() * sizeof(RowItem));
  if (ce == cudaSuccess) ce = up(pl->d_k4t, pl->k4t.data(), pl->k4t.size() * sizeof(TileItem));
  if (ce == cudaSuccess) ce = up(pl->d_k1t, pl->k1t.data(), pl->k1t.size() * sizeof(TileItem));
  if (ce == cudaSuccess) ce = up(pl->d_k1t_list, pl->k1t_list.data(), pl->k1t_list.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_k1t_off, pl->k1t_off.data(), pl->k1t_off.size() * sizeof(long long));
  if (ce == cudaSuccess) ce = up(pl->d_k3t, pl->k3t.data(), pl->k3t.size() * sizeof(TileItem));
  if (ce == cudaSuccess) ce = up(pl->d_k3t_list, pl->k3t_list.data(), pl->k3t_list.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_k3t_off, pl->k3t_off.data(), pl->k3t_off.size() * sizeof(long long));
  if (ce == cudaSuccess) ce = up(pl->d_k5, pl->k5.data(), pl->k5.size() * sizeof(RowItem));
  if (ce == cudaSuccess) ce = up(pl->d_pipe_items, pl->pipe_items.data(), pl->pipe_items.size() * sizeof(PipeItem));
  if (ce == cudaSuccess) ce = up(pl->d_kr_e, pl->kr_e.data(), pl->kr_e.size() * sizeof(RowsItem));
  if (ce == cudaSuccess) ce = up(pl->d_rq, pl->rq.data(), pl->rq.size() * sizeof(RqChunk));
  if (ce == cudaSuccess) ce = up(pl->d_rq_beg, pl->rq_beg.data(), pl->rq_beg.size() * sizeof(int));
  if (ce == cudaSuccess) ce = up(pl->d_rq_mats, pl->rq_mats.data(), pl->rq_mats.size() * sizeof(RqMat));
  if (ce == cudaSuccess) ce = up(pl->d_rq_blocks, pl->rq_blocks.data(), pl->rq_blocks.size() * sizeof(int2));
  if (ce == cudaSuccess) ce = cudaMemset(pl->d_pipe_ctr, 0, 2 * sizeof(int));
  if (ce == cudaSuccess) ce = cudaMemset(pl->d_counters, 0, (size_t)std::max(1, pl->n_tall_slabs) * sizeof(int));
  if (ce == cudaSuccess) ce = cudaMemset(pl->d_split_cnt, 0, std::max<size_t>(16, pl->splits.size() * sizeof(int)));
  if (ce != cudaSuccess) {
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
  const bool any_fused = pl->n_tall < pl->nmat;
  o->launches_ef_p = ((pl->k1.empty() && pl->nbias == 0) ? 0 : 1) + (pl->k1t.empty() ? 0 : 2);
  o->launches_orthogonalize = (pl->nmat + (pl->nbias > 0)) > 0 ? 1 : 0;
  int k2_in_q_ef;
  {  // same rules as psgd_orthogonalize and psgd_q_ef (where k3_pipe takes the pipeline's GS and maybe the bias)
    const bool small = pl->wlist.size() + pl->clist.size() > 0;
    const bool bias_in_k3 = !small && !pl->gram_items.empty() && !pl->g3.empty();
    o->launches_orthogonalize = ((small || pl->nbias > 0) ? 1 : 0) + (pl->gram_items.empty() ? 0 : 3);
    const bool gs3 = !pl->gs3_list.empty() && !pl->pipe_items.empty();
    const bool small3 = (gs3 ? pl->wlist3.size() + pl->clist3.size() : pl->wlist.size() + pl->clist.size()) > 0;
    const bool bias_k3 = !small3 && !pl->gram_items.empty() && (!pl->g3.empty() || !pl->rq.empty());
    const bool bias_pipe = gs3 && !small3 && !bias_k3;
    k2_in_q_ef = ((small3 || (pl->nbias > 0 && !bias_k3 && !bias_pipe)) ? 1 : 0) +
                 (pl->gram_items.empty() ? 0 : 2 + (pl->apply_mat_q.empty() ? 0 : 1));
    (void)bias_in_k3;
  }
  o->launches_q_ef = k2_in_q_ef + (pl->pipe_items.empty() ? 0 : 1) + (int)pl->gkr.size() + nonempty(pl->g3) +
                     nonempty(pl->g4) + nonempty(pl->g4t) +
                     nonempty(pl->g4t2) +
                     (pl->k3t.empty() ? 0 : 2) + (pl->rq.empty() ? 0 : 2);
  (void)any_fused;
  o->launches_decompress = nonempty(pl->g5);
  o->launches_step_single = o->launches_ef_p + o->launches_q_ef;
  o->opt_fusable = opt_fusable(pl) ? 1 : 0;
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
  o->repl_cols = md.rcols;
  o->n = md.n;
  o->m = md.m;
  o->r_eff = md.r;
  o->tall = md.tall ? 1 : 0;
  o->q_ld = md.qld;
  return PSGD_OK;
}

}  // extern "C"

// ----------------------------------------------------------------------------- launchers

namespace {

template <class Kern, class... Args>
cudaError_t launch_ex(Kern kern, int grid, int block, size_t smem, cudaStream_t st, bool pdl,
                      Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int RM>
int run_k1_tiles(const psgd_plan* pl, const float* g, const float* e, float* work, const float* q, float* p,
                 cudaStream_t st) {
  if (pl->k1t.empty()) return PSGD_OK;
  const long long flag_slot = pl->flag_off + pl->nflags - 1;
  PSGD_CUDA_CHECK(cudaMemsetAsync(p + flag_slot, 0, sizeof(float), st));
  const int nitems = (int)pl->k1t.size();
  k1_tile<RM><<<(nitems + 7) / 8, kThreads, 0, st>>>(pl->d_mats, pl->d_k1t, nitems, pl->d_k1t_off, g, e, work, q,
                                                     pl->d_k1t_part);
  PSGD_CUDA_CHECK(cudaGetLastError());
  long long maxnr = 0;
  for (int mi : pl->k1t_list) maxnr = std::max(maxnr, (long long)pl->mats[mi].n * pl->mats[mi].r);
  dim3 grid((unsigned)std::min<long long>((maxnr + 255) / 256, 64), (unsigned)pl->k1t_list.size());
  k1_tile_reduce<<<grid, 256, 0, st>>>(pl->d_mats, pl->d_k1t_list, pl->d_k1t_off, pl->d_k1t_part, p, flag_slot);
  PSGD_CUDA_CHECK(cudaGetLastError());
  return PSGD_OK;
}

template <int RM>
int run_k1(const psgd_plan* pl, const float* g, const float* e, float* work, const float* q, float* p,
           const float* bias_g, int* status, cudaStream_t st) {
  const int grid = (int)pl->k1_beg.size() - 1;
  {
    const int rc = run_k1_tiles<RM>(pl, g, e, work, q, p, st);
    if (rc) return rc;
  }
  if (pl->k1.empty() && pl->nbias == 0) {  // k1_ef_p (block 0) resets the status word; here nothing else does
    PSGD_CUDA_CHECK(cudaMemsetAsync(status, 0, sizeof(int), st));
    return PSGD_OK;
  }
  auto kern = k1_ef_p<RM>;
  const size_t smem = pl->k1l.total;
  PSGD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  PSGD_CUDA_CHECK(launch_ex(kern, std::max(1, grid), kTmaThreads, smem, st, false,
                            (const MatDev*)pl->d_mats, (const Chunk1*)pl->d_k1, (const int*)pl->d_k1_beg,
                            (const SplitRow*)pl->d_splits, pl->k1l, g, e, work, q, p, pl->d_psplit,
                            pl->d_split_cnt, bias_g, (long long)pl->nbias, (long long)pl->p_bias_off,
                            (long long)pl->flag_off, status));
  return PSGD_OK;
}

template <int R, bool EXACT>
struct RunK3 {
  static int run(const psgd_plan* pl, const Group& gp, float* work, const float* p, int divisor,
                 const double* repl, float* phat, float* qout, float* e, float* bias_out, long long nbias,
                 int* status, cudaStream_t st) {
    const int nitems = gp.end - gp.beg;
    if (nitems <= 0) return PSGD_OK;
    auto kern = gp.tall ? k3_slab<R, EXACT, true> : k3_slab<R, EXACT, false>;
    if (gp.smem > 48 * 1024)
      PSGD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, gp.smem));
    PSGD_CUDA_CHECK(launch_ex(kern, nitems, kThreads, gp.smem, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats,
                              (const SlabItem*)(pl->d_k3 + gp.beg), work, p, divisor, repl, phat, qout, e,
                              pl->d_wsq, pl->d_counters, bias_out, nbias,
                              (long long)pl->p_bias_off, (long long)pl->flag_off, pl->nflags,
                              pl->world == 1 ? 1 : 0, status));
    return PSGD_OK;
  }
};

template <int MODE>
struct RunK45Mode {
  template <int R, bool EXACT>
  struct F {
    static int run(const psgd_plan* pl, const RowItem* items, const Group& gp, float* work, float* e,
                   const float* phat, const float* qsrc, int divisor, float* qstore, int write_mhat,
                   const int* status, cudaStream_t st, SgdArgs sg = SgdArgs{}) {
      const int nitems = gp.end - gp.beg;
      if (nitems <= 0) return PSGD_OK;
      const int blocks = (nitems + 7) / 8;
      PSGD_CUDA_CHECK(launch_ex(k45_rows<R, EXACT, MODE>, blocks, kThreads, 0, st, PSGD_PDL != 0,
                                (const MatDev*)pl->d_mats, items, gp.beg, gp.end, work, e, phat, qsrc, divisor,
                                qstore, write_mhat, status, sg));
      return PSGD_OK;
    }
  };
};

template <int R, bool EXACT>
using RunK4 = RunK45Mode<0>::F<R, EXACT>;

template <int R, bool EXACT>
int RunK4T2<R, EXACT>::run(const psgd_plan* pl, const Group& gp, float* work, float* e, const float* phat,
                           const float* q, int write_mhat, const int* status, cudaStream_t st) {
  const int nitems = gp.end - gp.beg;
  if (nitems <= 0) return PSGD_OK;
  PSGD_CUDA_CHECK(launch_ex(k4_tile2<R, EXACT>, (nitems + 7) / 8, kThreads, 0, st, PSGD_PDL != 0,
                            (const MatDev*)pl->d_mats, (const TileItem*)pl->d_k4t, gp.beg, gp.end, work, e, phat, q,
                            write_mhat, status));
  return PSGD_OK;
}

template <int R, bool EXACT>
struct RunK4T {
  static int run(const psgd_plan* pl, const Group& gp, float* work, float* e, const float* phat, const float* q,
                 int write_mhat, const int* status, cudaStream_t st) {
    const int nitems = gp.end - gp.beg;
    if (nitems <= 0) return PSGD_OK;
    PSGD_CUDA_CHECK(launch_ex(k4_tile<R, EXACT>, (nitems + 7) / 8, kThreads, 0, st, PSGD_PDL != 0,
                              (const MatDev*)pl->d_mats, (const TileItem*)pl->d_k4t, gp.beg, gp.end, work, e, phat,
                              q, write_mhat, status));
    return PSGD_OK;
  }
};
template <int R, bool EXACT>
using RunK5 = RunK45Mode<1>::F<R, EXACT>;


// tensor maps of the pipeline's matrices inside `work` (encoded on the host; cached
// per work buffer — a CUDA graph captures the maps by value with the launch)
int encode_pipe_maps(const psgd_plan* pl, const float* work) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return fail(PSGD_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  for (size_t k = 0; k < pl->pipe_maps.size(); ++k) {
    const MatDev& md = pl->mats[pl->pipe_maps[k]];
    cuuint64_t dims[2] = {(cuuint64_t)md.m, (cuuint64_t)md.n};
    cuuint64_t strides[1] = {(cuuint64_t)md.m * 4};
    cuuint32_t box[2] = {(cuuint32_t)pl->pipe_mapC[k], (cuuint32_t)std::min(md.n, 256)};
    cuuint32_t es[2] = {1, 1};
    const CUresult cr = encode(&pl->maps.m[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                               const_cast<float*>(work) + md.flat_off, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(PSGD_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
  }
  pl->maps_for = work;
  return PSGD_OK;
}

template <int R>
int launch_pipe_r(const psgd_plan* pl, float* work, const float* phat, float* qout, float* e, int* status,
                  cudaStream_t st, const SgdArgs& sg, const K3GS& gs) {
  auto kern = k3_pipe<R>;
  const K3PLayout& L = sg.x ? pl->k3pl_f : pl->k3pl;
  PSGD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total));
  const int grid = (int)std::min<size_t>(pl->nsm, pl->pipe_items.size());
  K3Maps maps;
  {
    std::lock_guard<std::mutex> lk(pl->map_mu);
    if (pl->maps_for != work) {
      const int rc = encode_pipe_maps(pl, work);
      if (rc) return rc;
    }
    maps = pl->maps;
  }
  PSGD_CUDA_CHECK(launch_ex(kern, grid, K3P_CT + 32, (size_t)L.total, st, PSGD_PDL != 0, maps,
                            (const MatDev*)pl->d_mats, (const PipeItem*)pl->d_pipe_items, (int)pl->pipe_items.size(),
                            L, work, phat, qout, e, pl->world == 1 ? 1 : 0, pl->d_pipe_ctr, status, sg,
                            gs));
  return PSGD_OK;
}

int launch_pipe(const psgd_plan* pl, float* work, const float* phat, float* qout, float* e, int* status,
                cudaStream_t st, const SgdArgs& sg, const K3GS& gs) {
  if (pl->pipe_items.empty()) return PSGD_OK;
  switch (pl->pipe_rmax) {
    case 1: return launch_pipe_r<1>(pl, work, phat, qout, e, status, st, sg, gs);
    case 2: return launch_pipe_r<2>(pl, work, phat, qout, e, status, st, sg, gs);
    case 4: return launch_pipe_r<4>(pl, work, phat, qout, e, status, st, sg, gs);
    default: return launch_pipe_r<8>(pl, work, phat, qout, e, status, st, sg, gs);
  }
}

template <int R>
int launch_rows_r(const psgd_plan* pl, const psgd_plan::RowsGroup& gp, float* work, float* e, const float* phat,
                  const float* q, const int* status, cudaStream_t st) {
  PSGD_CUDA_CHECK(launch_ex(k4_rows<R>, gp.eend - gp.ebeg, KR_THREADS, 0, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats,
                            (const RowsItem*)(pl->d_kr_e + gp.ebeg), work, e, phat, q, pl->world == 1 ? 1 : 0,
                            status));
  return PSGD_OK;
}

// the EF pass of the k4_rows matrices
int launch_rows(const psgd_plan* pl, float* work, float* e, const float* phat, const float* q, const int* status,
                cudaStream_t st) {
  for (const auto& gp : pl->gkr) {
    int rc;
    switch (gp.R) {
      case 1: rc = launch_rows_r<1>(pl, gp, work, e, phat, q, status, st); break;
      case 2: rc = launch_rows_r<2>(pl, gp, work, e, phat, q, status, st); break;
      default: rc = launch_rows_r<4>(pl, gp, work, e, phat, q, status, st); break;
    }
    if (rc) return rc;
  }
  return PSGD_OK;
}

template <int R>
int launch_rq_r(const psgd_plan* pl, const float* work, float* phat, const float* p, float* bias_out,
                long long nbias, int divisor, int* status, cudaStream_t st) {
  auto kern = k3_rq<R>;
  PSGD_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl->rql.total));
  static const int dpol = getenv("PSGD_RQ_POL") ? atoi(getenv("PSGD_RQ_POL")) : 1;
  PSGD_CUDA_CHECK(launch_ex(kern, (int)pl->rq_beg.size() - 1, kTmaThreads, (size_t)pl->rql.total, st, PSGD_PDL != 0,
                            (const MatDev*)pl->d_mats, (const RqChunk*)pl->d_rq, (const int*)pl->d_rq_beg, pl->rql,
                            work, phat, pl->d_rq_ws, p, (const double*)pl->d_wsT, bias_out, nbias,
                            (long long)pl->p_bias_off, divisor,
                            pl->rq_rev, dpol, status));
  return PSGD_OK;
}

int launch_rq(const psgd_plan* pl, const float* work, float* phat, const float* p, float* bias_out,
              long long nbias, int divisor, float* q_out, int* status, cudaStream_t st) {
  int rc;
  switch (pl->rq_rmax) {
    case 1: rc = launch_rq_r<1>(pl, work, phat, p, bias_out, nbias, divisor, status, st); break;
    case 2: rc = launch_rq_r<2>(pl, work, phat, p, bias_out, nbias, divisor, status, st); break;
    default: rc = launch_rq_r<4>(pl, work, phat, p, bias_out, nbias, divisor, status, st); break;
  }
  if (rc) return rc;
  PSGD_CUDA_CHECK(launch_ex(k3_rq_reduce, (int)pl->rq_blocks.size(), 32 * RQR_GROUPS, 0, st, PSGD_PDL != 0,
                            (const MatDev*)pl->d_mats, (const RqMat*)pl->d_rq_mats, (const int2*)pl->d_rq_blocks,
                            (const float*)pl->d_rq_ws, q_out, (const int*)status));
  return PSGD_OK;
}

bool check_dev(const psgd_plan* pl) {
  int dev = -1;
  cudaGetDevice(&dev);
  return dev == pl->device;
}

int launch_k2(const psgd_plan* pl, bool with_bias, const float* p, float* phat, int divisor,
              const double* repl, float* bias_out, int* status, cudaStream_t st, bool skip_pipe = false,
              bool q_path = false) {
  // skip_pipe: the pipeline's matrices are orthogonalised inside k3_pipe
  const int nw = (int)(skip_pipe ? pl->wlist3 : pl->wlist).size();
  const int nci = (int)(skip_pipe ? pl->clist3 : pl->clist).size();
  const int* wl = skip_pipe ? pl->d_small_list3 : pl->d_small_list;
  const int* cl = wl + nw;
  const int nwb = (nw + K2_THREADS / 32 - 1) / (K2_THREADS / 32);
  const int bias_blocks =
      (with_bias && pl->nbias > 0) ? (int)std::min<long long>(64, (pl->nbias + K2_THREADS * 4 - 1) / (K2_THREADS * 4)) : 0;
  const int grid = nwb + nci + bias_blocks;
  if (grid > 0) {
    const size_t smem = (size_t)pl->k2_smem;
    if (smem > 48 * 1024)
      PSGD_CUDA_CHECK(cudaFuncSetAttribute(k2_gs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PSGD_CUDA_CHECK(launch_ex(k2_gs, grid, K2_THREADS, smem, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats, wl, nw,
                              nwb, cl, nci, pl->k2_wregion, p, phat, divisor, repl, bias_out,
                              (long long)pl->p_bias_off, (long long)pl->nbias, (long long)pl->flag_off, pl->nflags,
                              status));
  }
  if (!pl->gram_items.empty()) {
      for (int pass = 1; pass <= 2; ++pass)  // pass 2 (re-orthogonalisation) exits at once unless pass 1 asks for it
      PSGD_CUDA_CHECK(launch_ex(pass == 1 ? k2_gram<1> : k2_gram<2>, (int)pl->gram_items.size(), 256, 0, st,
                                PSGD_PDL != 0,
                                (const MatDev*)pl->d_mats, (const GramItem*)pl->d_gram_items, p, divisor, repl,
                                pl->d_wsg, pl->d_wsT, pl->d_gram_cnt, (long long)pl->flag_off, pl->nflags,
                                pl->d_gsws, phat, status));
    // in psgd_q_ef, k3_rq makes the P-hat of its Gram-space matrices itself
    const std::vector<int>& am = q_path ? pl->apply_mat_q : pl->apply_mat;
    if (!am.empty())
      PSGD_CUDA_CHECK(launch_ex(k2_apply, (int)am.size(), 256, 0, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats,
                                (const int*)pl->d_gram_list, (const int*)(q_path ? pl->d_apply_mat_q : pl->d_apply_mat),
                                (const int*)(q_path ? pl->d_apply_row0_q : pl->d_apply_row0), p, divisor,
                                (const double*)pl->d_wsT, phat, (const int*)status));
  }
  return PSGD_OK;
}

}  // namespace

extern "C" {

int psgd_ef_p(const psgd_plan* pl, const float* g, const float* e, float* work, const float* q,
              float* p, const float* bias_g, int32_t* status, void* stream) {
  if (!pl || !status || !p || (pl->nmat > 0 && (!g || !work || !q)) || (pl->nbias > 0 && !bias_g))
    return fail(PSGD_EINVAL, "psgd_ef_p: NULL argument");
  if (!check_dev(pl)) return fail(PSGD_EINVAL, "psgd_ef_p: plan belongs to another device");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (pl->rmax) {
    case 1: return run_k1<1>(pl, g, e, work, q, p, bias_g, (int*)status, st);
    case 2: return run_k1<2>(pl, g, e, work, q, p, bias_g, (int*)status, st);
    case 4: return run_k1<4>(pl, g, e, work, q, p, bias_g, (int*)status, st);
    case 8: return run_k1<8>(pl, g, e, work, q, p, bias_g, (int*)status, st);
    default: return run_k1<16>(pl, g, e, work, q, p, bias_g, (int*)status, st);
  }
}

int psgd_orthogonalize(const psgd_plan* pl, const float* p, int32_t divisor, const double* repl,
                       float* p_hat, float* bias_out, int32_t* status, void* stream) {
  if (!pl || !p || !p_hat || !status || divisor < 1 || (pl->nmat > 0 && !repl) ||
      (pl->nbias > 0 && !bias_out))
    return fail(PSGD_EINVAL, "psgd_orthogonalize: bad argument");
  return launch_k2(pl, true, p, p_hat, divisor, repl, bias_out, (int*)status,
                   static_cast<cudaStream_t>(stream));
}

int psgd_orthogonalize_f64(const psgd_plan* pl, int32_t i, const double* p, const double* repl, double* p_hat,
                           int32_t* status, void* stream) {
  if (!pl || !p || !p_hat || !repl || !status || i < 0 || i >= pl->nmat)
    return fail(PSGD_EINVAL, "psgd_orthogonalize_f64: bad argument");
  const MatDev& md = pl->mats[i];
  const int nth = (int)std::min<long long>(1024, std::max<long long>(32, ((long long)md.n + 31) / 32 * 32));
  k2_gs_f64<<<1, nth, 0, static_cast<cudaStream_t>(stream)>>>(pl->d_mats, i, p, repl, pl->d_gsws, p_hat,
                                                              (int*)status);
  PSGD_CUDA_CHECK(cudaGetLastError());
  return PSGD_OK;
}

}  // extern "C"

namespace {

// K2 + K3 (+ K4); sg: the fused optimizer update (W = 1 plans that are opt_fusable)
int q_ef_impl(const psgd_plan* pl, float* work, const float* p, int32_t divisor, const double* repl,
              float* p_hat, float* q_out, float* e, float* bias_out, int32_t* status, cudaStream_t st,
              const SgdArgs& sg) {
  int rc = PSGD_OK;
  // K2: P-hat = MGS(P / W) of every matrix (compressors.py:337-338) + the bias mean.
  // When every matrix is orthogonalised in Gram space (k2_gram checks the
  // non-finite flags) and a K3 slab launch follows, that launch writes the bias
  // mean, so k2_gs is not launched for the bias alone.
  // The pipeline's matrices are orthogonalised inside k3_pipe (its owner CTAs), so no
  // K2 launch sits between K1 (or the P all-reduce) and K3 for them.
  // (not with the fused optimizer: measured 11 us slower there, 93 -> 104 us, profiles/r2/sweeps/opt_ab*.txt)
  const bool gs3 = !pl->gs3_list.empty() && !pl->pipe_items.empty() && sg.x == nullptr;
  const bool k2_small = (gs3 ? pl->wlist3.size() + pl->clist3.size() : pl->wlist.size() + pl->clist.size()) > 0;
  const bool bias_in_k3 = !k2_small && !pl->gram_items.empty() && (!pl->g3.empty() || !pl->rq.empty());
  const bool bias_in_pipe = gs3 && !k2_small && !bias_in_k3;
  if (k2_small || !pl->gram_items.empty() || (pl->nbias > 0 && !bias_in_k3 && !bias_in_pipe)) {
    rc = launch_k2(pl, !bias_in_k3 && !bias_in_pipe, p, p_hat, divisor, repl, bias_out, (int*)status, st, gs3, true);
    if (rc) return rc;
  }
  bool bias_done = !bias_in_k3;
  K3GS gs{pl->d_gs3_list, gs3 ? (int)pl->gs3_list.size() : 0, pl->d_gs3_ready, p, repl,
          (bias_in_pipe && pl->nbias > 0) ? bias_out : nullptr, (long long)pl->flag_off, (long long)pl->p_bias_off,
          (long long)pl->nbias, pl->nflags, (int)divisor};
  rc = launch_pipe(pl, work, p_hat, q_out, e, (int*)status, st, sg, gs);  // K3 pipeline (n <= 512)
  if (rc) return rc;
  if (!pl->rq.empty()) {  // q pass of the k4_rows matrices (row blocks), then the slot reduction
    rc = launch_rq(pl, work, p_hat, p, bias_out, bias_done ? 0LL : (long long)pl->nbias, (int)divisor, q_out,
                   (int*)status, st);
    if (rc) return rc;
    bias_done = true;
  }
  for (const Group& gp : pl->g3) {  // K3: q (+ EF, M-hat) per slab (after K2: delta is final)
    rc = dispatch_r<RunK3>(gp.r, pl, gp, work, p, (int)divisor, repl, p_hat, q_out, e, bias_out,
                           bias_done ? 0LL : (long long)pl->nbias, (int*)status, st);
    if (rc) return rc;
    bias_done = true;
  }
  if (!pl->k3t.empty()) {  // K3 column tiles (tall, m % 4 == 0), then the in-order block reduction
    const int nitems = (int)pl->k3t.size();
    switch (pl->rmax) {
      case 1: PSGD_CUDA_CHECK(launch_ex(k3_tile<1>, (nitems + 7) / 8, kThreads, 0, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats, (const TileItem*)pl->d_k3t, nitems, (const long long*)pl->d_k3t_off, (const float*)work, (const float*)p_hat, pl->d_k3t_part, (const int*)status)); break;
      case 2: PSGD_CUDA_CHECK(launch_ex(k3_tile<2>, (nitems + 7) / 8, kThreads, 0, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats, (const TileItem*)pl->d_k3t, nitems, (const long long*)pl->d_k3t_off, (const float*)work, (const float*)p_hat, pl->d_k3t_part, (const int*)status)); break;
      case 4: PSGD_CUDA_CHECK(launch_ex(k3_tile<4>, (nitems + 7) / 8, kThreads, 0, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats, (const TileItem*)pl->d_k3t, nitems, (const long long*)pl->d_k3t_off, (const float*)work, (const float*)p_hat, pl->d_k3t_part, (const int*)status)); break;
      case 8: PSGD_CUDA_CHECK(launch_ex(k3_tile<8>, (nitems + 7) / 8, kThreads, 0, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats, (const TileItem*)pl->d_k3t, nitems, (const long long*)pl->d_k3t_off, (const float*)work, (const float*)p_hat, pl->d_k3t_part, (const int*)status)); break;
      default: PSGD_CUDA_CHECK(launch_ex(k3_tile<16>, (nitems + 7) / 8, kThreads, 0, st, PSGD_PDL != 0, (const MatDev*)pl->d_mats, (const TileItem*)pl->d_k3t, nitems, (const long long*)pl->d_k3t_off, (const float*)work, (const float*)p_hat, pl->d_k3t_part, (const int*)status)); break;
    }
    long long maxmr = 0;
    for (int mi : pl->k3t_list) maxmr = std::max(maxmr, (long long)pl->mats[mi].m * pl->mats[mi].r);
    dim3 grid((unsigned)std::min<long long>((maxmr + 255) / 256, 64), (unsigned)pl->k3t_list.size());
    {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = PSGD_PDL ? 1 : 0;
      PSGD_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k3_tile_reduce, (const MatDev*)pl->d_mats, (const int*)pl->d_k3t_list,
                                         (const long long*)pl->d_k3t_off, (const float*)pl->d_k3t_part, q_out,
                                         (const int*)status));
    }
  }
  rc = launch_rows(pl, work, e, p_hat, q_out, (const int*)status, st);  // tall, m = 2 mod 4: EF pass
  if (rc) return rc;
  for (const Group& gp : pl->g4) {
    rc = dispatch_r<RunK4>(gp.r, pl, (const RowItem*)pl->d_k4, gp, work, e, (const float*)p_hat,
                           (const float*)q_out, 1, (float*)nullptr, pl->world == 1 ? 1 : 0,
                           (const int*)status, st);
    if (rc) return rc;
  }
  for (const Group& gp : pl->g4t) {
    rc = dispatch_r<RunK4T>(gp.r, pl, gp, work, e, (const float*)p_hat, (const float*)q_out,
                            pl->world == 1 ? 1 : 0, (const int*)status, st);
    if (rc) return rc;
  }
  for (const Group& gp : pl->g4t2) {
    rc = dispatch_r<RunK4T2>(gp.r, pl, gp, work, e, (const float*)p_hat, (const float*)q_out,
                             pl->world == 1 ? 1 : 0, (const int*)status, st);
    if (rc) return rc;
  }
  return PSGD_OK;
}

int decompress_impl(const psgd_plan* pl, const float* p_hat, const float* q_sum, int32_t divisor,
                    float* q_store, float* mhat, const int32_t* status, cudaStream_t st, SgdArgs sg) {
  for (const Group& gp : pl->g5) {
    int rc = dispatch_r<RunK5>(gp.r, pl, (const RowItem*)pl->d_k5, gp, mhat, (float*)nullptr, p_hat,
                               q_sum, divisor, q_store, 1, (const int*)status, st, sg);
    if (rc) return rc;
    sg.nbias = 0;  // the first launch updates the bias parameters
  }
  return PSGD_OK;
}

bool opt_fusable(const psgd_plan* pl) {
  if (pl->nmat == 0) return false;
  if (pl->world > 1) return true;  // K5 writes every M-hat
  for (const MatDev& md : pl->mats)
    if (!md.pipe) return false;      // W = 1: k3_pipe writes every M-hat
  return true;
}

bool make_sgd(const psgd_plan* pl, const psgd_sgd* o, const float* bias_mean, SgdArgs* sg) {
  if (!o || !o->params || !o->mom || (pl->nbias > 0 && (!o->bias_params || !o->bias_mom || !bias_mean)))
    return false;
  *sg = SgdArgs{o->params, o->mom, o->bias_params, o->bias_mom, bias_mean, pl->nbias, o->lr, o->momentum,
                o->keep_update ? 1 : 0};
  return true;
}

}  // namespace

extern "C" {

int psgd_q_ef(const psgd_plan* pl, float* work, const float* p, int32_t divisor, const double* repl,
              float* p_hat, float* q_out, float* e, float* bias_out, int32_t* status, void* stream) {
  if (!pl || !status || divisor < 1 ||
      (pl->nmat > 0 && (!work || !p || !repl || !p_hat || !q_out || !e)) || (pl->nbias > 0 && !bias_out))
    return fail(PSGD_EINVAL, "psgd_q_ef: bad argument");
  return q_ef_impl(pl, work, p, divisor, repl, p_hat, q_out, e, bias_out, status, static_cast<cudaStream_t>(stream),
                   SgdArgs{});
}

int psgd_decompress(const psgd_plan* pl, const float* p_hat, const float* q_sum, int32_t divisor,
                    float* q_store, float* mhat, const int32_t* status, void* stream) {
  if (!pl || !status || divisor < 1 || (pl->nmat > 0 && (!p_hat || !q_sum || !mhat)))
    return fail(PSGD_EINVAL, "psgd_decompress: bad argument");
  return decompress_impl(pl, p_hat, q_sum, divisor, q_store, mhat, status, static_cast<cudaStream_t>(stream),
                         SgdArgs{});
}

int psgd_decompress_sgd(const psgd_plan* pl, const float* p_hat, const float* q_sum, int32_t divisor,
                        float* q_store, float* mhat, const float* bias_mean, const psgd_sgd* opt,
                        const int32_t* status, void* stream) {
  if (!pl || !status || divisor < 1 || (pl->nmat > 0 && (!p_hat || !q_sum || !mhat)))
    return fail(PSGD_EINVAL, "psgd_decompress_sgd: bad argument");
  if (pl->world < 2 || !opt_fusable(pl)) return fail(PSGD_EINVAL, "psgd_decompress_sgd: plan is not opt_fusable");
  SgdArgs sg;
  if (!make_sgd(pl, opt, bias_mean, &sg)) return fail(PSGD_EINVAL, "psgd_decompress_sgd: NULL optimizer buffer");
  return decompress_impl(pl, p_hat, q_sum, divisor, q_store, mhat, status, static_cast<cudaStream_t>(stream), sg);
}

int psgd_step_single(const psgd_plan* pl, const float* g, float* e, float* work, float* q, float* p,
                     float* p_hat, const float* bias_g, const double* repl, float* bias_out,
                     int32_t* status, void* stream) {
  if (!pl) return fail(PSGD_EINVAL, "NULL plan");
  if (pl->world != 1) return fail(PSGD_EINVAL, "psgd_step_single needs a world-1 plan");
  if (!status) return fail(PSGD_EINVAL, "NULL status");
  int rc = psgd_ef_p(pl, g, e, work, q, p, bias_g, status, stream);
  if (!rc) rc = psgd_q_ef(pl, work, p, 1, repl, p_hat, q, e, bias_out, status, stream);
  return rc;
}

int psgd_step_single_sgd(const psgd_plan* pl, const float* g, float* e, float* work, float* q, float* p,
                         float* p_hat, const float* bias_g, const double* repl, float* bias_out,
                         const psgd_sgd* opt, int32_t* status, void* stream) {
  if (!pl) return fail(PSGD_EINVAL, "NULL plan");
  if (pl->world != 1 || !opt_fusable(pl)) return fail(PSGD_EINVAL, "psgd_step_single_sgd: plan is not opt_fusable");
  if (!status || !repl || !p_hat || !e || (pl->nbias > 0 && !bias_out))
    return fail(PSGD_EINVAL, "psgd_step_single_sgd: NULL argument");
  SgdArgs sg;
  if (!make_sgd(pl, opt, bias_out, &sg)) return fail(PSGD_EINVAL, "psgd_step_single_sgd: NULL optimizer buffer");
  int rc = psgd_ef_p(pl, g, e, work, q, p, bias_g, status, stream);
  if (!rc)
    rc = q_ef_impl(pl, work, p, 1, repl, p_hat, q, e, bias_out, status, static_cast<cudaStream_t>(stream), sg);
  return rc;
}

int psgd_momentum_step(const psgd_plan* pl, float* params, float* mom, const float* update, float* bias_params,
                       float* bias_mom, const float* bias_update, float lr, float momentum, const int32_t* status,
                       void* stream) {
  if (!pl || (pl->nmat > 0 && (!params || !mom || !update)) ||
      (pl->nbias > 0 && (!bias_params || !bias_mom || !bias_update)))
    return fail(PSGD_EINVAL, "psgd_momentum_step: NULL argument");
  const long long n4 = pl->nmat > 0 ? pl->flat_elems / 4 : 0;
  const long long work = std::max(n4, (long long)pl->nbias);
  if (work == 0) return PSGD_OK;
  const int blocks = (int)std::min<long long>((work + 255) / 256, (long long)pl->nsm * 8);
  k_momentum<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(params, mom, update, n4, lr, momentum, bias_params,
                                                                     bias_mom, bias_update, pl->nbias,
                                                                     (const int*)status);
  PSGD_CUDA_CHECK(cudaGetLastError());
  return PSGD_OK;
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
