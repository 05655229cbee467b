// psgd_resident.cu — the on-chip-resident W = 1 PowerSGD step (sm_100a).
//
// One persistent cooperative kernel, one 512-thread CTA per SM.  Every matrix
// of the catalog is cut into column slabs that hold ALL n rows (n <= 512); a
// CTA owns a set of slabs and keeps their delta = g + e ON CHIP between the
// two halves of the step — in tensor memory (TMEM, 256 KB per SM, written with
// tcgen05.st and read back with tcgen05.ld; each thread uses its own lane as
// private storage) plus shared memory:
//
//   phase 1  read g, e once (HBM); delta -> TMEM / smem; P partial = delta Q
//            per (CTA, matrix) in smem; the last CTA of each group of parts
//            reduces the group, the last group reduces the matrix and
//            orthogonalises it in one warp (float64 register MGS,
//            linalg.py:61-90); optimizer.py:120, compressors.py:336-338
//   barrier  one grid barrier (it also carries the all-or-nothing non-finite
//            flag, optimizer.py:72-76)
//   phase 2  per slab: q = delta^T P-hat from the on-chip delta (reduced in
//            smem in a fixed order), Q <- q (W = 1: the mean is a copy,
//            comm.py:92-93, compressors.py:340,373), then e = delta - P-hat q^T
//            and M-hat = P-hat q^T written once (compressors.py:375-378,
//            optimizer.py:124-127).
//
// HBM traffic per step is 16 B per matrix element (read g, e; write e, M-hat)
// instead of the 24 B of the three-kernel step that parks delta in HBM.  All
// sums run in a fixed order: results are bitwise reproducible.

#include "resident.h"

#include "common.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

namespace psgd {
namespace {

constexpr int RT = 512;          // threads per CTA
constexpr int RW = RT / 32;      // warps
constexpr int TSLOTS = 32;       // float4 TMEM slots per thread (128 columns of its lane)
constexpr int RES_NMAX = 512;    // rows a slab holds

struct RMat {
  long long flat_off, p_off, q_off, repl_off, part_off;  // part_off: per-slab P partials
  int n, m, r, qld, nparts, reducer;                      // reducer: CTA that sums the partials
};

struct RSlab {  // columns [c0, c0 + C) x all rows of `mat`; slots [slot0, slot0 + nslots) of every thread
  int mat, c0, cql, vec, nslots, slot0, part, flush;  // part: the (CTA, matrix) run's partial; flush: run ends here
  int cend, pad;                                       // columns [c0, min(c0 + C, cend)) belong to the slab
};

struct RLayout {
  int sslots, off_ps, off_red, off_qs, total;
};

__device__ __forceinline__ int ld_acquire_gpu(const unsigned* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- TMEM as per-thread private storage: a warp can reach the 32 lanes of
// its quarter (warp % 4); the four warps of a quarter split the 512 columns.
__device__ __forceinline__ void tmem_st16(uint32_t addr, const float4 (&d)[4]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(__float_as_uint(d[0].x)), "r"(__float_as_uint(d[0].y)), "r"(__float_as_uint(d[0].z)),
      "r"(__float_as_uint(d[0].w)), "r"(__float_as_uint(d[1].x)), "r"(__float_as_uint(d[1].y)),
      "r"(__float_as_uint(d[1].z)), "r"(__float_as_uint(d[1].w)), "r"(__float_as_uint(d[2].x)),
      "r"(__float_as_uint(d[2].y)), "r"(__float_as_uint(d[2].z)), "r"(__float_as_uint(d[2].w)),
      "r"(__float_as_uint(d[3].x)), "r"(__float_as_uint(d[3].y)), "r"(__float_as_uint(d[3].z)),
      "r"(__float_as_uint(d[3].w))
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float4 (&d)[4]) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr)
      : "memory");
  // the registers are only valid after wait::ld: tie them to it so no use is hoisted above
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                 "+r"(v[15])
               :
               : "memory");
#pragma unroll
  for (int u = 0; u < 4; ++u)
    d[u] = make_float4(__uint_as_float(v[4 * u]), __uint_as_float(v[4 * u + 1]), __uint_as_float(v[4 * u + 2]),
                       __uint_as_float(v[4 * u + 3]));
}

// slots s..s+3 (s % 4 == 0): TMEM below TSLOTS, shared memory above
__device__ __forceinline__ void slots_store(int s, uint32_t tb, float4* sst, const float4 (&d)[4]) {
  if (s < TSLOTS) {
    tmem_st16(tb + 4 * s, d);
  } else {
    float4* p = sst + (s - TSLOTS) * RT + threadIdx.x;
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u * RT] = d[u];
  }
}
__device__ __forceinline__ void slots_load(int s, uint32_t tb, const float4* sst, float4 (&d)[4]) {
  if (s < TSLOTS) {
    tmem_ld16(tb + 4 * s, d);
  } else {
    const float4* p = sst + (s - TSLOTS) * RT + threadIdx.x;
#pragma unroll
    for (int u = 0; u < 4; ++u) d[u] = p[u * RT];
  }
}

// A (CTA, matrix) run accumulates its P partial rows in smem; every (row, k)
// has exactly one owner lane in the CTA, so no synchronisation is needed.  The
// run's last slab publishes the sum (fixed order: slab order within the run).
__device__ __forceinline__ void run_add(float* acc, float* dst, float v, int flush, bool& bad) {
  if (flush) {
    const float s = *acc + v;
    *dst = s;
    *acc = 0.f;
    bad |= !finite1(s);  // a non-finite delta poisons its row sum (inf * 0 = NaN too)
  } else {
    *acc += v;
  }
}

// ------------------------------------------------------------------ phase 1 of one slab
// thread t: column group cq = t % CQ (4 columns, or 1 when m % 4 != 0), row group
// rg = t / CQ; slot j holds row rg + RG j (vec 4) or rows rg + RG (4j + v) (vec 1).
template <int RM>
__device__ __forceinline__ void p1_slab(const RSlab& sb, int slot0, const RMat& md, const float* __restrict__ g,
                                        const float* __restrict__ e, const float* __restrict__ Q, float4* sst,
                                        uint32_t tb, float* pacc, float* __restrict__ part, bool& bad) {
  const int t = threadIdx.x;
  const int cql = sb.cql, CQ = 1 << cql, RG = RT >> cql;
  const int cq = t & (CQ - 1), rg = t >> cql;
  const int n = md.n, m = md.m, r = md.r;
  const bool v4 = sb.vec == 4;
  const int col = sb.c0 + (v4 ? 4 * cq : cq);
  const bool colok = col < sb.cend;
  float qv[4][RM];
#pragma unroll
  for (int k = 0; k < RM; ++k) {
    const float* qk = Q + md.q_off + (long long)k * md.qld + col;
    if (v4) {
      const float4 q4 = (colok && k < r) ? __ldg(reinterpret_cast<const float4*>(qk)) : make_float4(0.f, 0.f, 0.f, 0.f);
      qv[0][k] = q4.x; qv[1][k] = q4.y; qv[2][k] = q4.z; qv[3][k] = q4.w;
    } else {
      qv[0][k] = (colok && k < r) ? __ldg(qk) : 0.f;
      qv[1][k] = qv[2][k] = qv[3][k] = 0.f;
    }
  }
  const float* gp = g + md.flat_off + col;
  const float* ep = e + md.flat_off + col;
  // batches of 8 slots: 16 x 16 B loads in flight per thread (128 KB per SM)
  for (int j0 = 0; j0 < sb.nslots; j0 += 8) {
    float4 d[8];
    if (v4) {
      float4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int row = rg + RG * (j0 + u);
        a[u] = b[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (colok && j0 + u < sb.nslots && row < n) {
          a[u] = __ldcs(reinterpret_cast<const float4*>(gp + (long long)row * m));
          b[u] = __ldcs(reinterpret_cast<const float4*>(ep + (long long)row * m));
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) d[u] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
    } else {
      float a[32], b[32];
#pragma unroll
      for (int x = 0; x < 32; ++x) {
        const int row = rg + RG * (4 * j0 + x);
        a[x] = b[x] = 0.f;
        if (colok && (j0 + (x >> 2)) < sb.nslots && row < n) {
          a[x] = __ldcs(gp + (long long)row * m);
          b[x] = __ldcs(ep + (long long)row * m);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        d[u] = make_float4(a[4 * u] + b[4 * u], a[4 * u + 1] + b[4 * u + 1], a[4 * u + 2] + b[4 * u + 2],
                           a[4 * u + 3] + b[4 * u + 3]);
    }
    {
      const float4 h[4] = {d[0], d[1], d[2], d[3]};
      slots_store(slot0 + j0, tb, sst, h);
    }
    if (j0 + 4 < sb.nslots) {  // slab-uniform: units are multiples of 4
      const float4 h[4] = {d[4], d[5], d[6], d[7]};
      slots_store(slot0 + j0 + 4, tb, sst, h);
    }
    // P rows: reduce over the CQ threads of a row (consecutive lanes), fixed butterfly order
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + u;
      if (v4) {
        float pk[RM];
#pragma unroll
        for (int k = 0; k < RM; ++k) {
          float s = d[u].x * qv[0][k];
          s = fmaf(d[u].y, qv[1][k], s);
          s = fmaf(d[u].z, qv[2][k], s);
          pk[k] = fmaf(d[u].w, qv[3][k], s);
        }
        for (int off = 1; off < CQ; off <<= 1)
#pragma unroll
          for (int k = 0; k < RM; ++k) pk[k] += __shfl_xor_sync(0xffffffffu, pk[k], off);
        const int row = rg + RG * j;
        if (cq == 0 && j < sb.nslots && row < n)
#pragma unroll
          for (int k = 0; k < RM; ++k)
            if (k < r) run_add(pacc + row * RM + k, part + row * r + k, pk[k], sb.flush, bad);
      } else {
        const float dv[4] = {d[u].x, d[u].y, d[u].z, d[u].w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float pk[RM];
#pragma unroll
          for (int k = 0; k < RM; ++k) pk[k] = dv[v] * qv[0][k];
          for (int off = 1; off < CQ; off <<= 1)
#pragma unroll
            for (int k = 0; k < RM; ++k) pk[k] += __shfl_xor_sync(0xffffffffu, pk[k], off);
          const int row = rg + RG * (4 * j + v);
          if (cq == 0 && j < sb.nslots && row < n)
#pragma unroll
            for (int k = 0; k < RM; ++k)
              if (k < r) run_add(pacc + row * RM + k, part + row * r + k, pk[k], sb.flush, bad);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ phase 2 of one slab
template <int RM>
__device__ __forceinline__ void p2_slab(const RSlab& sb, int slot0, const RMat& md, float* __restrict__ Q, float* __restrict__ e,
                                        float* __restrict__ work, const float4* sst, uint32_t tb, const float* ps,
                                        float* red, float* qs) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int cql = sb.cql, CQ = 1 << cql, RG = RT >> cql;
  const int cq = t & (CQ - 1), rg = t >> cql;
  const int n = md.n, m = md.m, r = md.r;
  const bool v4 = sb.vec == 4;
  const int col = sb.c0 + (v4 ? 4 * cq : cq);
  const bool colok = col < sb.cend;
  float qp[4][RM];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < RM; ++k) qp[v][k] = 0.f;
  // q = delta^T P-hat over this thread's rows
  for (int j0 = 0; j0 < sb.nslots; j0 += 4) {
    float4 d[4];
    slots_load(slot0 + j0, tb, sst, d);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u;
      if (v4) {
        const int row = rg + RG * j;
        if (j < sb.nslots && row < n) {
#pragma unroll
          for (int k = 0; k < RM; ++k) {
            const float p = ps[row * RM + k];
            qp[0][k] = fmaf(d[u].x, p, qp[0][k]);
            qp[1][k] = fmaf(d[u].y, p, qp[1][k]);
            qp[2][k] = fmaf(d[u].z, p, qp[2][k]);
            qp[3][k] = fmaf(d[u].w, p, qp[3][k]);
          }
        }
      } else {
        const float dv[4] = {d[u].x, d[u].y, d[u].z, d[u].w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int row = rg + RG * (4 * j + v);
          if (j < sb.nslots && row < n)
#pragma unroll
            for (int k = 0; k < RM; ++k) qp[0][k] = fmaf(dv[v], ps[row * RM + k], qp[0][k]);
        }
      }
    }
  }
  // row groups inside the warp (lanes cq, cq + CQ, ...), then warps in order
  for (int off = CQ; off < 32; off <<= 1)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int k = 0; k < RM; ++k) qp[v][k] += __shfl_xor_sync(0xffffffffu, qp[v][k], off);
  if (lane < CQ)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int k = 0; k < RM; ++k) red[((warp * 32 + lane) * 4 + v) * RM + k] = qp[v][k];
  __syncthreads();
  const int nout = CQ * 4 * RM;
  for (int o = t; o < nout; o += RT) {
    float s = 0.f;
#pragma unroll 4
    for (int w = 0; w < RW; ++w) s += red[w * 32 * 4 * RM + o];
    qs[o] = s;
    // W = 1: q is Q-bar and the next step's warm start (column-major Q)
    const int c = o / (4 * RM), v = (o / RM) & 3, k = o % RM;
    const int cx = sb.c0 + (v4 ? 4 * c + v : c);
    if (k < r && cx < sb.cend && (v4 || v == 0)) Q[md.q_off + (long long)k * md.qld + cx] = s;
  }
  __syncthreads();
  float qv[4][RM];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < RM; ++k) qv[v][k] = qs[(cq * 4 + v) * RM + k];
  // e = delta - P-hat q^T, M-hat = P-hat q^T (W = 1: locals == aggregate)
  float* eb = e + md.flat_off + col;
  float* wb = work + md.flat_off + col;
  for (int j0 = 0; j0 < sb.nslots; j0 += 4) {
    float4 d[4];
    slots_load(slot0 + j0, tb, sst, d);
    if (!colok) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u;
      if (v4) {
        const int row = rg + RG * j;
        if (j < sb.nslots && row < n) {
          float4 mh = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int k = 0; k < RM; ++k) {
            const float p = ps[row * RM + k];
            mh.x = fmaf(p, qv[0][k], mh.x);
            mh.y = fmaf(p, qv[1][k], mh.y);
            mh.z = fmaf(p, qv[2][k], mh.z);
            mh.w = fmaf(p, qv[3][k], mh.w);
          }
          const long long a = (long long)row * m;
          __stcs(reinterpret_cast<float4*>(eb + a),
                 make_float4(d[u].x - mh.x, d[u].y - mh.y, d[u].z - mh.z, d[u].w - mh.w));
          __stcs(reinterpret_cast<float4*>(wb + a), mh);
        }
      } else {
        const float dv[4] = {d[u].x, d[u].y, d[u].z, d[u].w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int row = rg + RG * (4 * j + v);
          if (j < sb.nslots && row < n) {
            float mh = 0.f;
#pragma unroll
            for (int k = 0; k < RM; ++k) mh = fmaf(ps[row * RM + k], qv[0][k], mh);
            const long long a = (long long)row * m;
            __stcs(eb + a, dv[v] - mh);
            __stcs(wb + a, mh);
          }
        }
      }
    }
  }
  __syncthreads();  // red / qs free for the next slab
}


// ------------------------------------------------------------------ fast paths (m % 4 == 0, CQ = 2^CQL >= 8)
// Same slot mapping as p1_slab / p2_slab; per-thread slot bound instead of
// per-element predicates, pointer strides, and a register reduce-scatter for
// the P rows (each lane ends up owning one (slot, k) sum and issues its add).
template <int RM, int CQL>
__device__ __forceinline__ void p1_fast(const RSlab& sb, int slot0, const RMat& md, const float* __restrict__ g,
                                        const float* __restrict__ e, const float* __restrict__ Q, float4* sst,
                                        uint32_t tb, float* pacc, float* __restrict__ part, bool& bad) {
  constexpr int CQ = 1 << CQL, RG = RT >> CQL, V = 8 * RM;
  const int t = threadIdx.x, lane = t & 31;
  const int cq = t & (CQ - 1), rg = t >> CQL;
  const int n = md.n, m = md.m, r = md.r, ns = sb.nslots;
  const int col = sb.c0 + 4 * cq;
  const bool colok = col < sb.cend;
  const int jrow = max(0, min(ns, (n - rg + RG - 1) / RG));  // slots whose row exists
  const int jmax = colok ? jrow : 0;
  float qv[4][RM];
#pragma unroll
  for (int k = 0; k < RM; ++k) {
    const float4 q4 = (colok && k < r) ? __ldg(reinterpret_cast<const float4*>(Q + md.q_off + (long long)k * md.qld + col))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
    qv[0][k] = q4.x; qv[1][k] = q4.y; qv[2][k] = q4.z; qv[3][k] = q4.w;
  }
  const long long stride = (long long)RG * m;
  const float* gp = g + md.flat_off + (long long)rg * m + col;
  const float* ep = e + md.flat_off + (long long)rg * m + col;
  for (int j0 = 0; j0 < ns; j0 += 8) {
    float4 d[8];
    {
      float4 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] = b[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j0 + u < jmax) {
          a[u] = __ldcs(reinterpret_cast<const float4*>(gp + (j0 + u) * stride));
          b[u] = __ldcs(reinterpret_cast<const float4*>(ep + (j0 + u) * stride));
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) d[u] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
    }
    {
      const float4 h[4] = {d[0], d[1], d[2], d[3]};
      slots_store(slot0 + j0, tb, sst, h);
    }
    if (j0 + 4 < ns) {  // slab-uniform: units are multiples of 4
      const float4 h[4] = {d[4], d[5], d[6], d[7]};
      slots_store(slot0 + j0 + 4, tb, sst, h);
    }
    float v[V];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < RM; ++k) {
        float s = d[u].x * qv[0][k];
        s = fmaf(d[u].y, qv[1][k], s);
        s = fmaf(d[u].z, qv[2][k], s);
        v[u * RM + k] = fmaf(d[u].w, qv[3][k], s);
      }
    // reduce-scatter over the CQ lanes of a row group (fixed order => deterministic)
    int base = 0, h = V;
#pragma unroll
    for (int l = 0; l < CQL; ++l) {
      const int o = CQ >> (l + 1);
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
        if (up) base += h;
      } else {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      }
    }
    // lane holds sums of original indices base .. base + h - 1 (h >= 1; duplicates when V < CQ)
    const bool owner = V >= CQ || (lane & ((CQ / V) - 1)) == 0;
#pragma unroll
    for (int i = 0; i < (V >= CQ ? V / CQ : 1); ++i) {
      const int oi = base + i, u = oi / RM, k = oi - u * RM;
      if (owner && k < r && j0 + u < jrow) {
        const int row = rg + RG * (j0 + u);
        run_add(pacc + row * RM + k, part + row * r + k, v[i], sb.flush, bad);
      }
    }
  }
}

template <int RM, int CQL>
__device__ __forceinline__ void p2_fast(const RSlab& sb, int slot0, const RMat& md, float* __restrict__ Q,
                                        float* __restrict__ e, float* __restrict__ work, const float4* sst,
                                        uint32_t tb, const float* ps, float* red, float* qs) {
  constexpr int CQ = 1 << CQL, RG = RT >> CQL;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int cq = t & (CQ - 1), rg = t >> CQL;
  const int n = md.n, m = md.m, r = md.r, ns = sb.nslots;
  const int col = sb.c0 + 4 * cq;
  const bool colok = col < sb.cend;
  const int jmax = colok ? max(0, min(ns, (n - rg + RG - 1) / RG)) : 0;
  float qp[4][RM];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < RM; ++k) qp[v][k] = 0.f;
  for (int j0 = 0; j0 < ns; j0 += 4) {
    float4 d[4];
    slots_load(slot0 + j0, tb, sst, d);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j0 + u < jmax) {
        const float* pr = ps + (rg + RG * (j0 + u)) * RM;
#pragma unroll
        for (int k = 0; k < RM; ++k) {
          const float p = pr[k];
          qp[0][k] = fmaf(d[u].x, p, qp[0][k]);
          qp[1][k] = fmaf(d[u].y, p, qp[1][k]);
          qp[2][k] = fmaf(d[u].z, p, qp[2][k]);
          qp[3][k] = fmaf(d[u].w, p, qp[3][k]);
        }
      }
    }
  }
#pragma unroll
  for (int off = CQ; off < 32; off <<= 1)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int k = 0; k < RM; ++k) qp[v][k] += __shfl_xor_sync(0xffffffffu, qp[v][k], off);
  if (lane < CQ)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int k = 0; k < RM; ++k) red[((warp * 32 + lane) * 4 + v) * RM + k] = qp[v][k];
  __syncthreads();
  constexpr int NOUT = CQ * 4 * RM;
  for (int o = t; o < NOUT; o += RT) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < RW; ++w) s += red[w * 32 * 4 * RM + o];
    qs[o] = s;
    const int c = o / (4 * RM), v = (o / RM) & 3, k = o % RM;
    const int cx = sb.c0 + 4 * c + v;
    if (k < r && cx < sb.cend) Q[md.q_off + (long long)k * md.qld + cx] = s;  // W = 1: q is the next warm start
  }
  __syncthreads();
  float qv[4][RM];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int k = 0; k < RM; ++k) qv[v][k] = qs[(cq * 4 + v) * RM + k];
  const long long stride = (long long)RG * m;
  float* eb = e + md.flat_off + (long long)rg * m + col;
  float* wb = work + md.flat_off + (long long)rg * m + col;
  for (int j0 = 0; j0 < ns; j0 += 4) {
    float4 d[4];
    slots_load(slot0 + j0, tb, sst, d);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j0 + u < jmax) {
        const float* pr = ps + (rg + RG * (j0 + u)) * RM;
        float4 mh = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < RM; ++k) {
          const float p = pr[k];
          mh.x = fmaf(p, qv[0][k], mh.x);
          mh.y = fmaf(p, qv[1][k], mh.y);
          mh.z = fmaf(p, qv[2][k], mh.z);
          mh.w = fmaf(p, qv[3][k], mh.w);
        }
        const long long a = (j0 + u) * stride;
        __stcs(reinterpret_cast<float4*>(eb + a), make_float4(d[u].x - mh.x, d[u].y - mh.y, d[u].z - mh.z, d[u].w - mh.w));
        __stcs(reinterpret_cast<float4*>(wb + a), mh);
      }
    }
  }
  __syncthreads();  // red / qs free for the next slab
}

// One warp orthogonalises a matrix with n <= 512, r <= RM (register float64 MGS,
// linalg.py:61-90) from the float64 P accumulator.  Kept out of line so its
// register demand does not spill the streaming loops.
template <int RM>
__device__ __noinline__ void res_mgs_call(const float* P, int n, int r, const double* repl, float* out, int* status);
template <int RM>
__device__ __forceinline__ void res_mgs_body(const float* P, int n, int r, const double* repl, float* out, int* status) {
  int l = 0;
  while ((32 << l) < n) ++l;
  if (r == 1 || RM == 1) {
    warp_mgs_dispatch_r<1>(l, P, n, 1.0, repl, out, status);
  } else if (r == 2 || RM == 2) {
    warp_mgs_dispatch_r<(RM >= 2 ? 2 : 1)>(l, P, n, 1.0, repl, out, status);
  } else if (r == 3) {
    warp_mgs_dispatch_r<(RM >= 3 ? 3 : 1)>(l, P, n, 1.0, repl, out, status);
  } else {
    warp_mgs_dispatch_r<(RM >= 4 ? 4 : 1)>(l, P, n, 1.0, repl, out, status);
  }
}
template <int RM>
__device__ __noinline__ void res_mgs_call(const float* P, int n, int r, const double* repl, float* out, int* status) {
  res_mgs_body<RM>(P, n, r, repl, out, status);
}
// inline when the register budget allows (r <= 2), out of line for r = 4
template <int RM>
__device__ __forceinline__ void res_mgs(const float* P, int n, int r, const double* repl, float* out, int* status) {
  if (RM <= 2) res_mgs_body<RM>(P, n, r, repl, out, status);
  else res_mgs_call<RM>(P, n, r, repl, out, status);
}

// ------------------------------------------------------------------ the kernel
// gb: [0] grid barrier arrivals, [1] exits, [2] non-finite flag
template <int RM>
__global__ void __launch_bounds__(RT, 1)
    k_resident(const RMat* __restrict__ mats, const RSlab* __restrict__ slabs, const int* __restrict__ cta_beg,
               RLayout L, const float* __restrict__ g, float* __restrict__ e, float* __restrict__ work,
               float* __restrict__ Q, float* __restrict__ P, float* __restrict__ Phat,
               const double* __restrict__ repl, const float* __restrict__ bias_g, float* __restrict__ bias_out,
               long long nbias, int nmat, float* __restrict__ parts, int* __restrict__ ready,
               unsigned* __restrict__ gb, int* __restrict__ status, unsigned long long* __restrict__ dbg) {
#define RES_T(i)                                                                  \
  if (dbg != nullptr && threadIdx.x == 0) {                                      \
    unsigned long long _t;                                                        \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                        \
    dbg[blockIdx.x * 8 + (i)] = _t;                                               \
  }
#define RES_LOG(k, what)                                                          \
  if (dbg != nullptr && threadIdx.x == 0 && (k) < 16) {                          \
    unsigned long long _t;                                                        \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                        \
    dbg[gridDim.x * 8 + (blockIdx.x * 16 + (k)) * 4 + (what)] = _t;               \
  }
  extern __shared__ __align__(128) unsigned char smem[];
  float4* sst = reinterpret_cast<float4*>(smem);
  float* ps = reinterpret_cast<float*>(smem + L.off_ps);  // P-hat of the current matrix (phase 2)
  float* red = reinterpret_cast<float*>(smem + L.off_red);
  float* qs = reinterpret_cast<float*>(smem + L.off_qs);
  __shared__ uint32_t s_tmem;
  __shared__ int s_status, s_flag, s_bad;
  const int t = threadIdx.x, warp = t >> 5;
  const int sb0 = cta_beg[blockIdx.x], sb1 = cta_beg[blockIdx.x + 1];

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (t == 0) {
    s_status = 0;
    s_bad = 0;
    if (blockIdx.x == 0) *status = 0;
  }
  for (int i = t; i < RES_NMAX * RM; i += RT) ps[i] = 0.f;  // run accumulators of phase 1
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(128 * (warp >> 2));
  RES_T(0);

  bool bad = false;  // bias values, and matrix elements through their P partial rows
  for (long long x = (long long)blockIdx.x * RT + t; x < nbias; x += (long long)gridDim.x * RT)
    bad |= !finite1(bias_g[x]);

  // ---------------- phase 1: every warp streams its rows of the CTA's slabs (no CTA
  // sync): delta -> TMEM / smem, the slab's P partial rows -> parts (plain stores)
  for (int si = sb0; si < sb1; ++si) {
    const RSlab sb = slabs[si];
    const RMat md = mats[sb.mat];
    float* part = parts + md.part_off + (long long)sb.part * ((md.n * md.r + 3) & ~3);
    if (sb.vec == 4 && sb.cql == 5) p1_fast<RM, 5>(sb, sb.slot0, md, g, e, Q, sst, tb, ps, part, bad);
    else if (sb.vec == 4 && sb.cql == 4) p1_fast<RM, 4>(sb, sb.slot0, md, g, e, Q, sst, tb, ps, part, bad);
    else if (sb.vec == 4 && sb.cql == 3) p1_fast<RM, 3>(sb, sb.slot0, md, g, e, Q, sst, tb, ps, part, bad);
    else p1_slab<RM>(sb, sb.slot0, md, g, e, Q, sst, tb, ps, part, bad);
    RES_LOG(si - sb0, 0);
    if (dbg != nullptr && t == 0 && si - sb0 < 16)
      dbg[gridDim.x * 8 + (blockIdx.x * 16 + si - sb0) * 4 + 1] = sb.mat * 100000 + sb.c0 * 10 + sb.vec;
    // the next run (another matrix) maps rows to other owner lanes: every warp must
    // have published and zeroed this run's accumulators first
    if (sb.flush && si + 1 < sb1) __syncthreads();
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  RES_T(1);

  // ---------------- grid barrier (carries the non-finite flag)
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  RES_T(2);
  if (t == 0) {
    if (s_bad) atomicOr(gb + 2, 1u);
    __threadfence();
    atomicAdd(gb, 1u);
    while ((unsigned)ld_acquire_gpu(gb) < gridDim.x) __nanosleep(32);
    __threadfence();
    s_flag = (int)ld_acquire_gpu(gb + 2);
  }
  __syncthreads();
  const bool poisoned = s_flag != 0;
  RES_T(3);

  // ---------------- P = sum of the slab partials (fixed order), P-hat = MGS(P): one
  // reducer CTA per matrix; phase 2 of a matrix waits for its ready flag
  if (!poisoned) {
    for (int mi = 0; mi < nmat; ++mi) {
      const RMat md = mats[mi];
      if (md.reducer != (int)blockIdx.x) continue;
      // parts: nparts x ps4 float4 (stride padded to 4 floats); n * r <= 2048, so
      // ps4 <= RT and G >= 1 thread groups split the parts (fixed order below)
      const int nr = md.n * md.r, ps4 = (nr + 3) >> 2;
      const float4* src = reinterpret_cast<const float4*>(parts + md.part_off);
      const int G = RT / ps4;
      const int o = t % ps4, q = t / ps4;
      float4* gsum = reinterpret_cast<float4*>(red);  // G x ps4 group sums (red is free until phase 2)
      if (q < G) {
        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int p0 = q; p0 < md.nparts; p0 += 16 * G) {  // 16 loads in flight, summed in order
          float4 x[16];
#pragma unroll
          for (int u = 0; u < 16; ++u)
            x[u] = p0 + u * G < md.nparts ? __ldcg(src + (long long)(p0 + u * G) * ps4 + o) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            sum.x += x[u].x; sum.y += x[u].y; sum.z += x[u].z; sum.w += x[u].w;
          }
        }
        gsum[q * ps4 + o] = sum;
      }
      __syncthreads();
      for (int x = t; x < nr; x += RT) {
        const float* gs = reinterpret_cast<const float*>(gsum) + x;
        float s = 0.f;
        for (int qq = 0; qq < G; ++qq) s += gs[qq * 4 * ps4];
        P[md.p_off + x] = s;
      }
      __syncthreads();
      RES_T(6);
      if (dbg != nullptr && t == 0) dbg[blockIdx.x * 8 + 7] = mi;
      if (warp == 0) res_mgs<RM>(P + md.p_off, md.n, md.r, repl + md.repl_off, Phat + md.p_off, &s_status);
      __syncthreads();
      if (t == 0)  // release (cumulative over the CTA's writes ordered by bar.sync)
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready + mi), "r"(1) : "memory");
    }
  }
  RES_T(5);

  // ---------------- phase 2: q, Q, e, M-hat from the on-chip delta
  if (poisoned) {
    if (blockIdx.x == 0 && t == 0) atomicOr(status, PSGD_STATUS_NONFINITE_GRAD);  // mutate nothing
  } else {
    if (t == 0 && s_status) atomicOr(status, s_status);
    for (long long x = (long long)blockIdx.x * RT + t; x < nbias; x += (long long)gridDim.x * RT)
      bias_out[x] = bias_g[x];  // W = 1: the bias mean is the bias (optimizer.py:111-113)
    int cached = -1;
    for (int si = sb0; si < sb1; ++si) {
      const RSlab sb = slabs[si];
      const RMat md = mats[sb.mat];
      if (sb.mat != cached) {
        cached = sb.mat;
        if (t == 0)
          while (ld_acquire_gpu(reinterpret_cast<const unsigned*>(ready + sb.mat)) == 0) __nanosleep(20);
        __syncthreads();
        for (int idx = t; idx < md.n * RM; idx += RT) {
          const int i = idx / RM, kk = idx - i * RM;
          ps[idx] = kk < md.r ? __ldcg(Phat + md.p_off + (long long)i * md.r + kk) : 0.f;
        }
        __syncthreads();
      }
      if (sb.vec == 4 && sb.cql == 5) p2_fast<RM, 5>(sb, sb.slot0, md, Q, e, work, sst, tb, ps, red, qs);
      else if (sb.vec == 4 && sb.cql == 4) p2_fast<RM, 4>(sb, sb.slot0, md, Q, e, work, sst, tb, ps, red, qs);
      else if (sb.vec == 4 && sb.cql == 3) p2_fast<RM, 3>(sb, sb.slot0, md, Q, e, work, sst, tb, ps, red, qs);
      else p2_slab<RM>(sb, sb.slot0, md, Q, e, work, sst, tb, ps, red, qs);
      RES_LOG(si - sb0, 2);
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  RES_T(4);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
  if (t == 0 && atomicAdd(gb + 1, 1u) == gridDim.x - 1) {  // last CTA out resets the barrier words
    gb[0] = 0;
    gb[1] = 0;
    gb[2] = 0;
    for (int mi = 0; mi < nmat; ++mi) ready[mi] = 0;
  }
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

}  // namespace

struct ResPlan {
  int nmat = 0, ctas = 0, rm = 1;
  long long nbias = 0, part_elems = 0;
  RLayout L{};
  void* dev = nullptr;
  RMat* d_mats = nullptr;
  RSlab* d_slabs = nullptr;
  int* d_beg = nullptr;
  float* d_parts = nullptr;
  int* d_cnt = nullptr;
  unsigned* d_gb = nullptr;
  unsigned long long* d_dbg = nullptr;  // PSGD_RES_TIMING=1: per-CTA phase timestamps
};

struct HostPlan {
  int RM = 1, ctas = 0, cap = 0;
  RLayout L{};
  std::vector<RMat> mats;
  std::vector<RSlab> q;
  std::vector<int> beg, used;
  std::vector<double> load;
  long long ao = 0;
};

// The partition (host only, no CUDA calls): false + *why when not eligible.
static bool res_partition(const ResMatIn* in, int nmat, int nsm, HostPlan& hp, std::string* why) {
  auto fail_ = [&](const std::string& s) {
    if (why) *why = s;
    return false;
  };
  if (nmat < 1) return fail_("no matrices");
  int rmax = 1;
  for (int i = 0; i < nmat; ++i) {
    if (in[i].n > RES_NMAX) return fail_("n > 512");
    if (in[i].r > 4) return fail_("r > 4");
    rmax = std::max(rmax, in[i].r);
  }
  const int RM = rmax <= 1 ? 1 : rmax <= 2 ? 2 : 4;
  RLayout L{};
  const int ps_b = RES_NMAX * RM * 4, red_b = RW * 32 * 4 * RM * 4, qs_b = 32 * 4 * RM * 4;
  const int budget = 227 * 1024 - 1024;  // static smem + slack
  L.sslots = std::min(env_int("PSGD_RES_SSLOTS", 64), ((budget - ps_b - red_b - qs_b) / (RT * 16)) & ~3);
  if (L.sslots < 0) L.sslots = 0;
  L.off_ps = L.sslots * RT * 16;
  L.off_red = L.off_ps + ps_b;
  L.off_qs = L.off_red + red_b;
  L.total = L.off_qs + qs_b;
  const int cap = TSLOTS + L.sslots;  // float4 slots per thread
  const int slab_max = std::max(4, env_int("PSGD_RES_SLAB", 8));

  // ---- geometry per matrix: the widest slab (C = 4 CQ columns, all rows) with at
  // most slab_max slots per thread; partial slabs take the narrowest CQ >= 8 that fits
  std::vector<RMat> mats(nmat);
  std::vector<int> vecs(nmat), cqls(nmat);
  for (int i = 0; i < nmat; ++i) {
    const ResMatIn& mi = in[i];
    RMat& md = mats[i];
    md.flat_off = mi.flat_off;
    md.p_off = mi.p_off;
    md.q_off = mi.q_off;
    md.repl_off = mi.repl_off;
    md.n = mi.n;
    md.m = mi.m;
    md.r = mi.r;
    md.qld = mi.qld;
    const int vec = (mi.m % 4 == 0 && mi.flat_off % 4 == 0) ? 4 : 1;
    const int groups = (mi.m + vec - 1) / vec;
    int cql = 0;
    while (cql < 5 && (1 << cql) < groups) ++cql;
    auto slots_for = [&](int c) {
      const int rows_per = (RT >> c) * (vec == 4 ? 1 : 4);
      return (mi.n + rows_per - 1) / rows_per;
    };
    while (cql > 0 && slots_for(cql) > slab_max) --cql;
    vecs[i] = vec;
    cqls[i] = cql;
  }
  auto slots_of = [&](int i, int cql) {
    const int rows_per = (RT >> cql) * (vecs[i] == 4 ? 1 : 4);
    return (in[i].n + rows_per - 1) / rows_per;
  };
  // ---- exact contiguous partition: every CTA gets an equal share of the catalog's
  // elements; large matrices are split at 4-column granularity (a CTA holds
  // adjacent column ranges, so a matrix has ~(its share of the CTAs) partials)
  // one geometry per matrix: a (CTA, matrix) run accumulates its P rows in smem
  // without synchronisation, which needs the same row -> owner-lane map in every
  // slab of the run (a partial slab keeps the full geometry, idle columns masked)
  auto part_cql = [&](int i, int w) {
    (void)w;
    return cqls[i];
  };
  auto units_for = [&](int i, int w) {
    const int C = (1 << cqls[i]) * vecs[i];
    int u = (w / C) * ((slots_of(i, cqls[i]) + 3) & ~3);
    if (w % C) u += (slots_of(i, part_cql(i, w % C)) + 3) & ~3;
    return u;
  };
  double total = 0;
  for (int i = 0; i < nmat; ++i) total += (double)in[i].n * in[i].m;
  const int ctas = nsm;
  const double quota = total / ctas;
  struct S {
    int mat, c0, cend, cql, vec, nslots, units;
  };
  std::vector<std::vector<S>> own(ctas);
  std::vector<double> load(ctas, 0.0);
  std::vector<int> used(ctas, 0);
  int c = 0;
  double rem = quota;
  // small matrices first (whole-slab granularity), the big ones last: the final
  // CTAs then split a large matrix at 4-column granularity and come out even
  std::vector<int> walk(nmat);
  std::iota(walk.begin(), walk.end(), 0);
  std::stable_sort(walk.begin(), walk.end(), [&](int a, int b) {
    return (long long)in[a].n * in[a].m < (long long)in[b].n * in[b].m;
  });
  for (int i : walk) {
    const int n = in[i].n, m = in[i].m, vec = vecs[i], C = (1 << cqls[i]) * vec;
    const int ufull = (slots_of(i, cqls[i]) + 3) & ~3;
    const int gran = (vec == 1 || m <= C) ? C : 4;  // narrow / scalar-column matrices: whole slabs
    int col = 0;
    while (col < m) {
      int take;
      if (c == ctas - 1) {
        take = m - col;
      } else {
        take = (int)(rem / n) / gran * gran;
        if (take < gran && rem < 0.5 * (double)n * gran && !own[c].empty()) {
          ++c;
          rem += quota;
          continue;
        }
        take = std::min(std::max(take, gran), m - col);
        if (m - col - take < gran) take = m - col;  // no sliver left behind
        while (take > 0 && used[c] + units_for(i, take) > cap) take -= gran;
        if (take <= 0) {
          ++c;
          rem += quota;
          continue;
        }
      }
      for (int c0 = col; c0 < col + take; c0 += C) {
        const int w = std::min(C, col + take - c0);
        const int cq = w == C ? cqls[i] : (vec == 4 ? part_cql(i, w) : cqls[i]);
        const int ns = slots_of(i, cq);
        own[c].push_back({i, c0, c0 + w, cq, vec, ns, (ns + 3) & ~3});
        used[c] += (ns + 3) & ~3;
      }
      load[c] += (double)n * take;
      rem -= (double)n * take;
      col += take;
      if (rem < 0.5 * 4 * n && c + 1 < ctas) {
        ++c;
        rem += quota;
      }
    }
  }
  for (int k = 0; k < ctas; ++k)
    if (used[k] > cap) {
      if (env_int("PSGD_RES_DEBUG", 0)) {
        fprintf(stderr, "[resident] CTA %d uses %d > %d slots:", k, used[k], cap);
        for (auto& x : own[k]) fprintf(stderr, " m%d[%d,%d)cq%d:%d", x.mat, x.c0, x.cend, x.cql, x.units);
        fprintf(stderr, "\n");
      }
      return fail_("delta does not fit in TMEM + shared memory");
    }
  std::vector<RSlab> q;
  std::vector<int> beg(1, 0);
  for (int k = 0; k < ctas; ++k) {
    auto& v = own[k];
    int slot = 0;
    for (size_t j = 0; j < v.size(); ++j) {
      const S& x = v[j];
      const bool flush = j + 1 == v.size() || v[j + 1].mat != x.mat;
      q.push_back({x.mat, x.c0, x.cql, x.vec, x.nslots, slot, mats[x.mat].nparts, flush ? 1 : 0, x.cend, 0});
      if (flush) mats[x.mat].nparts++;
      slot += x.units;
    }
    beg.push_back((int)q.size());
  }
  std::vector<int> nsl(nmat, 0);
  for (auto& x : q) nsl[x.mat]++;
  long long ao = 0;
  for (auto& md : mats) {  // partial buffers, 16-B aligned rows of parts
    md.part_off = ao;
    ao += (long long)md.nparts * (((long long)md.n * md.r + 3) & ~3LL);
  }
  // reducers: the big matrices to the CTAs with the least phase load
  {
    std::vector<int> mo(nmat), co(ctas);
    std::iota(mo.begin(), mo.end(), 0);
    std::iota(co.begin(), co.end(), 0);
    std::stable_sort(mo.begin(), mo.end(), [&](int a, int b) {
      return (long long)mats[a].n * mats[a].r * nsl[a] > (long long)mats[b].n * mats[b].r * nsl[b];
    });
    std::stable_sort(co.begin(), co.end(), [&](int a, int b) { return load[a] < load[b]; });
    for (int k = 0; k < nmat; ++k) mats[mo[k]].reducer = co[k % ctas];
  }
  if (env_int("PSGD_RES_DEBUG", 0)) {
    double mx = 0, tot = 0;
    int umax = 0;
    for (int c = 0; c < ctas; ++c) {
      mx = std::max(mx, load[c]);
      tot += load[c];
      umax = std::max(umax, used[c]);
    }
    fprintf(stderr, "[resident] %zu slabs on %d CTAs, cap %d slots (%d smem), max/avg load %.3f, max slots %d\n",
            q.size(), ctas, cap, L.sslots, mx / (tot / ctas), umax);
  }
  hp.RM = RM;
  hp.ctas = ctas;
  hp.cap = cap;
  hp.L = L;
  hp.mats = std::move(mats);
  hp.q = std::move(q);
  hp.beg = std::move(beg);
  hp.used = std::move(used);
  hp.load = std::move(load);
  hp.ao = ao;
  return true;
}

ResPlan* res_plan_create(const ResMatIn* in, int nmat, long long nbias, int nsm, std::string* why) {
  auto no = [&](const std::string& s) -> ResPlan* {
    if (why) *why = s;
    return nullptr;
  };
  // opt-in: measured slower than the three-kernel step on B200 so far
  if (env_int("PSGD_RESIDENT", 0) == 0) return no("not enabled (PSGD_RESIDENT=1 opts in)");
  HostPlan hp;
  if (!res_partition(in, nmat, nsm, hp, why)) return nullptr;
  const int RM = hp.RM, ctas = hp.ctas;
  const RLayout L = hp.L;
  const std::vector<RMat>& mats = hp.mats;
  const std::vector<RSlab>& q = hp.q;
  const std::vector<int>& beg = hp.beg;
  const long long ao = hp.ao;
  // ---- device block
  ResPlan* rp = new ResPlan();
  rp->nmat = nmat;
  rp->ctas = ctas;
  rp->rm = RM;
  rp->nbias = nbias;
  rp->part_elems = ao;
  rp->L = L;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_m = 0, o_s = al(o_m + mats.size() * sizeof(RMat)), o_b = al(o_s + q.size() * sizeof(RSlab)),
               o_a = al(o_b + beg.size() * sizeof(int)), o_c = al(o_a + std::max<long long>(1, ao) * sizeof(float)),
               o_g = al(o_c + std::max(1, nmat) * sizeof(int)), dev_bytes = al(o_g + 4 * sizeof(unsigned));
  if (cudaMalloc(&rp->dev, dev_bytes) != cudaSuccess) {
    cudaGetLastError();
    delete rp;
    return no("cudaMalloc failed");
  }
  char* b = static_cast<char*>(rp->dev);
  rp->d_mats = reinterpret_cast<RMat*>(b + o_m);
  rp->d_slabs = reinterpret_cast<RSlab*>(b + o_s);
  rp->d_beg = reinterpret_cast<int*>(b + o_b);
  rp->d_parts = reinterpret_cast<float*>(b + o_a);
  rp->d_cnt = reinterpret_cast<int*>(b + o_c);
  rp->d_gb = reinterpret_cast<unsigned*>(b + o_g);
  cudaError_t ce = cudaMemcpy(rp->d_mats, mats.data(), mats.size() * sizeof(RMat), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemcpy(rp->d_slabs, q.data(), q.size() * sizeof(RSlab), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemcpy(rp->d_beg, beg.data(), beg.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMemset(rp->d_cnt, 0, std::max(1, nmat) * sizeof(int));
  if (ce == cudaSuccess) ce = cudaMemset(rp->d_gb, 0, 4 * sizeof(unsigned));
  if (ce != cudaSuccess) {
    cudaGetLastError();
    res_plan_destroy(rp);
    return no("plan upload failed");
  }
  if (env_int("PSGD_RES_TIMING", 0) && cudaMalloc(&rp->d_dbg, (size_t)ctas * (8 + 64) * 8) != cudaSuccess) {
    cudaGetLastError();
    rp->d_dbg = nullptr;
  }
  return rp;
}

int res_dryrun(const ResMatIn* in, int nmat, int nsm, double* stats, std::string* why) {
  HostPlan hp;
  if (!res_partition(in, nmat, nsm, hp, why)) return 0;
  double mx = 0, tot = 0;
  int umax = 0;
  for (int c = 0; c < hp.ctas; ++c) {
    mx = std::max(mx, hp.load[c]);
    tot += hp.load[c];
    umax = std::max(umax, hp.used[c]);
  }
  stats[0] = hp.ctas;
  stats[1] = (double)hp.q.size();
  stats[2] = tot > 0 ? mx / (tot / hp.ctas) : 0;
  stats[3] = umax;
  stats[4] = hp.cap;
  return 1;
}

int res_debug_times(const ResPlan* rp, long long* out, long long cap) {
  if (!rp || !rp->d_dbg) return 0;
  const long long nv = std::min<long long>(cap, (long long)rp->ctas * (8 + 64));
  if (cudaMemcpy(out, rp->d_dbg, nv * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return (int)nv;
}

void res_plan_destroy(ResPlan* rp) {
  if (!rp) return;
  if (rp->d_dbg) cudaFree(rp->d_dbg);
  if (rp->dev) cudaFree(rp->dev);
  delete rp;
}

int res_ctas(const ResPlan* rp) { return rp ? rp->ctas : 0; }

template <int RM>
static cudaError_t res_launch(const ResPlan* rp, const float* g, float* e, float* work, float* Q, float* P,
                              float* Phat, const double* repl, const float* bias_g, float* bias_out, int* status,
                              cudaStream_t st) {
  auto kern = k_resident<RM>;
  cudaError_t ce = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, rp->L.total);
  if (ce != cudaSuccess) return ce;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(rp->ctas);
  cfg.blockDim = dim3(RT);
  cfg.dynamicSmemBytes = rp->L.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident: the grid barrier is safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, (const RMat*)rp->d_mats, (const RSlab*)rp->d_slabs, (const int*)rp->d_beg,
                            rp->L, g, e, work, Q, P, Phat, repl, bias_g, bias_out, rp->nbias,
                            rp->nmat, rp->d_parts, rp->d_cnt, rp->d_gb, status, rp->d_dbg);
}

cudaError_t res_step(const ResPlan* rp, const float* g, float* e, float* work, float* Q, float* P, float* Phat,
                     const double* repl, const float* bias_g, float* bias_out, int* status, cudaStream_t st) {
  switch (rp->rm) {
    case 1: return res_launch<1>(rp, g, e, work, Q, P, Phat, repl, bias_g, bias_out, status, st);
    case 2: return res_launch<2>(rp, g, e, work, Q, P, Phat, repl, bias_g, bias_out, status, st);
    default: return res_launch<4>(rp, g, e, work, Q, P, Phat, repl, bias_g, bias_out, status, st);
  }
}

}  // namespace psgd
