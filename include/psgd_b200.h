/*
 * psgd_b200.h — C ABI of the B200-native PowerSGD compression hot path.
 *
 * This is the drop-in boundary for the reference's compressor plug-in path
 * (`/root/reference/pkg/src/gradcomp`).  The reference is pure Python/numpy, so
 * the "FFI" a maintainer adds is a ctypes binding; the
 * Python adapter `paper_1905_13727_b200.compressor.PowerSGD` is that binding
 * and mirrors `Compressor` (compressors.py:221-249) / `PowerSGD`
 * (compressors.py:344-397) name for name.
 *
 * Every call is asynchronous on the caller's CUDA stream; pointers are device
 * pointers to caller-owned fp32 buffers laid out as `psgd_plan_matrix` reports.
 * Return value: 0 on success, a negative PSGD_E* code otherwise (message via
 * psgd_last_error()).  Numerical outcomes that the reference raises on are
 * reported through the device status word (PSGD_STATUS_*), which every later
 * kernel of the step checks before mutating state, so a failing step leaves
 * the error-feedback memory and the warm-start Q untouched — the same
 * guarantee as the reference's check-before-mutate in optimizer.py:72-76,106.
 *
 * Per-step call sequence (one data-parallel worker = one GPU):
 *   psgd_ef_p            delta = g + e ; P = delta Q ; bias -> P tail   (optimizer.py:115-121, compressors.py:336)
 *   [all-reduce(sum) of P incl. bias tail over the workers]              (compressors.py:337, optimizer.py:111-113)
 *   psgd_q_ef            P-hat = MGS(P / W) ; q_w = delta^T P-hat ;       (compressors.py:338-339, linalg.py:61-90)
 *                        e = delta - P-hat q_w^T ; bias mean              (compressors.py:376-378, optimizer.py:124-127)
 *                        (W == 1: also M-hat and the warm-start Q; done)
 *   [all-reduce(sum) of q over the workers]                               (compressors.py:340)
 *   psgd_decompress      Q = q_sum / W (warm start) ; M-hat = P-hat Q^T   (compressors.py:373-375)
 */
#ifndef PSGD_B200_H
#define PSGD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSGD_OK        0
#define PSGD_EINVAL   -1   /* bad argument -> ContractViolation (linalg.py:20, compressors.py:230) */
#define PSGD_ECUDA    -2   /* CUDA launch / allocation error -> RuntimeError */
#define PSGD_ENOMEM   -3

/* device status word bits (int32, caller-owned; psgd_ef_p resets it each step) */
#define PSGD_STATUS_NONFINITE_GRAD  1  /* optimizer.py:72-76 NonFiniteGradient */
#define PSGD_STATUS_NONFINITE_P     2  /* linalg.py:35-36 via orthogonalize(as_matrix) */
#define PSGD_STATUS_REPLACEMENT     4  /* linalg.py:82-88 needed more replacement draws than the table holds */

#define PSGD_MAX_RANK   16
#define PSGD_MAX_TREE   64
#define PSGD_REPL_ATTEMPTS 3  /* replacement draws per column held on the device (linalg.py:82-88 attempt 0..2) */

typedef struct psgd_plan psgd_plan;

typedef struct {
    int64_t flat_elems;   /* length of the g / e / work buffers (matrices packed, 16-B aligned starts) */
    int64_t p_elems;      /* length of the packed P buffer: sum n*r_eff (aligned) + bias tail + flags */
    int64_t p_bias_off;   /* offset of the bias tail inside the P buffer */
    int64_t q_elems;      /* length of the packed Q buffers: sum r_eff * q_ld */
    int64_t repl_elems;   /* doubles in the degenerate-column replacement table (PSGD_REPL_ATTEMPTS draws per column) */
    int64_t nbias;        /* bias scalars carried uncompressed */
    int32_t nmat;
    int32_t rank;
    int32_t world;
    int32_t n_tall;       /* matrices taking the split-n (non-fused) path */
    int64_t items_k1;     /* warp work items of psgd_ef_p */
    int64_t items_k3;     /* CTA work items of psgd_q_ef */
    int32_t launches_ef_p;        /* kernel launches issued by one psgd_ef_p call */
    int32_t launches_orthogonalize;
    int32_t launches_q_ef;
    int32_t launches_decompress;
    int32_t launches_step_single; /* kernel launches issued by one psgd_step_single call */
    int32_t opt_fusable;  /* 1: psgd_step_single_sgd (world 1) / psgd_decompress_sgd (world > 1) accept this plan */
} psgd_plan_info;

/* Heavy-ball optimizer state for the fused update of optimizer.py:131-134
 * (m = momentum * m + u ; x -= lr * (u + m), u = M-hat / the bias mean): params
 * and mom in the plan's flat layout (flat_elems), bias_params / bias_mom in the
 * bias layout (nbias).  keep_update = 0: M-hat is consumed in registers and not
 * written to `work` (the bias mean is still written to bias_out). */
typedef struct {
    float* params;
    float* mom;
    float* bias_params;
    float* bias_mom;
    float lr;
    float momentum;
    int32_t keep_update;
    int32_t pad;
} psgd_sgd;

typedef struct {
    int64_t flat_off;     /* element offset of the n x m row-major matrix in g / e / work */
    int64_t p_off;        /* element offset of its n x r_eff P block */
    int64_t q_off;        /* element offset of its Q block: column-major, (j, k) at q_off + k * q_ld + j */
    int64_t repl_off;     /* double offset of its replacement table: column j, attempt a (linalg.py:54-58)
                             at repl_off + (a * repl_cols + j) * n; shared by every matrix with the same n */
    int32_t n, m, r_eff;
    int32_t tall;         /* 1: n > fused limit, q via split-n partials + separate EF pass */
    int32_t q_ld;         /* column stride of the Q block (m rounded up to a multiple of 4) */
    int32_t repl_cols;    /* columns per attempt in its replacement table (max r_eff over matrices with this n) */
} psgd_matrix_info;

/* Plan: shapes -> packed layout, per-kernel work lists, plan-owned scratch.
 * Replaces the per-parameter loop of optimizer.py:110-129 (shapes from
 * catalogs.py:37-42; r_eff = min(n, m, rank) as compressors.py:359-360).
 * Allocates device memory on the current device.  A plan's scratch is used by
 * psgd_orthogonalize / psgd_q_ef, so one plan serves one stream at a time. */
int psgd_plan_create(int32_t nmat, const int64_t* n, const int64_t* m, int32_t rank,
                     int32_t world, int64_t nbias, psgd_plan** out);
int psgd_plan_destroy(psgd_plan* plan);
int psgd_plan_get_info(const psgd_plan* plan, psgd_plan_info* out);
int psgd_plan_matrix(const psgd_plan* plan, int32_t i, psgd_matrix_info* out);

/* K1 — replaces optimizer.py:115-121 (delta = g + e), compressors.py:336
 * (P_w = delta Q) and the bias pack for optimizer.py:111-113.
 * g, e: flat_elems (e may be NULL: error feedback off, optimizer.py:118-119).
 * work: out delta.  q: warm-start Q (q_elems).  p: out P (p_elems; the bias
 * tail receives bias_g, the flag tail one non-finite flag per CTA, so the P
 * all-reduce carries them to every worker; K2 raises PSGD_STATUS_NONFINITE_GRAD
 * from them).  status: reset to 0 by every call. */
int psgd_ef_p(const psgd_plan* plan, const float* g, const float* e, float* work,
              const float* q, float* p, const float* bias_g, int32_t* status, void* stream);

/* K2 — standalone Gram-Schmidt: replaces compressors.py:337-338 after the sum,
 * P = P_sum / divisor (comm.py:97-98; divisor 1 = the W=1 copy), then
 * orthogonalize (linalg.py:61-90) in float64 with the seeded replacement
 * columns `repl` (linalg.py:54-58, laid out per psgd_matrix_info.repl_off).
 * Writes P-hat to p_hat (may equal p) and the bias mean to bias_out.
 * psgd_q_ef performs the same orthogonalisation itself; this entry point
 * serves linalg.orthogonalize and callers that want P-hat alone. */
int psgd_orthogonalize(const psgd_plan* plan, const float* p, int32_t divisor, const double* repl,
                       float* p_hat, float* bias_out, int32_t* status, void* stream);

/* linalg.orthogonalize (linalg.py:61-90) on float64 input, computed in float64
 * exactly as the reference (no fp32 rounding of the input): P-hat of the plan's
 * matrix i (n x r_eff, row-major doubles) with the seeded replacement loop
 * (linalg.py:82-88) drawing from `repl`.  p and p_hat may alias. */
int psgd_orthogonalize_f64(const psgd_plan* plan, int32_t i, const double* p, const double* repl,
                           double* p_hat, int32_t* status, void* stream);

/* K3 (+ tall-matrix kernels) — replaces compressors.py:338 (P-hat = GS(P / W)),
 * :339 (q_w = delta^T P-hat), :376-378 (locals = P-hat q_w^T) and
 * optimizer.py:124-127 (e = delta - local), plus the bias mean of
 * optimizer.py:111-113.  p: the summed P buffer from psgd_ef_p (after the
 * all-reduce when W > 1); p_hat receives P-hat; work: in delta, and when the
 * plan's world == 1 it is overwritten with M-hat (compressors.py:375; M-hat ==
 * local at W=1) and q_out is the next warm start.  When world > 1, q_out
 * receives the local q_w to be all-reduced.  A non-finite gradient on any
 * worker (flags carried in p) leaves every buffer untouched. */
int psgd_q_ef(const psgd_plan* plan, float* work, const float* p, int32_t divisor, const double* repl,
              float* p_hat, float* q_out, float* e, float* bias_out, int32_t* status, void* stream);

/* K5 — replaces compressors.py:340 (after the sum), :373 (warm-start store)
 * and :375 (M-hat = P-hat Q-bar^T).  Q-bar = q_sum / divisor; if q_store is
 * non-NULL and differs from q_sum it receives Q-bar.  mhat: flat_elems. */
int psgd_decompress(const psgd_plan* plan, const float* p_hat, const float* q_sum,
                    int32_t divisor, float* q_store, float* mhat, const int32_t* status,
                    void* stream);

/* One W == 1 step: psgd_ef_p + psgd_q_ef. */
int psgd_step_single(const psgd_plan* plan, const float* g, float* e, float* work, float* q,
                     float* p, float* p_hat, const float* bias_g, const double* repl,
                     float* bias_out, int32_t* status, void* stream);

/* One W == 1 step with the optimizer update (optimizer.py:131-134) fused into
 * the M-hat epilogue: K3 applies m = momentum m + M-hat, x -= lr (M-hat + m) from
 * the registers that hold M-hat (and the bias update from the bias mean), so M-hat
 * never makes an HBM round trip.  Replaces psgd_step_single + psgd_momentum_step.
 * PSGD_EINVAL unless psgd_plan_info.opt_fusable.  A failed step (status) leaves
 * params and mom untouched. */
int psgd_step_single_sgd(const psgd_plan* plan, const float* g, float* e, float* work, float* q,
                         float* p, float* p_hat, const float* bias_g, const double* repl,
                         float* bias_out, const psgd_sgd* opt, int32_t* status, void* stream);

/* K5 with the optimizer update fused (world > 1): psgd_decompress, then
 * optimizer.py:131-134 on M-hat in registers and on bias_mean (the bias mean
 * psgd_q_ef wrote).  Replaces psgd_decompress + psgd_momentum_step. */
int psgd_decompress_sgd(const psgd_plan* plan, const float* p_hat, const float* q_sum, int32_t divisor,
                        float* q_store, float* mhat, const float* bias_mean, const psgd_sgd* opt,
                        const int32_t* status, void* stream);

/* Simulated-worker mean — replaces comm.py:84-98 (tree_reduce :51-67 then / W)
 * for the single-GPU W-list mode: out = tree_sum(bufs[0..nbuf)) / nbuf, in the
 * reference's pairing order.  bufs is a HOST array of device pointers. */
int psgd_tree_mean(const float* const* bufs, int32_t nbuf, int64_t count, float* out, void* stream);

/* Heavy-ball update of every parameter in one pass (optimizer.py:131-134,
 * reference_momentum_step :163-171): m = momentum * m + u ; x -= lr * (u + m),
 * u = M-hat in the plan's flat layout (`work` after a step) and the bias mean.
 * params / mom use the same flat layout (flat_elems floats) and bias layout. */
int psgd_momentum_step(const psgd_plan* plan, float* params, float* mom, const float* update,
                       float* bias_params, float* bias_mom, const float* bias_update, float lr,
                       float momentum, const int32_t* status, void* stream);

const char* psgd_last_error(void);
int32_t psgd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PSGD_B200_H */
