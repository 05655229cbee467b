// resident.h — internal interface of the on-chip-resident W = 1 step (psgd_resident.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace psgd {

struct ResMatIn {  // one matrix of the main plan (offsets into the caller's buffers)
  long long flat_off, p_off, q_off, repl_off;
  int n, m, r, qld;
};

struct ResPlan;

// nullptr (and *why) when the catalog is not eligible: W != 1, n > 512, r > 4,
// or delta does not fit in TMEM + shared memory of the SMs.
ResPlan* res_plan_create(const ResMatIn* mats, int nmat, long long nbias, int nsm, std::string* why);
void res_plan_destroy(ResPlan* rp);
int res_ctas(const ResPlan* rp);
// host-only partition check: 1 and stats {ctas, slabs, max/avg load, max slots, slot cap}, or 0 and *why
int res_dryrun(const ResMatIn* in, int nmat, int nsm, double* stats, std::string* why);
// PSGD_RES_TIMING=1 at plan creation: 8 globaltimer stamps per CTA of the last step
int res_debug_times(const ResPlan* rp, long long* out, long long cap);

cudaError_t res_step(const ResPlan* rp, const float* g, float* e, float* work, float* Q, float* P, float* Phat,
                     const double* repl, const float* bias_g, float* bias_out, int* status, cudaStream_t st);

}  // namespace psgd
