// Internal launch helpers shared between the stencil kernels and the V-cycle plan.
#pragma once
#include "common.cuh"

namespace mgsr {

constexpr int kSmallN = 64;

int grid_for(int64_t work, int threads);
int scratch_alloc(void **ptr, size_t bytes, cudaStream_t st);   // API scratch from a library-private pool
int launch_gs(const double *p_in, double *p_out, double *tmp, FSrc fs, int n, double h2, int sweeps,
              int zero_init, double *rc, double *rc_mean, double *mean_out, void *red_ws, cudaStream_t st);
int launch_prolong_add(const double *c, int nc, int s, const double *base, const double *bshift, double *out,
                       double *mean_out, void *red_slot, cudaStream_t st);
int launch_add2(const double *base, const double *bshift, const double *up, const double *ushift, double *out,
                int64_t count, double *mean_out, void *red_slot, cudaStream_t st);
int launch_res_restrict(const double *p, FSrc fs, int n, int s, double *rc, double *rc_mean, void *red_slot,
                        cudaStream_t st);
int launch_finalize(const double *out, const double *mean_ptr, double *p, FSrc fs, int n, double *acc3,
                    double *stats2, void *red_slot, cudaStream_t st);
bool prolong_finalize_applies(int n);
int launch_prolong_finalize(const double *S, const double *bshift, const double *c, int nc, const double *out_mean,
                            double *p, FSrc fs, double *acc3, double *stats2, void *red_slot, cudaStream_t st);
int launch_affine(const double *a, double *out, int64_t count, const double *shift, double scale, cudaStream_t st);
// correction of a whole ratio-2 sub-ladder with sides[0] <= kSmallN in one CTA (spline prolongation)
// a whole spline V-cycle + logging pass of a ratio-2 ladder with sides[0] <= kSmallN in one CTA
int launch_vcycle_small(double *p, const double *f, const int *sides, int nlev, int n_smooth, int coarse_sweeps,
                        double *stats, cudaStream_t st);
int launch_correction_small(const double *rc0, const double *rc0_mean, double *d0, const int *sides, int nlev,
                            int n_smooth, int coarse_sweeps, cudaStream_t st);

}  // namespace mgsr
