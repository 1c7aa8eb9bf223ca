/* mgsr_b200 -- C ABI of the B200-native V-cycle hot path.
 *
 * Drop-in boundary for the reference package ``mgsr`` (arXiv 2403.07936
 * reference, /root/reference/pkg/src/mgsr).  Every entry point is
 * ``extern "C"``, takes plain device pointers and sizes (fp64 row-major n x n
 * grids unless stated), a ``cudaStream_t`` passed as ``void*`` LAST, and
 * returns an ``int`` status: 0 = ok, negative = error (see MGSR_E_*; the
 * Python shim maps them to the reference's ValueError texts).  Caller owns
 * all buffers; handles are immutable after creation except the V-cycle plan,
 * which owns its level buffers and captured graphs.  No global mutable state.
 *
 * Each declaration names the reference interface it replaces (file:line).
 */
#ifndef MGSR_B200_H
#define MGSR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    MGSR_OK = 0,
    MGSR_E_ODD_SIDE = -1,      /* "red-black coloring needs an even side"   (_stencil.pyx:15-16) */
    MGSR_E_BAD_ARG = -2,       /* negative sweeps, n < 2, null pointer        (smoother.py:68-69)  */
    MGSR_E_RATIO = -3,         /* "transfer ratio must be a power of two"     (transfer.py:22-24)  */
    MGSR_E_NOT_DIVISIBLE = -4, /* "fine side ... is not divisible by ratio"   (transfer.py:34-35)  */
    MGSR_E_PROLONG_RATIO = -5, /* "prolongation ratio must be one of"         (transfer.py:71-72)  */
    MGSR_E_SR_RATIO = -6,      /* "unsupported SR ratio"                      (srmodel.py:479-480) */
    MGSR_E_WINDOW = -7,        /* coarse side must be >= 6 and even           (srmodel.py:416-419) */
    MGSR_E_CUDA = -8,          /* CUDA runtime error (message via mgsr_last_error) */
    MGSR_E_WORKSPACE = -9,     /* workspace too small                                            */
    MGSR_E_UNSUPPORTED = -10,  /* configuration not supported by this build                      */
    MGSR_E_LADDER = -11        /* "no valid ladder"                           (solver.py:107-117)  */
};

/* Last error text of the calling thread (thread-local, never NULL). */
const char *mgsr_last_error(void);
/* Build/version string; also proves the library loads. */
const char *mgsr_version(void);

/* ---- stencil kernels: the MGSR_BACKEND plugin point (kernels/__init__.py:35-49) ---- */

/* Bytes of device workspace mgsr_gs_sweeps / mgsr_residual / mgsr_restrict need for side n.
 * Any contents: each call resets the reduction tickets it uses (stream-ordered). */
size_t mgsr_workspace_bytes(int64_t n);

/* API scratch (mgsr_gs_sweeps' temporary, mgsr_generator_forward's buffers) comes from a memory pool
 * private to this library, one per device, which keeps freed blocks mapped; the process-wide default
 * pool is never modified. */

/* In-place red-black Gauss-Seidel, red=(i+j) even first, mean subtracted
 * (deferred to once per call; <=6e-16 from per-sweep).
 * Replaces kernels.gs_sweeps(p, f, h2, sweeps)  (_stencil.pyx:12-45). */
int mgsr_gs_sweeps(double *p, const double *f, int64_t n, double h2, int32_t sweeps,
                   void *ws, size_t ws_bytes, void *stream);

/* out = (nb - 4p) * inv_h2, periodic; any n >= 2.
 * Replaces kernels.laplacian(p, inv_h2)  (_stencil.pyx:48-63). */
int mgsr_laplacian(const double *p, double *out, int64_t n, double inv_h2, void *stream);

/* r = f - L p, then r -= mean(r).  Replaces smoother.residual (smoother.py:52-57). */
int mgsr_residual(const double *p, const double *f, double *r, int64_t n,
                  void *ws, size_t ws_bytes, void *stream);

/* coarse = fine[::s, ::s] (- its mean if subtract_mean).
 * Replaces transfer.restrict (transfer.py:27-39). */
int mgsr_restrict(const double *fine, double *coarse, int64_t n, int32_t s, int32_t subtract_mean,
                  void *ws, size_t ws_bytes, void *stream);

/* out (nc*s)^2 = separable periodic Keys(a=-1/2) interpolation of c (nc^2).
 * Replaces transfer.spline_prolong (transfer.py:64-74). */
int mgsr_spline_prolong(const double *c, int64_t nc, int32_t s, double *out, void *stream);

/* Reductions used by Grid.rms / diff_norm (grid.py:67-78): out[0] = sqrt(mean((a-b)^2))
 * (b may be NULL -> rms(a)). Deterministic fixed-order reduction.  The result is a HOST value,
 * so this call synchronises `stream` (the reference returns a Python float, grid.py:74-78);
 * the V-cycle plan computes its norms on the device without synchronising. */
int mgsr_rms_diff(const double *a, const double *b, int64_t count, double *out_host,
                  void *ws, size_t ws_bytes, void *stream);

/* ---- generator (srmodel.py:90-487) ---- */

typedef struct mgsr_gen mgsr_gen;

enum { MGSR_PREC_FP32 = 0, MGSR_PREC_BF16 = 1, MGSR_PREC_FP16 = 2, MGSR_PREC_MIXED = 3 };

/* Build an immutable generator from the MGSR1 tensor set (host float32 arrays in
 * the canonical order of expected_tensor_shapes(B), srmodel.py:90-114), i.e.
 * head.conv.weight, head.prelu.alpha, res{i}.{conv1.weight, bn1.gamma, bn1.beta,
 * bn1.mean, bn1.var, prelu.alpha, conv2.weight, bn2.gamma, bn2.beta, bn2.mean,
 * bn2.var} for i < B, post.conv.weight, post.bn.{gamma,beta,mean,var},
 * up.conv.weight, up.prelu.alpha, tail.conv.weight, tail.conv.bias.
 * Replaces srmodel.GeneratorWeights / load_weights (srmodel.py:117-248). */
int mgsr_generator_create(const float *const *tensors, int32_t num_tensors, int32_t blocks,
                          double tanh_scale, mgsr_gen **out);
int mgsr_generator_destroy(mgsr_gen *g);

/* y (N,3,2h,2h) = generator(x (N,3,h,h)), fp64 in/out, any h >= 1 (fp32 compute).
 * Replaces srmodel.generator_forward / _forward_batch (srmodel.py:330-354). */
int mgsr_generator_forward(const mgsr_gen *g, const double *x, int64_t batch, int64_t side,
                           double *y, void *stream);

/* Windowed SR prolongation by s in {2,4,8,16}: normalise, 6x6 windows at
 * stride 2, generator, channel mean, stitch, denormalise with output signs,
 * mean-subtract (per pass).  precision: MGSR_PREC_FP32 (CUDA-core fp32),
 * MGSR_PREC_BF16 / MGSR_PREC_FP16 (tcgen05 megakernel with bf16 / fp16 operands,
 * fp32 accumulation; ratio-2 passes and ratio-4 passes), MGSR_PREC_MIXED (fp16
 * tensor cores, except the first pass of a two-pass ratio x8 / x16, which runs in
 * fp32: the second pass re-normalises its output logarithmically and amplifies its
 * operand rounding ~25x).
 * Replaces srmodel.sr_prolong (srmodel.py:470-487). */
size_t mgsr_sr_workspace_bytes(int64_t nc, int32_t s);
int mgsr_sr_prolong(const mgsr_gen *g, const double *c, int64_t nc, int32_t s,
                    double p_min, double p_max, int32_t precision, double *out,
                    void *ws, size_t ws_bytes, void *stream);

/* ---- V-cycle driver (solver.py:100-330) ---- */

typedef struct mgsr_plan mgsr_plan;

typedef struct {
    int64_t n;             /* fine side */
    int32_t n_step;        /* RunConfig.N_step */
    int32_t r_min;         /* RunConfig.r_min */
    int32_t n_smooth;      /* RunConfig.N_smooth */
    int32_t coarse_sweeps; /* RunConfig.coarse_sweeps */
    double p_min, p_max;   /* RunConfig.p_min / p_max (SR normalisation band) */
    int32_t precision;     /* MGSR_PREC_* for SR prolongations */
    uint32_t sr_level_mask;/* bit l set: prolongation from level l+1 into level l may use SR
                              when the cycle's operator is "sr" (all ones = reference behaviour) */
} mgsr_plan_config;

/* Plan: level ladder (solver.py:100-119), per-level buffers, and one CUDA graph
 * per operator variant captured on first use.  gen may be NULL (spline only). */
int mgsr_plan_create(const mgsr_plan_config *cfg, const mgsr_gen *gen, mgsr_plan **out);
int mgsr_plan_destroy(mgsr_plan *plan);
int32_t mgsr_plan_levels(const mgsr_plan *plan, int64_t *sides_out /* >= 32 entries */);

/* One V-cycle on iterate p (in place) with RHS f, then the solve-loop logging
 * pass: stats[0] = diff_norm(new_p, old_p), stats[1] = residual(new_p).rms()
 * (solver.py:311-313), written to the device buffer stats_dev (2 doubles).
 * use_sr: 0 -> operator "spline", 1 -> operator "sr".  One graph launch.
 * Replaces solver.v_cycle (solver.py:158-197) + solver.py:312-313. */
int mgsr_plan_vcycle(mgsr_plan *plan, double *p, const double *f, int32_t use_sr,
                     double *stats_dev, void *stream);

/* Device-resident solve loop: up to n_iter V-cycles in ONE graph launch (a WHILE
 * conditional node; per iteration the operator follows schedule_operator and the
 * latch rule on device, the cycle runs, and the logging pass's stats are
 * recorded).  mode: 0 spline, 1 sr, 2 hybrid.  Hybrid cadence: cadence =
 * max(1, round(N_GAN)) (or of 1/N_GAN), first_sr = 1 when N_GAN >= 1, ngan_one =
 * (N_GAN == 1).  records_dev: n_iter x 4 doubles (diff_norm, residual rms,
 * operator 1=sr/0=spline, latched before the iteration); iterations_dev: one
 * int32, the number of iterations run (stop when diff_norm < tol).
 * Replaces solver.solve's loop (solver.py:280-330). */
int mgsr_plan_solve(mgsr_plan *plan, double *p, const double *f, int32_t mode, int32_t n_iter, double tol,
                    double s_thres, int32_t cadence, int32_t first_sr, int32_t ngan_one,
                    double *records_dev, int32_t *iterations_dev, void *stream);

/* Batched device-resident solves (BASELINE config 5; the reference fans independent
 * solves out over processes, cli.py:202-250): B plans of one configuration and
 * generator (plans[b] with its iterate p[b] and RHS f[b]) run their solve loops in
 * lockstep inside ONE graph launch, each with its own operator schedule, latch and
 * stopping rule, and every SR level's generator runs as ONE persistent launch over
 * the windows of all grids that prolong by SR in that iteration.  Each grid sees
 * its mgsr_plan_solve kernel sequence, so p[b] and its records are bitwise those
 * of mgsr_plan_solve.  records_dev: B x n_iter x 4 doubles; iterations_dev: B
 * int32.  1 <= B <= 1024. */
int mgsr_plan_solve_batch(mgsr_plan *const *plans, int32_t B, double *const *p, const double *const *f,
                          int32_t mode, int32_t n_iter, double tol, double s_thres, int32_t cadence,
                          int32_t first_sr, int32_t ngan_one, double *records_dev, int32_t *iterations_dev,
                          void *stream);

/* Instrumentation for bench.py.  mgsr_plan_timing_enable(plan, k): the next k
 * V-cycle launches record CUDA events (event-record nodes inside the graph,
 * re-targeted per launch) around (0) the finest-level generator kernel,
 * (1) the finest-level Gauss-Seidel kernel, (2) the whole cycle.
 * mgsr_plan_timing_read: synchronises those events and returns the mean
 * duration in ms of each over the recorded launches (0 when absent). */
int mgsr_plan_timing_enable(mgsr_plan *plan, int32_t max_launches);
int mgsr_plan_timing_read(mgsr_plan *plan, double *ms_out /* 3 */, int32_t *launches_out);
/* Number of kernel nodes in the captured graph of an operator (0 if not captured yet). */
int32_t mgsr_plan_kernel_nodes(mgsr_plan *plan, int32_t use_sr);

/* ---- seeded start of solve() (solver.py:298-300) ---- */

/* out[i] = U_i - mean(U) with U_i = low + (high - low) * d_i, d_i the i-th double of
 * numpy's PCG64 stream whose 128-bit state / increment are default_rng(seed).bit_generator
 * .state (the SeedSequence hashing stays on the host), mean = numpy's pairwise sum / count.
 * Bit-exact with np.random.default_rng(seed).uniform(low, high, count) minus its .mean().
 * count must be a power of two >= 128.  Replaces the host draw of solver.py:298-300. */
size_t mgsr_initial_iterate_workspace_bytes(int64_t count);
int mgsr_initial_iterate(double *out, int64_t count, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                         uint64_t inc_lo, double low, double high, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MGSR_B200_H */
