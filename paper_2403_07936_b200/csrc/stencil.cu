// fp64 stencil kernels of the V-cycle: red-black Gauss-Seidel (temporally
// blocked: TMA-fed windows relaxed in registers on the large levels, whole
// grids in one CTA's shared memory at the bottom of the ladder), fused
// residual -> half-injection restriction, Keys spline prolongation fused with
// the correction add, and the solve-loop logging pass.  Compiled with --fmad=false so every product and
// sum rounds exactly as the reference's -ffp-contract=off C loops
// (pkg/setup.py:37-39).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "stencil.cuh"

namespace mgsr {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }

__device__ __forceinline__ int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// t -> (t / d, t % d) with a shift when d is a power of two (every N_step = 1 ladder)
__device__ __forceinline__ void split_idx(int t, int d, int dsh, int &q, int &r) {
    if (dsh >= 0) { q = t >> dsh; r = t & (d - 1); }
    else { q = t / d; r = t - q * d; }
}
__device__ __forceinline__ int pow2_shift(int d) { return (d & (d - 1)) == 0 ? __ffs(d) - 1 : -1; }

// Row-parallel 2-D loops: threads of a block cover consecutive columns (coalesced), blocks
// stride over rows.  No per-element 64-bit division (which dominated the 1-D
// grid-stride versions: k_finalize ran at 1.3 TB/s on a 4096^2 grid).
#define MGSR_ROWS(i, nrows) for (int i = blockIdx.y; i < (nrows); i += gridDim.y)
#define MGSR_COLS(j, ncols) for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < (ncols); j += gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// Gauss-Seidel.  Reference: _stencil.pyx:25-37 -- per cell
//   nb = ((p[i-1,j] + p[i+1,j]) + p[i,j-1]) + p[i,j+1];  p = (nb - h2 f) * 0.25
// red (i+j even) cells first, then black.  The per-sweep mean subtraction of
// _stencil.pyx:38-45 commutes with the update up to rounding (SURVEY §0.9:
// <= 6e-16), so it is deferred: the kernels compute the raw iterate and the
// grid sum of the last sweep; consumers subtract that mean.

// One colour over the whole grid, in place (global memory).  Used for the
// small/medium levels; every cell of the colour is independent.
__global__ void k_gs_half(double *__restrict__ p, FSrc fs, int n, double h2, int color) {
    const int half = n >> 1;
    const double sh = fs.load_shift();
    MGSR_ROWS(i, n) {
        const int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        MGSR_COLS(k, half) {
            int j = 2 * k + ((i + color) & 1);
            int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
            int64_t c = int64_t(i) * n + j;
            double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[int64_t(i) * n + jm1]) +
                        p[int64_t(i) * n + jp1];
            p[c] = (nb - h2 * fs.at(c, sh)) * 0.25;
        }
    }
}

// Sum of a grid -> result[0] = mean (deterministic).
__global__ void k_mean(const double *__restrict__ a, int64_t count, RedSlot slot, double *result) {
    double v[1] = {0.0};
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count;
         t += int64_t(gridDim.x) * blockDim.x)
        v[0] += a[t];
    grid_reduce<1>(v, slot, result, 1.0 / double(count));
}

// ---------------------------------------------------------------------------
// Whole coarse sub-ladder in ONE CTA: correction(rhs, l) of solver.py:181-190 for
// a level with side <= kSmallN and every level below it (ratio-2 ladder, spline
// prolongation).  Per level: GS from zero with the exact per-sweep mean
// subtraction (_stencil.pyx:38-45), the residual at the injected points and its
// half-injection 0.5 (r - mean(r)) as the next level's RHS; the coarsest level
// relaxes coarse_sweeps times; then each level adds the Keys ratio-2
// prolongation of the level below (the k_prolong2_add arithmetic).  Replaces
// ~4 launches per level on the latency-bound bottom of every V-cycle.
constexpr int kSmallMaxLev = 8;
constexpr int kSmallThreads = 256;   // fewer, busier threads: the bottom levels are latency- and issue-bound

struct SmallLadder {
    int nlev;
    int side[kSmallMaxLev];
};

__device__ double block_sum_1024(double v, double *sred) {
    const int tid = threadIdx.x, nt = blockDim.x;
    v = warp_sum(v);
    __syncthreads();
    if ((tid & 31) == 0) sred[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
        double w = tid < (nt >> 5) ? sred[tid] : 0.0;
        w = warp_sum(w);
        if (tid == 0) sred[32] = w;
    }
    __syncthreads();
    return sred[32];
}

// GS sweeps from the current contents of sp with the exact per-sweep mean subtraction
// (_stencil.pyx:25-45), whole grid in one CTA's shared memory.
__device__ void small_gs(double *sp, const double *sf, int n, double h2, int sweeps, double *sred) {
    const int tid = threadIdx.x, nt = blockDim.x, nn = n * n, half = nn >> 1;
    const int hn = n >> 1, hsh = pow2_shift(hn);
    for (int s = 0; s < sweeps; ++s) {
        for (int color = 0; color < 2; ++color) {
            for (int t = tid; t < half; t += nt) {
                int i, k;
                split_idx(t, hn, hsh, i, k);
                int jj = 2 * k + ((i + color) & 1);
                int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
                int jm1 = jj > 0 ? jj - 1 : n - 1, jp1 = jj < n - 1 ? jj + 1 : 0;
                double nb = ((sp[im1 * n + jj] + sp[ip1 * n + jj]) + sp[i * n + jm1]) + sp[i * n + jp1];
                sp[i * n + jj] = (nb - h2 * sf[i * n + jj]) * 0.25;
            }
            __syncthreads();
        }
        double acc = 0.0;
        for (int c = tid; c < nn; c += nt) acc += sp[c];
        const double mean = block_sum_1024(acc, sred) * (1.0 / double(nn));
        for (int c = tid; c < nn; c += nt) sp[c] -= mean;
        __syncthreads();
    }
}

// The same sweeps with the mean subtracted once at the end: Gauss-Seidel is shift-equivariant (every update
// (sum of neighbours - h^2 f) / 4 moves by c when all values move by c), so the per-sweep subtractions add up
// to subtracting the final mean (the deferred-mean identity, as k_gs_rb uses it).  Saves four
// barriers and two passes per sweep on the latency-bound bottom of the ladder.
__device__ void small_gs_deferred(double *sp, const double *sf, int n, double h2, int sweeps, double *sred) {
    const int tid = threadIdx.x, nt = blockDim.x, nn = n * n, half = nn >> 1;
    const int hn = n >> 1, hsh = pow2_shift(hn);
    for (int s = 0; s < sweeps; ++s) {
        for (int color = 0; color < 2; ++color) {
            for (int t = tid; t < half; t += nt) {
                int i, k;
                split_idx(t, hn, hsh, i, k);
                int jj = 2 * k + ((i + color) & 1);
                int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
                int jm1 = jj > 0 ? jj - 1 : n - 1, jp1 = jj < n - 1 ? jj + 1 : 0;
                double nb = ((sp[im1 * n + jj] + sp[ip1 * n + jj]) + sp[i * n + jm1]) + sp[i * n + jp1];
                sp[i * n + jj] = (nb - h2 * sf[i * n + jj]) * 0.25;
            }
            __syncthreads();
        }
    }
    double acc = 0.0;
    for (int c = tid; c < nn; c += nt) acc += sp[c];
    const double mean = block_sum_1024(acc, sred) * (1.0 / double(nn));
    for (int c = tid; c < nn; c += nt) sp[c] -= mean;
    __syncthreads();
}

// Raw residual f - L p at the injected (even, even) points of an n-grid -> fr (n/2 x n/2); returns
// the mean (block sum).  Arithmetic of k_res_restrict / the fused residual of k_gs_rb.
__device__ double small_residual_inject(const double *sp, const double *sf, int n, double *fr, double *sred) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const double h = 2.0 * M_PI / n, inv_h2 = 1.0 / (h * h);
    const int nc = n >> 1, ncc = nc * nc, csh = pow2_shift(nc);
    double acc = 0.0;
    for (int t = tid; t < ncc; t += nt) {
        int ic, jc;
        split_idx(t, nc, csh, ic, jc);
        const int i = 2 * ic, jj = 2 * jc;
        const int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        const int jm1 = jj > 0 ? jj - 1 : n - 1, jp1 = jj < n - 1 ? jj + 1 : 0;
        const int c = i * n + jj;
        double nb = ((sp[im1 * n + jj] + sp[ip1 * n + jj]) + sp[i * n + jm1]) + sp[i * n + jp1];
        const double res = sf[c] - ((nb - 4.0 * sp[c]) * inv_h2);
        fr[t] = res;
        acc += res;
    }
    return block_sum_1024(acc, sred) * (1.0 / double(ncc));
}

// out (2nc x 2nc) += Keys ratio-2 prolongation of c (k_prolong2_add arithmetic, base shift 0)
__device__ void small_prolong2_add(const double *c, int nc, double *out) {
    const int tid = threadIdx.x, nt = blockDim.x, n = 2 * nc;
    const double w0 = -0.0625, w1 = 0.5625;
    const int csh = pow2_shift(nc);
    for (int t = tid; t < nc * nc; t += nt) {
        int bi, bj;
        split_idx(t, nc, csh, bi, bj);
        int ri[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            const int r = bi + o - 1;
            ri[o] = r < 0 ? r + nc : (r >= nc ? r - nc : r);
        }
        double R0[4], R1[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int cb = bj + b - 1;
            cb = cb < 0 ? cb + nc : (cb >= nc ? cb - nc : cb);
            const double c0 = c[ri[0] * nc + cb], c1 = c[ri[1] * nc + cb];
            const double c2 = c[ri[2] * nc + cb], c3 = c[ri[3] * nc + cb];
            R0[b] = c1;
            double row = 0.0;
            row += w0 * c0;
            row += w1 * c1;
            row += w1 * c2;
            row += w0 * c3;
            R1[b] = row;
        }
        double a01 = 0.0, a11 = 0.0;
        a01 += w0 * R0[0]; a01 += w1 * R0[1]; a01 += w1 * R0[2]; a01 += w0 * R0[3];
        a11 += w0 * R1[0]; a11 += w1 * R1[1]; a11 += w1 * R1[2]; a11 += w0 * R1[3];
        const int t0 = (2 * bi) * n + 2 * bj, t1 = t0 + n;
        out[t0] = (out[t0] - 0.0) + R0[1];
        out[t0 + 1] = (out[t0 + 1] - 0.0) + a01;
        out[t1] = (out[t1] - 0.0) + R1[1];
        out[t1 + 1] = (out[t1 + 1] - 0.0) + a11;
    }
    __syncthreads();
}

// The same three level operations with the side N a compile-time constant (the power-of-two sides of the
// N_step = 1 ladders: 64, 32, 16, 8): index arithmetic folds to shifts and masks and each thread's cells are
// an unrolled, fixed-count loop whose shared-memory loads issue together, instead of a runtime-bounded loop
// of dependent address computations.  Per cell the arithmetic is the generic functions', and every
// per-thread partial sum visits its cells in the same order, so results are bitwise identical.
template <int N>
__device__ __forceinline__ void small_level_down(double *sp, double *sf, int sweeps, double *fr, double *sred) {
    constexpr int NT = kSmallThreads, NN = N * N, HALF = NN / 2, HN = N / 2, NC = N / 2, NCC = NC * NC;
    const int tid = threadIdx.x;
    for (int it = 0; it < (NN + NT - 1) / NT; ++it)
        if (tid + it * NT < NN) sp[tid + it * NT] = 0.0;
    __syncthreads();
    const double h = 2.0 * M_PI / N, h2 = h * h;
#pragma unroll 1
    for (int s = 0; s < sweeps; ++s) {
#pragma unroll
        for (int color = 0; color < 2; ++color) {
#pragma unroll
            for (int it = 0; it < (HALF + NT - 1) / NT; ++it) {
                const int t = tid + it * NT;
                if (t < HALF) {
                    const int i = t / HN, k = t % HN;
                    const int jj = 2 * k + ((i + color) & 1);
                    const int im1 = (i + N - 1) % N, ip1 = (i + 1) % N, jm1 = (jj + N - 1) % N, jp1 = (jj + 1) % N;
                    double nb = ((sp[im1 * N + jj] + sp[ip1 * N + jj]) + sp[i * N + jm1]) + sp[i * N + jp1];
                    sp[i * N + jj] = (nb - h2 * sf[i * N + jj]) * 0.25;
                }
            }
            __syncthreads();
        }
    }
    {
        double acc = 0.0;
#pragma unroll
        for (int it = 0; it < (NN + NT - 1) / NT; ++it)
            if (tid + it * NT < NN) acc += sp[tid + it * NT];
        const double mean = block_sum_1024(acc, sred) * (1.0 / double(NN));
#pragma unroll
        for (int it = 0; it < (NN + NT - 1) / NT; ++it)
            if (tid + it * NT < NN) sp[tid + it * NT] -= mean;
        __syncthreads();
    }
    if (!fr) return;
    const double inv_h2 = 1.0 / (h * h);
    double acc = 0.0, res[(NCC + NT - 1) / NT];
#pragma unroll
    for (int it = 0; it < (NCC + NT - 1) / NT; ++it) {
        const int t = tid + it * NT;
        res[it] = 0.0;
        if (t < NCC) {
            const int i = 2 * (t / NC), jj = 2 * (t % NC);
            const int im1 = (i + N - 1) % N, ip1 = (i + 1) % N, jm1 = (jj + N - 1) % N, jp1 = (jj + 1) % N;
            const int c = i * N + jj;
            double nb = ((sp[im1 * N + jj] + sp[ip1 * N + jj]) + sp[i * N + jm1]) + sp[i * N + jp1];
            res[it] = sf[c] - ((nb - 4.0 * sp[c]) * inv_h2);
            acc += res[it];
        }
    }
    const double mean = block_sum_1024(acc, sred) * (1.0 / double(NCC));
#pragma unroll
    for (int it = 0; it < (NCC + NT - 1) / NT; ++it)
        if (tid + it * NT < NCC) fr[tid + it * NT] = (res[it] - mean) * 0.5;
    __syncthreads();
}

template <int NC>
__device__ __forceinline__ void small_prolong2_add_t(const double *c, double *out) {
    constexpr int NT = kSmallThreads, N = 2 * NC;
    const double w0 = -0.0625, w1 = 0.5625;
    const int tid = threadIdx.x;
#pragma unroll
    for (int it = 0; it < (NC * NC + NT - 1) / NT; ++it) {
        const int t = tid + it * NT;
        if (t >= NC * NC) continue;
        const int bi = t / NC, bj = t % NC;
        double R0[4], R1[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int cb = (bj + b - 1 + NC) % NC;
            const double c0 = c[((bi + NC - 1) % NC) * NC + cb], c1 = c[bi * NC + cb];
            const double c2 = c[((bi + 1) % NC) * NC + cb], c3 = c[((bi + 2) % NC) * NC + cb];
            R0[b] = c1;
            double row = 0.0;
            row += w0 * c0;
            row += w1 * c1;
            row += w1 * c2;
            row += w0 * c3;
            R1[b] = row;
        }
        double a01 = 0.0, a11 = 0.0;
        a01 += w0 * R0[0]; a01 += w1 * R0[1]; a01 += w1 * R0[2]; a01 += w0 * R0[3];
        a11 += w0 * R1[0]; a11 += w1 * R1[1]; a11 += w1 * R1[2]; a11 += w0 * R1[3];
        const int t0 = (2 * bi) * N + 2 * bj, t1 = t0 + N;
        out[t0] = (out[t0] - 0.0) + R0[1];
        out[t0 + 1] = (out[t0 + 1] - 0.0) + a01;
        out[t1] = (out[t1] - 0.0) + R1[1];
        out[t1 + 1] = (out[t1 + 1] - 0.0) + a11;
    }
    __syncthreads();
}

// correction(rhs, l) of solver.py:181-190 for a ratio-2 sub-ladder in shared memory: D[j], F[j]
// per level, F[0] filled by the caller; leaves the correction of level 0 in D[0].
__device__ void small_ladder(double *const *D, double *const *F, const SmallLadder &L, int n_smooth,
                             int coarse_sweeps, double *sred) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int j = 0; j < L.nlev; ++j) {
        const int n = L.side[j], nn = n * n;
        const int sweeps = j == L.nlev - 1 ? coarse_sweeps : n_smooth;
        double *const fr = j < L.nlev - 1 ? F[j + 1] : nullptr;
#ifndef MGSR_EXACT_SMALL_MEANS
        if (nt == kSmallThreads && (n == 64 || n == 32 || n == 16 || n == 8)) {
            if (n == 64) small_level_down<64>(D[j], F[j], sweeps, fr, sred);
            else if (n == 32) small_level_down<32>(D[j], F[j], sweeps, fr, sred);
            else if (n == 16) small_level_down<16>(D[j], F[j], sweeps, fr, sred);
            else small_level_down<8>(D[j], F[j], sweeps, fr, sred);
            continue;
        }
#endif
        for (int c = tid; c < nn; c += nt) D[j][c] = 0.0;
        __syncthreads();
        const double h = 2.0 * M_PI / n;
#ifdef MGSR_EXACT_SMALL_MEANS
        small_gs(D[j], F[j], n, h * h, sweeps, sred);
#else
        small_gs_deferred(D[j], F[j], n, h * h, sweeps, sred);
#endif
        if (fr) {   // residual at the injected points -> next RHS 0.5 (r - mean(r))
            const int ncc = (n >> 1) * (n >> 1);
            const double mean = small_residual_inject(D[j], F[j], n, fr, sred);
            for (int t = tid; t < ncc; t += nt) fr[t] = (fr[t] - mean) * 0.5;
            __syncthreads();
        }
    }
    for (int j = L.nlev - 2; j >= 0; --j) {   // ascend
        const int nc = L.side[j + 1];
        if (nt == kSmallThreads && nc == 32) small_prolong2_add_t<32>(D[j + 1], D[j]);
        else if (nt == kSmallThreads && nc == 16) small_prolong2_add_t<16>(D[j + 1], D[j]);
        else if (nt == kSmallThreads && nc == 8) small_prolong2_add_t<8>(D[j + 1], D[j]);
        else small_prolong2_add(D[j + 1], nc, D[j]);
    }
}

// Whole small grid in one CTA: all sweeps with the reference's per-sweep mean subtraction done
// exactly in order (block reduction).  n <= kSmallN.
__global__ void __launch_bounds__(kSmallThreads) k_gs_small(double *__restrict__ p, FSrc fs, int n, double h2,
                                                           int sweeps, int zero_init, double *mean_out) {
    extern __shared__ double sm[];
    double *sp = sm, *sf = sm + n * n;
    __shared__ double sred[33];
    const int tid = threadIdx.x, nt = blockDim.x, nn = n * n;
    const double sh = fs.load_shift();
    for (int c = tid; c < nn; c += nt) {
        sp[c] = zero_init ? 0.0 : p[c];
        sf[c] = fs.at(c, sh);
    }
    __syncthreads();
    small_gs(sp, sf, n, h2, sweeps, sred);
    for (int c = tid; c < nn; c += nt) p[c] = sp[c];
    if (tid == 0 && mean_out) *mean_out = 0.0;   // already gauge-fixed
}

__global__ void __launch_bounds__(kSmallThreads) k_correction_small(const double *__restrict__ rc0, const double *rc0_mean,
                                                           double *__restrict__ d0, SmallLadder L, int n_smooth,
                                                           int coarse_sweeps) {
    extern __shared__ double sm[];
    __shared__ double sred[33];
    const int tid = threadIdx.x, nt = blockDim.x;
    double *D[kSmallMaxLev], *F[kSmallMaxLev];
    {
        int off = 0;
        for (int j = 0; j < L.nlev; ++j) {
            const int nn = L.side[j] * L.side[j];
            D[j] = sm + off;
            F[j] = sm + off + nn;
            off += 2 * nn;
        }
    }
    {   // level 0 RHS: 0.5 * (rc0 - mean)
        const int nn = L.side[0] * L.side[0];
        const double m = *rc0_mean;
        for (int c = tid; c < nn; c += nt) F[0][c] = (rc0[c] - m) * 0.5;
    }
    small_ladder(D, F, L, n_smooth, coarse_sweeps, sred);
    const int nn = L.side[0] * L.side[0];
    for (int c = tid; c < nn; c += nt) d0[c] = D[0][c];
}

// A whole spline V-cycle of a small grid (side <= kSmallN, ratio-2 ladder) plus the solve loop's
// logging pass in ONE CTA (solver.py:158-197 + 311-313): N_smooth GS sweeps on p with the exact
// per-sweep mean, the injected residual, the sub-ladder correction, the Keys prolongation added,
// new p = out - mean(out), stats = (diff_norm, residual rms).  Same per-element arithmetic as the
// multi-kernel cycle; the means are block sums.  Replaces ~5 launches per cycle on config 1.
__global__ void __launch_bounds__(kSmallThreads) k_vcycle_small(double *__restrict__ p, const double *__restrict__ f,
                                                       SmallLadder L, int n_smooth, int coarse_sweeps,
                                                       double *stats) {
    extern __shared__ double sm[];
    __shared__ double sred[33];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int n = L.side[0], nn = n * n;
    double *P = sm, *S = sm + nn, *Fp = sm + 2 * nn;
    double *D[kSmallMaxLev], *F[kSmallMaxLev];
    SmallLadder Lc{};
    Lc.nlev = L.nlev - 1;
    {
        int off = 3 * nn;
        for (int j = 0; j < Lc.nlev; ++j) {
            Lc.side[j] = L.side[j + 1];
            const int m = Lc.side[j] * Lc.side[j];
            D[j] = sm + off;
            F[j] = sm + off + m;
            off += 2 * m;
        }
    }
    for (int c = tid; c < nn; c += nt) {
        P[c] = p[c];
        S[c] = P[c];
        Fp[c] = f[c];
    }
    __syncthreads();
    {
        const double h = 2.0 * M_PI / n;
        small_gs(S, Fp, n, h * h, n_smooth, sred);                       // S: gauge-fixed smoothed iterate
    }
    {
        const double rm = small_residual_inject(S, Fp, n, F[0], sred);   // level-1 RHS 0.5 (r - mean(r))
        const int ncc = (n >> 1) * (n >> 1);
        for (int t = tid; t < ncc; t += nt) F[0][t] = (F[0][t] - rm) * 0.5;
        __syncthreads();
    }
    small_ladder(D, F, Lc, n_smooth, coarse_sweeps, sred);
    small_prolong2_add(D[0], Lc.side[0], S);                             // out = (S - 0) + P(d1)
    double acc = 0.0;
    for (int c = tid; c < nn; c += nt) acc += S[c];
    const double m = block_sum_1024(acc, sred) * (1.0 / double(nn));
    const double h = 2.0 * M_PI / n, inv_h2 = 1.0 / (h * h);
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int c = tid; c < nn; c += nt) {
        const int i = c / n, j = c - i * n;
        const int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        const int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
        const double o = S[c];
        const double nb = ((S[im1 * n + j] + S[ip1 * n + j]) + S[i * n + jm1]) + S[i * n + jp1];
        const double np_ = o - m;
        const double d = np_ - P[c];
        const double r = Fp[c] - ((nb - 4.0 * o) * inv_h2);
        p[c] = np_;
        v0 += d * d;
        v1 += r;
        v2 += r * r;
    }
    v0 = block_sum_1024(v0, sred) * (1.0 / double(nn));
    v1 = block_sum_1024(v1, sred) * (1.0 / double(nn));
    v2 = block_sum_1024(v2, sred) * (1.0 / double(nn));
    if (tid == 0) {
        stats[0] = sqrt(v0);
        const double var = v2 - v1 * v1;
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
    }
}

// ---------------------------------------------------------------------------
// Temporally blocked K-sweep GS on the large levels (side >= 128): 2K half-sweeps on a
// window of the grid whose halo (HE >= 2K, +1 when the residual is fused) keeps the
// interior exact; HBM traffic is read p, f and write p once per K sweeps.  With RC the
// residual at the coarse (even, even) interior points is computed from the final values and
// written raw (half-injection input, solver.py:178-179).  Data movement:
//   * a 64 x 64 window (tile interior + an even halo HE >= 2K (+1 with RC)) of
//     p and f lands in shared memory by per-row cp.async.bulk copies (rows and
//     the column wrap of edge tiles split into <= 2 segments per row), tracked
//     by one mbarrier; as soon as the threads copied the window into registers,
//     the NEXT tile's window is requested, so HBM streams while this tile
//     relaxes (two CTAs per SM, each one tile ahead);
//   * thread (warp w, lane l) holds rows 8w..8w+7, columns 2l, 2l+1 of the
//     window in registers.  A half-sweep updates one cell per row (the colour
//     parity of a row is a compile-time constant because the window origin is
//     even): left/right neighbours come from the thread itself or lane l -+ 1
//     by shuffle, up/down from its own rows, and across warps from the rows
//     every warp publishes in shared memory after each half-sweep (one
//     barrier per half-sweep, double-buffered);
//   * interior written with 16-byte stores; tiles of the last row/column are
//     shifted inwards (x0 = n - TX) rather than masked: they recompute cells
//     of their neighbour bit for bit and only count their own cells in the sums.
#ifndef MGSR_RB_ROWS
#define MGSR_RB_ROWS 8
#endif
constexpr int kRbW = 64, kRbRows = MGSR_RB_ROWS, kRbWarps = kRbW / kRbRows, kRbThreads = 32 * kRbWarps, kRbMinN = 128,
              kRbMaxK = 4;
static_assert(kRbRows % 2 == 0 && kRbW % kRbRows == 0, "even rows per warp");

__device__ __forceinline__ void rb_mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void rb_bulk(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void rb_tma2d(uint32_t dst, const CUtensorMap *tm, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// The window of one tile -> shared memory; the barrier was armed with the byte count.  Windows inside the
// grid: one 2-D tensor copy per array (thread 0).  Windows that wrap (periodic edge tiles): per-row bulk
// copies, rows w * 8 .. w * 8 + 7 issued by lanes 0..7 of warp w, each row in one or two column segments.
__device__ __forceinline__ void rb_issue(const CUtensorMap *tm_p, const CUtensorMap *tm_f, const double *pin,
                                         const double *f, int n, int X0, int Y0, bool load_p, uint32_t sp,
                                         uint32_t sf, uint32_t bar, int w, int lane) {
    if (X0 >= 0 && Y0 >= 0 && X0 + kRbW <= n && Y0 + kRbW <= n) {
        if (w == 0 && lane == 0) {
            rb_tma2d(sf, tm_f, X0, Y0, bar);
            if (load_p) rb_tma2d(sp, tm_p, X0, Y0, bar);
        }
        return;
    }
    if (lane >= kRbRows) return;
    const int r = w * kRbRows + lane;
    int gy = Y0 + r;
    gy = gy < 0 ? gy + n : (gy >= n ? gy - n : gy);
    const int64_t row = int64_t(gy) * n;
    const uint32_t so = uint32_t(r * kRbW * 8);
    // column segments [X0, X0 + 64) mod n: one or two contiguous pieces (all even -> 16-byte aligned)
    int a0 = X0, len0 = kRbW, len1 = 0;
    if (X0 < 0) { a0 = X0 + n; len0 = -X0; len1 = kRbW + X0; }
    else if (X0 + kRbW > n) { len0 = n - X0; len1 = kRbW - len0; }
    rb_bulk(sf + so, f + row + a0, uint32_t(len0 * 8), bar);
    if (len1) rb_bulk(sf + so + uint32_t(len0 * 8), f + row, uint32_t(len1 * 8), bar);
    if (load_p) {
        rb_bulk(sp + so, pin + row + a0, uint32_t(len0 * 8), bar);
        if (len1) rb_bulk(sp + so + uint32_t(len0 * 8), pin + row, uint32_t(len1 * 8), bar);
    }
}

template <int K, bool RC>
__global__ void __launch_bounds__(kRbThreads, 2)
    k_gs_rb(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_f,
            const double *__restrict__ pin, double *__restrict__ pout, FSrc fs, int n, double h2, int zero_init,
            double inv_h2, double *__restrict__ rc, RedSlot slot, double *mean_out, double *rc_mean_out) {
    constexpr int H = 2 * K + (RC ? 1 : 0);
    constexpr int HE = (H + 1) & ~1;            // even: 16-byte aligned rows, fixed colour parity per row
    constexpr int TX = kRbW - 2 * HE, TY = kRbW - 2 * HE;
    constexpr int R = kRbRows;
    extern __shared__ __align__(128) double sm[];
    double *const sp = sm;                        // [64][64] p window
    double *const sf = sm + kRbW * kRbW;          // [64][64] f window
    double *const xb = sm + 2 * kRbW * kRbW;      // [2][warps][2][32] published boundary cells
    __shared__ __align__(8) uint64_t bar_storage;
    const uint32_t bar = uint32_t(__cvta_generic_to_shared(&bar_storage));
    const uint32_t sp_a = uint32_t(__cvta_generic_to_shared(sp)), sf_a = uint32_t(__cvta_generic_to_shared(sf));
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const double sh = fs.load_shift();
    const bool shifted = fs.shift != nullptr;
    const int tiles_x = (n + TX - 1) / TX, tiles_y = (n + TY - 1) / TY, ntiles = tiles_x * tiles_y;
    const bool load_p = !zero_init;
    const uint32_t tx_bytes = uint32_t(kRbW * kRbW * 8) * (load_p ? 2u : 1u);
    auto origin = [&](int tile, int &x0, int &y0, int &xs, int &ys) {
        const int by = tile / tiles_x, bx = tile - by * tiles_x;
        xs = bx * TX;
        ys = by * TY;
        x0 = min(xs, n - TX);
        y0 = min(ys, n - TY);
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0 && int(blockIdx.x) < ntiles)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx_bytes) : "memory");
    __syncthreads();
    if (int(blockIdx.x) < ntiles) {
        int x0, y0, xs, ys;
        origin(blockIdx.x, x0, y0, xs, ys);
        rb_issue(&tm_p, &tm_f, pin, fs.f, n, x0 - HE, y0 - HE, load_p, sp_a, sf_a, bar, w, lane);
    }
    double v[2] = {0.0, 0.0};
    uint32_t phase = 0;
#pragma unroll 1
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int x0, y0, xs, ys;
        origin(tile, x0, y0, xs, ys);
        double p[R][2], f[R][2], hu[2], hd[2];
        rb_mbar_wait(bar, phase);
        phase ^= 1u;
        {
            const int c2 = 2 * lane;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int o = (w * R + r) * kRbW + c2;
                const double2 ff = *reinterpret_cast<const double2 *>(sf + o);
                f[r][0] = shifted ? (ff.x - sh) * fs.scale : ff.x;
                f[r][1] = shifted ? (ff.y - sh) * fs.scale : ff.y;
                if (load_p) {
                    const double2 pp = *reinterpret_cast<const double2 *>(sp + o);
                    p[r][0] = pp.x;
                    p[r][1] = pp.y;
                } else {
                    p[r][0] = 0.0;
                    p[r][1] = 0.0;
                }
            }
            hu[0] = hu[1] = hd[0] = hd[1] = 0.0;
            if (load_p) {
                if (w > 0) {
                    const double2 t = *reinterpret_cast<const double2 *>(sp + (w * R - 1) * kRbW + c2);
                    hu[0] = t.x;
                    hu[1] = t.y;
                }
                if (w < kRbWarps - 1) {
                    const double2 t = *reinterpret_cast<const double2 *>(sp + (w * R + R) * kRbW + c2);
                    hd[0] = t.x;
                    hd[1] = t.y;
                }
            }
        }
        const bool more = tile + int(gridDim.x) < ntiles;
        // arm the next phase before the barrier: every thread has passed this phase's wait by then, and
        // no copy of the next window can complete before it is issued below
        if (tid == 0 && more)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx_bytes) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();   // window consumed: the next tile's copies may overwrite it
        if (more) {
            int nx0, ny0, nxs, nys;
            origin(tile + gridDim.x, nx0, ny0, nxs, nys);
            rb_issue(&tm_p, &tm_f, pin, fs.f, n, nx0 - HE, ny0 - HE, load_p, sp_a, sf_a, bar, w, lane);
        }
        // 2K half-sweeps; red (global (i + j) even) first.  The window origin (x0 - HE, y0 - HE) is even,
        // so in window row r (even w * R) the colour-c cell of a thread's pair is element (c + r) & 1.
#pragma unroll
        for (int hs = 0; hs < 2 * K; ++hs) {
            const int c = hs & 1;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int e = (c + r) & 1;
                const double up = r > 0 ? p[r - 1][e] : hu[e];
                const double dn = r < R - 1 ? p[r + 1][e] : hd[e];
                double left, right;
                if (e == 0) {
                    left = __shfl_up_sync(0xffffffffu, p[r][1], 1);
                    right = p[r][1];
                } else {
                    left = p[r][0];
                    right = __shfl_down_sync(0xffffffffu, p[r][0], 1);
                }
                const double nb = ((up + dn) + left) + right;
                p[r][e] = (nb - h2 * f[r][e]) * 0.25;
            }
            if (hs < 2 * K - 1 || RC) {   // publish the boundary rows for the next half-sweep (or the residual)
                // only the cells this half-sweep updated change: row 0's element c and row R-1's element
                // (c + R - 1) & 1 = 1 - c (R even) -- exactly the neighbours the next half-sweep (colour
                // 1 - c) reads across the warp boundaries (and the residual's up neighbours)
                double *xo = xb + (hs & 1) * (kRbWarps * 64);
                xo[(w * 2 + 0) * 32 + lane] = p[0][c];
                xo[(w * 2 + 1) * 32 + lane] = p[R - 1][1 - c];
                __syncthreads();
                if (w > 0) hu[1 - c] = xo[((w - 1) * 2 + 1) * 32 + lane];
                if (w < kRbWarps - 1) hd[c] = xo[((w + 1) * 2 + 0) * 32 + lane];
            }
        }
        // interior: window rows [HE, HE + TY), columns [HE, HE + TX)
        const bool col_in = 2 * lane >= HE && 2 * lane < HE + TX;
        const int gj = x0 + 2 * lane - HE;
        const bool col_own = col_in && gj >= xs;   // cells this tile counts (shifted edge tiles overlap)
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int lr = w * R + r;
            const bool row_in = lr >= HE && lr < HE + TY;
            const int gi = y0 + lr - HE;
            if (row_in && col_in) {
                *reinterpret_cast<double2 *>(pout + int64_t(gi) * n + gj) = make_double2(p[r][0], p[r][1]);
                if (col_own && gi >= ys) v[0] += p[r][0] + p[r][1];
            }
            if (RC && !(r & 1)) {
                // (even, even) cell = element 0 of an even row: colour 0; neighbours are the final black values
                const double left = __shfl_up_sync(0xffffffffu, p[r][1], 1);
                const double up = r > 0 ? p[r - 1][0] : hu[0];
                const double dn = p[r + 1][0];
                if (row_in && col_in) {
                    const double nb = ((up + dn) + left) + p[r][1];
                    const double res = f[r][0] - ((nb - 4.0 * p[r][0]) * inv_h2);
                    rc[int64_t(gi >> 1) * (n >> 1) + (gj >> 1)] = res;
                    if (col_own && gi >= ys) v[1] += res;
                }
            }
        }
    }
    double *const outs[2] = {mean_out, RC ? rc_mean_out : nullptr};
    const double scales[2] = {1.0 / (double(n) * double(n)), 4.0 / (double(n) * double(n))};
    grid_reduce_to<2>(v, slot, outs, scales);
}

// ---------------------------------------------------------------------------
// Residual / restriction.  Reference: smoother.py:52-57 (r = f - L p, minus
// mean) and transfer.py:27-39 (coarse = fine[::s, ::s] minus mean).  Inside
// the V-cycle only the injected points are needed; dropping the fine-grid mean
// changes the coarse RHS by <= 8.7e-17 relative.
__global__ void k_res_restrict(const double *__restrict__ p, FSrc fs, int n, int s, double inv_h2,
                               double *__restrict__ rc, RedSlot slot, double *mean_out) {
    const int nc = n / s;
    const int64_t total = int64_t(nc) * nc;
    const double sh = fs.load_shift();
    double v[1] = {0.0};
    MGSR_ROWS(ic, nc) {
        const int i = ic * s;
        const int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        MGSR_COLS(jc, nc) {
            int j = jc * s;
            int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
            int64_t c = int64_t(i) * n + j;
            double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[int64_t(i) * n + jm1]) +
                        p[int64_t(i) * n + jp1];
            double res = fs.at(c, sh) - ((nb - 4.0 * p[c]) * inv_h2);
            rc[int64_t(ic) * nc + jc] = res;
            v[0] += res;
        }
    }
    grid_reduce<1>(v, slot, mean_out, 1.0 / double(total));
}

// Full-grid laplacian (API kernel; reference kernels.laplacian).
__global__ void k_laplacian(const double *__restrict__ p, double *__restrict__ out, int n, double inv_h2) {
    MGSR_ROWS(i, n) {
        const int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        MGSR_COLS(j, n) {
            int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
            int64_t t = int64_t(i) * n + j;
            double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[t - j + jm1]) + p[t - j + jp1];
            out[t] = (nb - 4.0 * p[t]) * inv_h2;
        }
    }
}

// r = f - L p (raw) and its mean; API residual then subtracts.
__global__ void k_residual_raw(const double *__restrict__ p, const double *__restrict__ f, double *__restrict__ r,
                               int n, double inv_h2, RedSlot slot, double *mean_out) {
    const int64_t total = int64_t(n) * n;
    double v[1] = {0.0};
    MGSR_ROWS(i, n) {
        const int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        MGSR_COLS(j, n) {
            int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
            int64_t t = int64_t(i) * n + j;
            double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[t - j + jm1]) + p[t - j + jp1];
            double res = f[t] - ((nb - 4.0 * p[t]) * inv_h2);
            r[t] = res;
            v[0] += res;
        }
    }
    grid_reduce<1>(v, slot, mean_out, 1.0 / double(total));
}

// a[i] = (a[i] - *shift) * scale  (or  out[i] = ... when out != a)
__global__ void k_affine(const double *__restrict__ a, double *__restrict__ out, int64_t count,
                         const double *shift, double scale) {
    const double sh = shift ? *shift : 0.0;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count;
         t += int64_t(gridDim.x) * blockDim.x)
        out[t] = (a[t] - sh) * scale;
}

// fine[::s, ::s] gather
__global__ void k_inject(const double *__restrict__ fine, double *__restrict__ coarse, int n, int s,
                         RedSlot slot, double *mean_out) {
    const int nc = n / s;
    const int64_t total = int64_t(nc) * nc;
    double v[1] = {0.0};
    MGSR_ROWS(ic, nc) MGSR_COLS(jc, nc) {
        double x = fine[int64_t(ic) * s * n + int64_t(jc) * s];
        coarse[int64_t(ic) * nc + jc] = x;
        v[0] += x;
    }
    grid_reduce<1>(v, slot, mean_out, 1.0 / double(total));
}

// ---------------------------------------------------------------------------
// Spline prolongation.  Reference transfer.py:42-74: the dense periodic
// operator op (n_f x n_c) has exactly four non-zeros per row, Keys(a=-1/2)
// weights of t - o for offsets o = -1..2 at columns (i/s + o) mod n_c with
// t = (i mod s)/s; spline_prolong = op @ c @ op.T.  Evaluated here in the
// separable banded form (<= 3.7e-16 from the dense sandwich),
// fused with the correction add  out = (base - *bshift) + P(c)  and, when
// slot is given, the grid sum of out.
__device__ __forceinline__ double keys_w(double d) {
    d = fabs(d);
    double near = (1.5 * d - 2.5) * d * d + 1.0;
    double far = ((-0.5 * d + 2.5) * d - 4.0) * d + 2.0;
    return d <= 1.0 ? near : (d < 2.0 ? far : 0.0);
}

__global__ void k_prolong_add(const double *__restrict__ c, int nc, int s, const double *__restrict__ base,
                              const double *bshift, double *__restrict__ out, RedSlot slot, double *mean_out,
                              int do_mean) {
    const int n = nc * s;
    const int64_t total = int64_t(n) * n;
    const double bsh = (base && bshift) ? *bshift : 0.0;
    const double inv_s = 1.0 / double(s);
    double v[1] = {0.0};
    MGSR_ROWS(I, n) MGSR_COLS(J, n) {
        const int64_t t = int64_t(I) * n + J;
        int bi = I / s, bj = J / s;
        double ti = double(I - bi * s) * inv_s, tj = double(J - bj * s) * inv_s;
        // numpy: frac / s with frac integer -> identical to (I mod s) * (1/s) only
        // for powers of two, which is all PROLONG_RATIOS allows.
        double wi[4], wj[4];
        int ri[4], cj[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            wi[o] = keys_w(ti - double(o - 1));
            wj[o] = keys_w(tj - double(o - 1));
            ri[o] = wrap(bi + o - 1, nc);
            cj[o] = wrap(bj + o - 1, nc);
        }
        // op @ c first (rows), then @ op.T (columns): out = sum_b wj[b] * (sum_a wi[a] c[ra, cb])
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            double row = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) row += wi[a] * c[int64_t(ri[a]) * nc + cj[b]];
            acc += wj[b] * row;
        }
        double val = base ? (base[t] - bsh) + acc : acc;
        out[t] = val;
        v[0] += val;
    }
    if (do_mean) grid_reduce<1>(v, slot, mean_out, 1.0 / double(total));
}

// Ratios 4/8/16 (power of two, s <= 16): the same arithmetic as k_prolong_add with the Keys
// weights of each phase tabulated once per block (the phase is I mod s), the column's weights,
// indices and phase hoisted out of the row loop, and shifts instead of divisions.  Threads own
// a column J and walk rows, so the coarse neighbourhood is shared through L1 by the s threads of
// a coarse block.  Bitwise identical to k_prolong_add.
__global__ void k_prolong_add_pow2(const double *__restrict__ c, int nc, int s, int ssh, int ps,
                                   const double *__restrict__ base, const double *bshift, double *__restrict__ out,
                                   RedSlot slot, double *mean_out, int do_mean) {
    __shared__ double wtab[16][4];
    const int n = nc * s;
    const int64_t total = int64_t(n) * n;
    const double bsh = (base && bshift) ? *bshift : 0.0;
    const double inv_s = 1.0 / double(s);
    if (int(threadIdx.x) < 4 * s) {
        const int ph = threadIdx.x >> 2, o = threadIdx.x & 3;
        wtab[ph][o] = keys_w(double(ph) * inv_s - double(o - 1));
    }
    __syncthreads();
    double v[1] = {0.0};
    MGSR_COLS(J, n) {
        const int bj = J >> ssh, pj = J & (s - 1);
        double wj[4];
        int cj[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            wj[o] = wtab[pj][o];
            cj[o] = wrap(bj + o - 1, nc);
        }
        // item = (coarse row bi, a run of ps of its s fine rows): the 4 x 4 coarse neighbourhood stays in
        // registers for those fine rows (ps < s only to spread small grids over more blocks)
        const int nrun = s / ps;
        MGSR_ROWS(item, nc * nrun) {
            const int bi = item / nrun, p0 = (item - bi * nrun) * ps;
            double cc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const double *cr = c + int64_t(wrap(bi + a - 1, nc)) * nc;
#pragma unroll
                for (int b = 0; b < 4; ++b) cc[a][b] = __ldg(cr + cj[b]);
            }
#pragma unroll 4
            for (int pi = p0; pi < p0 + ps; ++pi) {
                const int I = (bi << ssh) + pi;
                const int64_t t = int64_t(I) * n + J;
                double acc = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    double row = 0.0;
#pragma unroll
                    for (int a = 0; a < 4; ++a) row += wtab[pi][a] * cc[a][b];
                    acc += wj[b] * row;
                }
                const double val = base ? (__ldg(base + t) - bsh) + acc : acc;
                out[t] = val;
                v[0] += val;
            }
        }
    }
    if (do_mean) grid_reduce<1>(v, slot, mean_out, 1.0 / double(total));
}

// Ratio-2 specialisation: one thread per coarse cell (bi, bj) produces the 2x2
// fine block (2bi + {0,1}, 2bj + {0,1}).  With s = 2, t is 0 or 1/2 and the
// Keys weights are exact constants: t = 0 gives (0, 1, 0, 0), whose weighted
// sum in the order above is exactly the centre value, and t = 1/2 gives
// (-1/16, 9/16, 9/16, -1/16).  Same operation order per output as
// k_prolong_add, so results are bitwise identical; ~8x fewer fp64 ops.
__global__ void k_prolong2_add(const double *__restrict__ c, int nc, const double *base, const double *bshift,
                               double *out, RedSlot slot, double *mean_out, int do_mean) {
    const int n = 2 * nc;
    const double bsh = (base && bshift) ? *bshift : 0.0;
    const double w0 = -0.0625, w1 = 0.5625;
    double v[1] = {0.0};
    MGSR_ROWS(bi, nc) {
        int ri[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) ri[o] = wrap(bi + o - 1, nc);
        MGSR_COLS(bj, nc) {
            double R0[4], R1[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int cb = wrap(bj + b - 1, nc);
                const double c0 = c[int64_t(ri[0]) * nc + cb], c1 = c[int64_t(ri[1]) * nc + cb];
                const double c2 = c[int64_t(ri[2]) * nc + cb], c3 = c[int64_t(ri[3]) * nc + cb];
                R0[b] = c1;
                double row = 0.0;
                row += w0 * c0;
                row += w1 * c1;
                row += w1 * c2;
                row += w0 * c3;
                R1[b] = row;
            }
            double a01 = 0.0, a11 = 0.0;
            a01 += w0 * R0[0]; a01 += w1 * R0[1]; a01 += w1 * R0[2]; a01 += w0 * R0[3];
            a11 += w0 * R1[0]; a11 += w1 * R1[1]; a11 += w1 * R1[2]; a11 += w0 * R1[3];
            const int64_t t0 = int64_t(2 * bi) * n + 2 * bj, t1 = t0 + n;
            double2 y0 = make_double2(R0[1], a01), y1 = make_double2(R1[1], a11);
            if (base) {
                const double2 b0 = *reinterpret_cast<const double2 *>(base + t0);
                const double2 b1 = *reinterpret_cast<const double2 *>(base + t1);
                y0.x = (b0.x - bsh) + y0.x; y0.y = (b0.y - bsh) + y0.y;
                y1.x = (b1.x - bsh) + y1.x; y1.y = (b1.y - bsh) + y1.y;
            }
            *reinterpret_cast<double2 *>(out + t0) = y0;
            *reinterpret_cast<double2 *>(out + t1) = y1;
            v[0] += ((y0.x + y0.y) + (y1.x + y1.y));
        }
    }
    if (do_mean) grid_reduce<1>(v, slot, mean_out, 1.0 / (double(n) * double(n)));
}

// Row-marching form of k_prolong2_add (same per-output arithmetic, bitwise identical values):
// thread = coarse column bj (fine columns 2bj, 2bj+1), a block = 256 columns x a strip of
// coarse rows sized for one wave; the 4 x 4 coarse neighbourhood slides down one coarse row per
// step (4 new L1 loads instead of 16), the next row's loads are issued before the current
// 2 x 2 fine block is computed.
__global__ void __launch_bounds__(256, 4) k_prolong2_rows(const double *__restrict__ c, int nc,
                                                          const double *__restrict__ base, const double *bshift,
                                                          double *__restrict__ out, RedSlot slot, double *mean_out,
                                                          int do_mean, int rows) {
    const int n = 2 * nc;
    const double bsh = (base && bshift) ? *bshift : 0.0;
    const double w0 = -0.0625, w1 = 0.5625;
    double v[1] = {0.0};
    const int bj = blockIdx.x * blockDim.x + threadIdx.x;
    const int b0 = blockIdx.y * rows, b1 = min(b0 + rows, nc);
    if (bj < nc && b0 < b1) {
        int cb[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) cb[b] = wrap(bj + b - 1, nc);
        auto crow = [&](int r, double (&dst)[4]) {
            const double *cr = c + int64_t(wrap(r, nc)) * nc;
#pragma unroll
            for (int b = 0; b < 4; ++b) dst[b] = __ldg(cr + cb[b]);
        };
        double c0[4], c1[4], c2[4], c3[4];
        crow(b0 - 1, c0);
        crow(b0, c1);
        crow(b0 + 1, c2);
        crow(b0 + 2, c3);
#pragma unroll 1
        for (int bi = b0; bi < b1; ++bi) {
            double nx[4] = {0.0, 0.0, 0.0, 0.0};
            if (bi + 1 < b1) crow(bi + 3, nx);
            const int64_t t0 = int64_t(2 * bi) * n + 2 * bj, t1 = t0 + n;
            double2 b0v = make_double2(0.0, 0.0), b1v = make_double2(0.0, 0.0);
            if (base) {
                b0v = __ldg(reinterpret_cast<const double2 *>(base + t0));
                b1v = __ldg(reinterpret_cast<const double2 *>(base + t1));
            }
            double R0[4], R1[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                R0[b] = c1[b];
                double row = 0.0;
                row += w0 * c0[b];
                row += w1 * c1[b];
                row += w1 * c2[b];
                row += w0 * c3[b];
                R1[b] = row;
            }
            double a01 = 0.0, a11 = 0.0;
            a01 += w0 * R0[0]; a01 += w1 * R0[1]; a01 += w1 * R0[2]; a01 += w0 * R0[3];
            a11 += w0 * R1[0]; a11 += w1 * R1[1]; a11 += w1 * R1[2]; a11 += w0 * R1[3];
            double2 y0 = make_double2(R0[1], a01), y1 = make_double2(R1[1], a11);
            if (base) {
                y0.x = (b0v.x - bsh) + y0.x; y0.y = (b0v.y - bsh) + y0.y;
                y1.x = (b1v.x - bsh) + y1.x; y1.y = (b1v.y - bsh) + y1.y;
            }
            *reinterpret_cast<double2 *>(out + t0) = y0;
            *reinterpret_cast<double2 *>(out + t1) = y1;
            v[0] += ((y0.x + y0.y) + (y1.x + y1.y));
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                c0[b] = c1[b];
                c1[b] = c2[b];
                c2[b] = c3[b];
                c3[b] = nx[b];
            }
        }
    }
    if (do_mean) grid_reduce<1>(v, slot, mean_out, 1.0 / (double(n) * double(n)));
}

// out = (base - *bshift) + (up - *ushift), optional grid mean of out (SR correction add,
// solver.py:190 / 196 with srmodel.py:486's mean subtraction folded in).
__global__ void k_add2(const double *__restrict__ base, const double *bshift, const double *__restrict__ up,
                       const double *ushift, double *__restrict__ out, int64_t count, RedSlot slot,
                       double *mean_out, int do_mean) {
    const double bsh = bshift ? *bshift : 0.0, ush = ushift ? *ushift : 0.0;
    double v[1] = {0.0};
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count;
         t += int64_t(gridDim.x) * blockDim.x) {
        double val = base ? (base[t] - bsh) + (up[t] - ush) : (up[t] - ush);
        out[t] = val;
        v[0] += val;
    }
    if (do_mean) grid_reduce<1>(v, slot, mean_out, 1.0 / double(count));
}

// Solve-loop logging pass (solver.py:196-197, 311-313): new_p = out - mean(out)
// written into p (the old iterate, read first), and
//   stats[0] = sqrt(mean((new_p - old_p)^2))           diff_norm  (grid.py:74-78)
//   stats[1] = sqrt(mean(r^2) - mean(r)^2), r = f - L new_p   residual(...).rms()
// L is evaluated on `out`; a constant shift leaves it unchanged up to rounding.
__global__ void k_finalize(const double *__restrict__ out, const double *mean_ptr, double *__restrict__ p,
                           FSrc fs, int n, double inv_h2, RedSlot slot, double *acc_out) {
    const int64_t total = int64_t(n) * n;
    const double m = *mean_ptr;
    const double sh = fs.load_shift();
    double v[3] = {0.0, 0.0, 0.0};
    MGSR_ROWS(i, n) {
        const int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        MGSR_COLS(j, n) {
            int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
            int64_t t = int64_t(i) * n + j;
            double o = out[t];
            double nb = ((out[int64_t(im1) * n + j] + out[int64_t(ip1) * n + j]) + out[t - j + jm1]) + out[t - j + jp1];
            double np_ = o - m;
            double d = np_ - p[t];
            double r = fs.at(t, sh) - ((nb - 4.0 * o) * inv_h2);
            // Tie the store to the load of p[t]: a store issued while the load of the same
            // address is in flight drops this pass from ~4.4 to ~1 TB/s (measured).
            asm volatile("" : "+d"(np_) : "d"(d));
            p[t] = np_;
            v[0] += d * d;
            v[1] += r;
            v[2] += r * r;
        }
    }
    grid_reduce<3>(v, slot, acc_out, 1.0 / double(total));
}

// Row-marching form of k_finalize (same per-cell arithmetic): thread = two adjacent columns, a
// block = 256 column pairs x a strip of rows (sized for one wave); the out rows above / at / below stay in registers
// (out is read once per cell), left / right neighbours come by shuffle (lanes 0 / 31 load theirs),
// the next row's loads are issued before the current row is computed.  The last block also
// writes stats (k_stats_sqrt folded in).  n % 64 == 0.
__global__ void __launch_bounds__(256, 4) k_finalize_rows(const double *__restrict__ out, const double *mean_ptr,
                                                       double *__restrict__ p, FSrc fs, int n, double inv_h2,
                                                       RedSlot slot, double *acc_out, double *stats, int rows) {
    const int lane = threadIdx.x & 31;
    const int pj = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = 2 * pj < n;   // whole warps (n / 2 is a multiple of 32)
    const int c0 = 2 * pj;
    const int cl = c0 == 0 ? n - 1 : c0 - 1, cr = c0 + 2 >= n ? c0 + 2 - n : c0 + 2;
    const int r0 = blockIdx.y * rows, r1 = min(r0 + rows, n);
    const double m = *mean_ptr;
    const double sh = fs.load_shift();
    const bool shifted = fs.shift != nullptr;
    double v[3] = {0.0, 0.0, 0.0};
    if (active) {
        auto row2 = [&](const double *a, int i) {
            return __ldg(reinterpret_cast<const double2 *>(a + int64_t(i) * n + c0));
        };
        double2 up = row2(out, r0 == 0 ? n - 1 : r0 - 1), cur = row2(out, r0);
        double2 dn = row2(out, r0 + 1 >= n ? r0 + 1 - n : r0 + 1);
        double2 pp = *reinterpret_cast<const double2 *>(p + int64_t(r0) * n + c0), ff = row2(fs.f, r0);
        double el = 0.0, er = 0.0;
        if (lane == 0) el = __ldg(out + int64_t(r0) * n + cl);
        if (lane == 31) er = __ldg(out + int64_t(r0) * n + cr);
#pragma unroll 1
        for (int i = r0; i < r1; ++i) {
            // next row's loads first
            const int i1 = i + 1 >= n ? i + 1 - n : i + 1, i2 = i + 2 >= n ? i + 2 - n : i + 2;
            const bool more = i + 1 < r1;
            double2 dn2 = dn, pp2 = pp, ff2 = ff;
            double el2 = 0.0, er2 = 0.0;
            if (more) {
                dn2 = row2(out, i2);
                pp2 = *reinterpret_cast<const double2 *>(p + int64_t(i1) * n + c0);
                ff2 = row2(fs.f, i1);
                if (lane == 0) el2 = __ldg(out + int64_t(i1) * n + cl);
                if (lane == 31) er2 = __ldg(out + int64_t(i1) * n + cr);
            }
            double left = __shfl_up_sync(0xffffffffu, cur.y, 1);
            double right = __shfl_down_sync(0xffffffffu, cur.x, 1);
            if (lane == 0) left = el;
            if (lane == 31) right = er;
            const double nb0 = ((up.x + dn.x) + left) + cur.y;
            const double nb1 = ((up.y + dn.y) + cur.x) + right;
            const double f0 = shifted ? (ff.x - sh) * fs.scale : ff.x;
            const double f1 = shifted ? (ff.y - sh) * fs.scale : ff.y;
            const double np0 = cur.x - m, np1 = cur.y - m;
            const double d0 = np0 - pp.x, d1 = np1 - pp.y;
            const double q0 = f0 - ((nb0 - 4.0 * cur.x) * inv_h2);
            const double q1 = f1 - ((nb1 - 4.0 * cur.y) * inv_h2);
            *reinterpret_cast<double2 *>(p + int64_t(i) * n + c0) = make_double2(np0, np1);
            v[0] += d0 * d0;
            v[0] += d1 * d1;
            v[1] += q0;
            v[1] += q1;
            v[2] += q0 * q0;
            v[2] += q1 * q1;
            up = cur;
            cur = dn;
            dn = dn2;
            pp = pp2;
            ff = ff2;
            el = el2;
            er = er2;
        }
    }
    double *const outs[3] = {acc_out, acc_out + 1, acc_out + 2};
    const double inv = 1.0 / (double(n) * double(n));
    const double scales[3] = {inv, inv, inv};
    if (grid_reduce_to<3>(v, slot, outs, scales)) {
        stats[0] = sqrt(acc_out[0]);
        const double var = acc_out[2] - acc_out[1] * acc_out[1];
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
    }
}


// Keys ratio-2 weights applied in k_prolong2_rows' order (vertical: rows a-1..a+2; horizontal: columns)
__device__ __forceinline__ double pf_vert(double c0, double c1, double c2, double c3) {
    const double w0 = -0.0625, w1 = 0.5625;
    double row = 0.0;
    row += w0 * c0;
    row += w1 * c1;
    row += w1 * c2;
    row += w0 * c3;
    return row;
}
__device__ __forceinline__ double pf_hint(double q0, double q1, double q2, double q3) {
    const double w0 = -0.0625, w1 = 0.5625;
    double a = 0.0;
    a += w0 * q0; a += w1 * q1; a += w1 * q2; a += w0 * q3;
    return a;
}

// The finest spline prolongation fused with the solve-loop logging pass (k_prolong2_rows + k_finalize_rows
// without the out field in HBM): out = (S - *bshift) + P(c) is evaluated row by row from S and the coarse
// correction c (Keys ratio 2, the k_prolong2_rows arithmetic), and immediately consumed by the logging
// pass: p <- out - m, diff and residual accumulators, stats.  m = *out_mean, the mean of out, is taken as
// the mean of c (the Keys weights of every coarse value sum to 4 fine cells, so mean(P(c)) = mean(c), and
// mean(S - *bshift) = 0): a grid-wide reduction of out before the pass is not needed.  34 B per fine cell
// (S, p, f read, p written, c read once per 4 cells) instead of 18 + 32.
// Thread = coarse column bj (fine columns 2 bj, 2 bj + 1), marching down a strip of fine rows; the own
// column's coarse rows a - 1 .. a + 2 stay in registers (one new coarse row per two fine rows), the
// neighbouring columns' values come by shuffle; lanes 0 / 31 also carry the two coarse columns beyond the
// warp and evaluate the out values left / right of the warp for the Laplacian.  nc % 32 == 0.
__global__ void __launch_bounds__(256, 2) k_prolong_finalize_rows(
    const double *__restrict__ S, const double *bshift, const double *__restrict__ c, int nc,
    const double *out_mean, double *__restrict__ p, FSrc fs, double inv_h2, RedSlot slot, double *acc_out,
    double *stats, int rows) {
    const int n = 2 * nc;
    const int lane = threadIdx.x & 31;
    const int bj = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = bj < nc;   // whole warps
    const int c0 = 2 * bj;
    const double bsh = *bshift, m = *out_mean;
    const double sh = fs.load_shift();
    const bool shifted = fs.shift != nullptr;
    const int r0 = blockIdx.y * rows, r1 = min(r0 + rows, n);
    double v[3] = {0.0, 0.0, 0.0};
    if (active && r0 < r1) {
        // extra coarse columns: lane 0 -> bj - 2, bj - 1; lane 31 -> bj + 1, bj + 2
        const int xa = lane == 0 ? wrap(bj - 2, nc) : wrap(bj + 1, nc), xb = lane == 0 ? wrap(bj - 1, nc) : wrap(bj + 2, nc);
        const bool edge = lane == 0 || lane == 31;
        // coarse rows a - 1 .. a + 2 of the own column (w*) and the extra columns (a*, b*)
        double w_0, w_1, w_2, w_3, a_0 = 0.0, a_1 = 0.0, a_2 = 0.0, a_3 = 0.0, b_0 = 0.0, b_1 = 0.0, b_2 = 0.0, b_3 = 0.0;
#define PF_LOAD(K, ROW)                                               \
    {                                                                 \
        const double *cr_ = c + int64_t(wrap((ROW), nc)) * nc;        \
        w_##K = __ldg(cr_ + bj);                                      \
        if (edge) {                                                   \
            a_##K = __ldg(cr_ + xa);                                  \
            b_##K = __ldg(cr_ + xb);                                  \
        }                                                             \
    }
        int i = r0 == 0 ? n - 1 : r0 - 1;
        int a = i >> 1;
        PF_LOAD(0, a - 1) PF_LOAD(1, a) PF_LOAD(2, a + 1) PF_LOAD(3, a + 2)
        // out row ii from the window and its S values (s2 = the own pair, sl / sr_ = the halo S of lanes 0 / 31):
        // the own pair (x = 2 bj, y = 2 bj + 1) and the values left of 2 bj / right of 2 bj + 1
        auto out_row = [&](bool odd, double2 s2, double sl, double sr_, double2 &o, double &hl, double &hr) {
            const double Ro = odd ? pf_vert(w_0, w_1, w_2, w_3) : w_1;
            double Ra = 0.0, Rb = 0.0;
            if (edge) {
                Ra = odd ? pf_vert(a_0, a_1, a_2, a_3) : a_1;
                Rb = odd ? pf_vert(b_0, b_1, b_2, b_3) : b_1;
            }
            const double up1 = __shfl_up_sync(0xffffffffu, Ro, 1);
            const double dn1 = __shfl_down_sync(0xffffffffu, Ro, 1);
            const double dn2 = __shfl_down_sync(0xffffffffu, Ro, 2);
            const double l31a = __shfl_sync(0xffffffffu, Ra, 31);   // lane 31's R at bj + 1 (= bj + 2 of lane 30)
            const double Rm1 = lane == 0 ? Rb : up1;                  // coarse column bj - 1
            const double Rp1 = lane == 31 ? Ra : dn1;                 // bj + 1
            const double Rp2 = lane == 31 ? Rb : (lane == 30 ? l31a : dn2);   // bj + 2
            o.x = (s2.x - bsh) + Ro;
            o.y = (s2.y - bsh) + pf_hint(Rm1, Ro, Rp1, Rp2);
            hl = __shfl_up_sync(0xffffffffu, o.y, 1);
            hr = __shfl_down_sync(0xffffffffu, o.x, 1);
            if (lane == 0) hl = (sl - bsh) + pf_hint(Ra, Rb, Ro, Rp1);
            if (lane == 31) hr = (sr_ - bsh) + Rp1;
        };
        const int cl = c0 == 0 ? n - 1 : c0 - 1, crr = c0 + 2 >= n ? c0 + 2 - n : c0 + 2;
        auto load_s = [&](int ii, double2 &s2, double &sl, double &sr_) {
            const double *srow = S + int64_t(ii) * n;
            s2 = __ldg(reinterpret_cast<const double2 *>(srow + c0));
            if (lane == 0) sl = __ldg(srow + cl);
            if (lane == 31) sr_ = __ldg(srow + crr);
        };
        double2 up, cur, dn, s2;
        double sl = 0.0, srr = 0.0, hl_c, hr_c, hl_d, hr_d, tl, tr;
        load_s(i, s2, sl, srr);
        out_row(i & 1, s2, sl, srr, up, tl, tr);
        // one fine row down: the window moves by one coarse row when the coarse row index changes
        {
            const int an = r0 >> 1;
            if (an != a) {
                a = an;
                w_0 = w_1; w_1 = w_2; w_2 = w_3;
                a_0 = a_1; a_1 = a_2; a_2 = a_3;
                b_0 = b_1; b_1 = b_2; b_2 = b_3;
                PF_LOAD(3, a + 2)
            }
        }
        i = r0;
        load_s(i, s2, sl, srr);
        out_row(i & 1, s2, sl, srr, cur, hl_c, hr_c);
        // prefetched operands of the next iteration: S of row i + 1, p / f of row i, the coarse row the window
        // needs at row i + 1
        int i1 = i + 1 >= n ? i + 1 - n : i + 1;
        double2 sN, pN, fN;
        double slN = 0.0, srN = 0.0, cwN = 0.0, caN = 0.0, cbN = 0.0;
        load_s(i1, sN, slN, srN);
        pN = *reinterpret_cast<const double2 *>(p + int64_t(i) * n + c0);
        fN = __ldg(reinterpret_cast<const double2 *>(fs.f + int64_t(i) * n + c0));
        bool shiftN = (i1 >> 1) != a;
        if (shiftN) {
            const double *cr_ = c + int64_t(wrap((i1 >> 1) + 2, nc)) * nc;
            cwN = __ldg(cr_ + bj);
            if (edge) { caN = __ldg(cr_ + xa); cbN = __ldg(cr_ + xb); }
        }
#pragma unroll 1
        for (; i < r1; ++i) {
            const double2 pp = pN, ff = fN, sc2 = sN;
            const double scl = slN, scr = srN;
            if (shiftN) {
                a = i1 >> 1;
                w_0 = w_1; w_1 = w_2; w_2 = w_3; w_3 = cwN;
                a_0 = a_1; a_1 = a_2; a_2 = a_3; a_3 = caN;
                b_0 = b_1; b_1 = b_2; b_2 = b_3; b_3 = cbN;
            }
            const bool odd1 = i1 & 1;
            // next iteration's loads first
            if (i + 1 < r1) {
                const int i2 = i1 + 1 >= n ? i1 + 1 - n : i1 + 1;
                load_s(i2, sN, slN, srN);
                pN = *reinterpret_cast<const double2 *>(p + int64_t(i1) * n + c0);
                fN = __ldg(reinterpret_cast<const double2 *>(fs.f + int64_t(i1) * n + c0));
                shiftN = (i2 >> 1) != a;
                if (shiftN) {
                    const double *cr_ = c + int64_t(wrap((i2 >> 1) + 2, nc)) * nc;
                    cwN = __ldg(cr_ + bj);
                    if (edge) { caN = __ldg(cr_ + xa); cbN = __ldg(cr_ + xb); }
                }
                i1 = i2;
            }
            out_row(odd1, sc2, scl, scr, dn, hl_d, hr_d);
            const double nb0 = ((up.x + dn.x) + hl_c) + cur.y;
            const double nb1 = ((up.y + dn.y) + cur.x) + hr_c;
            const double f0 = shifted ? (ff.x - sh) * fs.scale : ff.x;
            const double f1 = shifted ? (ff.y - sh) * fs.scale : ff.y;
            const double np0 = cur.x - m, np1 = cur.y - m;
            const double d0 = np0 - pp.x, d1 = np1 - pp.y;
            const double q0 = f0 - ((nb0 - 4.0 * cur.x) * inv_h2);
            const double q1 = f1 - ((nb1 - 4.0 * cur.y) * inv_h2);
            *reinterpret_cast<double2 *>(p + int64_t(i) * n + c0) = make_double2(np0, np1);
            v[0] += d0 * d0;
            v[0] += d1 * d1;
            v[1] += q0;
            v[1] += q1;
            v[2] += q0 * q0;
            v[2] += q1 * q1;
            up = cur;
            cur = dn;
            hl_c = hl_d;
            hr_c = hr_d;
        }
    }
#undef PF_LOAD
    double *const outs[3] = {acc_out, acc_out + 1, acc_out + 2};
    const double inv = 1.0 / (double(n) * double(n));
    const double scales[3] = {inv, inv, inv};
    if (grid_reduce_to<3>(v, slot, outs, scales)) {
        stats[0] = sqrt(acc_out[0]);
        const double var = acc_out[2] - acc_out[1] * acc_out[1];
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
    }
}

// k_prolong_finalize_rows restated two fine rows per iteration (same per-cell arithmetic and thread -> column
// mapping).  ncu showed the row-at-a-time form issue-bound, not bandwidth-bound: ~300 warp instructions per
// 64-cell warp row (parity selects, divergent edge-lane blocks with two extra coarse columns each, window
// slides behind branches, per-row index arithmetic) at 4 warps per scheduler.  Here an iteration handles the
// coarse row a of a strip that starts on an even fine row: the odd fine row 2a + 1 (vertical Keys weights over
// coarse rows a - 1 .. a + 2) and the even fine row 2a + 2 (coarse row a + 1 itself), so row parity is
// compile-time; every lane carries ONE extra coarse column (lane 0: bj0 - 1, lane 1: bj0 - 2, lane 31:
// bj0 + 32, lane 30: bj0 + 33; other lanes a dummy), so the columns beyond the warp cost one uniform
// vertical evaluation and an xor-1 shuffle instead of two divergent ones; the operands of the next
// iteration (two rows of S, p, f, one coarse row: ~100 B per thread) are requested before this one computes.
__device__ __forceinline__ void pf2_out_row(int lane, double Ro, double E, double2 s2, double sx, double bsh,
                                            double2 &o, double &hl, double &hr) {
    const double up1 = __shfl_up_sync(0xffffffffu, Ro, 1);
    const double dn1 = __shfl_down_sync(0xffffffffu, Ro, 1);
    const double dn2 = __shfl_down_sync(0xffffffffu, Ro, 2);
    const double xe = __shfl_xor_sync(0xffffffffu, E, 1);
    const double Rm1 = lane == 0 ? E : up1;       // coarse column bj - 1
    const double Rp1 = lane == 31 ? E : dn1;      // bj + 1
    const double Rp2 = lane >= 30 ? xe : dn2;     // bj + 2
    o.x = (s2.x - bsh) + Ro;
    o.y = (s2.y - bsh) + pf_hint(Rm1, Ro, Rp1, Rp2);
    // the out values left of the warp (odd fine column of bj0 - 1) / right of it (even fine column of bj0 + 32)
    const double t = pf_hint(xe, E, Ro, Rp1);
    const double X = (sx - bsh) + (lane == 0 ? t : Rp1);
    const double l = __shfl_up_sync(0xffffffffu, o.y, 1);
    const double r = __shfl_down_sync(0xffffffffu, o.x, 1);
    hl = lane == 0 ? X : l;
    hr = lane == 31 ? X : r;
}

__device__ __forceinline__ void pf2_finalize(double2 up, double2 cur, double2 dn, double hl, double hr, double2 pp,
                                             double2 ff, double m, double inv_h2, double *__restrict__ prow,
                                             double (&v)[3]) {
    const double nb0 = ((up.x + dn.x) + hl) + cur.y;
    const double nb1 = ((up.y + dn.y) + cur.x) + hr;
    const double np0 = cur.x - m, np1 = cur.y - m;
    const double d0 = np0 - pp.x, d1 = np1 - pp.y;
    const double q0 = ff.x - ((nb0 - 4.0 * cur.x) * inv_h2);
    const double q1 = ff.y - ((nb1 - 4.0 * cur.y) * inv_h2);
    *reinterpret_cast<double2 *>(prow) = make_double2(np0, np1);
    v[0] += d0 * d0;
    v[0] += d1 * d1;
    v[1] += q0;
    v[1] += q1;
    v[2] += q0 * q0;
    v[2] += q1 * q1;
}

// rows even (strips start on even fine rows), nc % 256 == 0, f unshifted
__global__ void __launch_bounds__(256, 2) k_prolong_finalize_pairs(
    const double *__restrict__ S, const double *bshift, const double *__restrict__ c, int nc,
    const double *out_mean, double *__restrict__ p, const double *__restrict__ f, double inv_h2, RedSlot slot,
    double *acc_out, double *stats, int rows) {
    const int n = 2 * nc;
    const int lane = threadIdx.x & 31;
    const int bj = blockIdx.x * blockDim.x + threadIdx.x;
    const int c0 = 2 * bj;
    const double bsh = *bshift, m = *out_mean;
    const int r0 = blockIdx.y * rows, r1 = min(r0 + rows, n);
    double v[3] = {0.0, 0.0, 0.0};
    if (r0 < r1) {
        const bool edge = lane <= 1 || lane >= 30;
        const bool sedge = lane == 0 || lane == 31;
        const int xcol = wrap(bj + (lane == 0 ? -1 : (lane == 1 ? -3 : (lane == 30 ? 3 : 1))), nc);
        const int scol = lane == 0 ? (c0 == 0 ? n - 1 : c0 - 1) : (c0 + 2 >= n ? c0 + 2 - n : c0 + 2);
        const int a0 = r0 >> 1, a1 = r1 >> 1;   // coarse rows of the strip: a0 .. a1 - 1
        auto ld_c = [&](int row, double &w, double &e) {
            const double *cr = c + int64_t(wrap(row, nc)) * nc;
            w = __ldg(cr + bj);
            e = 0.0;
            if (edge) e = __ldg(cr + xcol);
        };
        auto ld_s = [&](int row, double2 &s2, double &sx) {   // row already in [0, n)
            const double *sr = S + int64_t(row) * n;
            s2 = __ldg(reinterpret_cast<const double2 *>(sr + c0));
            sx = 0.0;
            if (sedge) sx = __ldg(sr + scol);
        };
        double w0, w1, w2, w3, e0, e1, e2, e3;
        double2 up, cur, dn, dn2;
        double hl_c, hr_c, hl_d, hr_d, hl_e, hr_e;
        {
            // out rows r0 - 1 (odd row of coarse row a0 - 1: window a0 - 2 .. a0 + 1) and r0 (coarse row a0)
            double wm, em, sx;
            double2 s2;
            ld_c(a0 - 2, wm, em);
            ld_c(a0 - 1, w0, e0);
            ld_c(a0, w1, e1);
            ld_c(a0 + 1, w2, e2);
            ld_c(a0 + 2, w3, e3);
            ld_s(r0 == 0 ? n - 1 : r0 - 1, s2, sx);
            pf2_out_row(lane, pf_vert(wm, w0, w1, w2), pf_vert(em, e0, e1, e2), s2, sx, bsh, up, hl_c, hr_c);
            ld_s(r0, s2, sx);
            pf2_out_row(lane, w1, e1, s2, sx, bsh, cur, hl_c, hr_c);
        }
        // operands of iteration a: S rows 2a + 1, 2a + 2 (the last one of the grid wraps to row 0), p and f rows
        // 2a, 2a + 1, coarse row a + 3
        double2 nS1, nS2, nP0, nP1, nF0, nF1;
        double nX1, nX2, nCw, nCe;
        auto prefetch = [&](int a) {
            const int i = 2 * a;
            ld_s(i + 1, nS1, nX1);
            ld_s(i + 2 >= n ? 0 : i + 2, nS2, nX2);
            const int64_t o = int64_t(i) * n + c0;
            nP0 = *reinterpret_cast<const double2 *>(p + o);
            nP1 = *reinterpret_cast<const double2 *>(p + o + n);
            nF0 = __ldg(reinterpret_cast<const double2 *>(f + o));
            nF1 = __ldg(reinterpret_cast<const double2 *>(f + o + n));
            ld_c(a + 3, nCw, nCe);
        };
        prefetch(a0);
#pragma unroll 1
        for (int a = a0; a < a1; ++a) {
            const double2 s1 = nS1, s2 = nS2, p0 = nP0, p1 = nP1, f0 = nF0, f1 = nF1;
            const double x1 = nX1, x2 = nX2, cw = nCw, ce = nCe;
            if (a + 1 < a1) prefetch(a + 1);
            double *const prow = p + int64_t(2 * a) * n + c0;
            pf2_out_row(lane, pf_vert(w0, w1, w2, w3), pf_vert(e0, e1, e2, e3), s1, x1, bsh, dn, hl_d, hr_d);
            pf2_finalize(up, cur, dn, hl_c, hr_c, p0, f0, m, inv_h2, prow, v);
            pf2_out_row(lane, w2, e2, s2, x2, bsh, dn2, hl_e, hr_e);
            pf2_finalize(cur, dn, dn2, hl_d, hr_d, p1, f1, m, inv_h2, prow + n, v);
            up = dn;
            cur = dn2;
            hl_c = hl_e;
            hr_c = hr_e;
            w0 = w1; w1 = w2; w2 = w3; w3 = cw;
            e0 = e1; e1 = e2; e2 = e3; e3 = ce;
        }
    }
    double *const outs[3] = {acc_out, acc_out + 1, acc_out + 2};
    const double inv = 1.0 / (double(n) * double(n));
    const double scales[3] = {inv, inv, inv};
    if (grid_reduce_to<3>(v, slot, outs, scales)) {
        stats[0] = sqrt(acc_out[0]);
        const double var = acc_out[2] - acc_out[1] * acc_out[1];
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
    }
}

// k_prolong_finalize_rows with its operands staged by the bulk-copy engine (same per-cell arithmetic, same
// launch geometry, so bitwise identical results).  The register-prefetch form keeps one fine row of S, p, f
// and one coarse row in flight per thread: ~28 KB per SM against the ~35 KB the HBM latency-bandwidth
// product asks for, so it ran latency-bound at ~4.6 TB/s.  Here a CTA (512 fine columns of a row strip)
// streams its rows through a ring of kPfNst shared-memory stages; stage k holds fine row g = r0 - 1 + k:
// S over columns c_blk - 2 .. c_blk + 513 (the halo the edge lanes read), p and f over the CTA's 512
// columns (rows r0 .. r1 - 1 only), and, when g is even, the coarse row (g >> 1) + 2 that slides into the
// Keys window, over coarse columns bj_blk - 2 .. bj_blk + 257.  Thread 0 issues the copies (1-D
// cp.async.bulk, one or two pieces per periodic segment) on a full mbarrier per stage; each warp releases a
// stage on its empty mbarrier once it read it, and thread 0 refills the slot two iterations later, so
// ~4 rows (~100 KB per SM at 2 CTAs) are in flight.
constexpr int kPfCols = 512;                                 // fine columns per CTA (256 threads x 2)
constexpr int kPfSegS = kPfCols + 4;                         // S: c_blk - 2 .. c_blk + 513
constexpr int kPfSegC = kPfCols / 2 + 4;                     // coarse: bj_blk - 2 .. bj_blk + 257
constexpr int kPfOffP = kPfSegS, kPfOffF = kPfOffP + kPfCols, kPfOffC = kPfOffF + kPfCols;
constexpr int kPfStage = kPfOffC + kPfSegC;                  // 1800 doubles = 14400 B (16-B multiple)
constexpr int kPfNst = 7;
constexpr size_t kPfSmem = size_t(kPfStage) * kPfNst * 8 + 2 * kPfNst * 8;

// [x0, x0 + len) of a periodic row of length n (len < n) -> shared memory, in one or two 16-B aligned pieces
__device__ __forceinline__ void pf_seg(uint32_t dst, const double *row, int x0, int len, int n, uint32_t bar) {
    if (x0 < 0) {
        rb_bulk(dst, row + x0 + n, uint32_t(-x0 * 8), bar);
        rb_bulk(dst + uint32_t(-x0 * 8), row, uint32_t((len + x0) * 8), bar);
    } else if (x0 + len > n) {
        rb_bulk(dst, row + x0, uint32_t((n - x0) * 8), bar);
        rb_bulk(dst + uint32_t((n - x0) * 8), row, uint32_t((len - (n - x0)) * 8), bar);
    } else {
        rb_bulk(dst, row + x0, uint32_t(len * 8), bar);
    }
}

__global__ void __launch_bounds__(256, 2) k_prolong_finalize_tma(
    const double *__restrict__ S, const double *bshift, const double *__restrict__ c, int nc,
    const double *out_mean, double *__restrict__ p, FSrc fs, double inv_h2, RedSlot slot, double *acc_out,
    double *stats, int rows) {
    extern __shared__ __align__(128) double pf_sm[];
    uint64_t *const bars = reinterpret_cast<uint64_t *>(pf_sm + size_t(kPfStage) * kPfNst);   // full[kPfNst], empty[kPfNst]
    const uint32_t sm0 = uint32_t(__cvta_generic_to_shared(pf_sm));
    const uint32_t full0 = uint32_t(__cvta_generic_to_shared(bars)), empty0 = full0 + 8 * kPfNst;
    const int n = 2 * nc;
    const int tid = threadIdx.x, lane = tid & 31;
    const int bj = blockIdx.x * blockDim.x + tid;
    const int c_blk = blockIdx.x * kPfCols, bj_blk = blockIdx.x * (kPfCols / 2);
    const double bsh = *bshift, m = *out_mean;
    const double sh = fs.load_shift();
    const bool shifted = fs.shift != nullptr;
    const int r0 = blockIdx.y * rows, r1 = min(r0 + rows, n);
    const int R = r1 - r0;   // >= 1 by the launch geometry
    const int nstages = R + 2;
    auto grow = [&](int k) { return wrap(r0 - 1 + k, n); };
    auto issue = [&](int k) {   // thread 0: stage k -> slot k % kPfNst
        const int g = grow(k);
        const bool pf = k >= 1 && k <= R, cr = k >= 1 && !(g & 1);
        const uint32_t bytes = uint32_t(kPfSegS * 8) + (pf ? uint32_t(2 * kPfCols * 8) : 0u) +
                               (cr ? uint32_t(kPfSegC * 8) : 0u);
        const uint32_t bar = full0 + 8u * uint32_t(k % kPfNst);
        const uint32_t dst = sm0 + uint32_t((k % kPfNst) * kPfStage * 8);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        const int64_t ro = int64_t(g) * n;
        pf_seg(dst, S + ro, c_blk - 2, kPfSegS, n, bar);
        if (pf) {
            rb_bulk(dst + kPfOffP * 8, p + ro + c_blk, kPfCols * 8, bar);
            rb_bulk(dst + kPfOffF * 8, fs.f + ro + c_blk, kPfCols * 8, bar);
        }
        if (cr) pf_seg(dst + kPfOffC * 8, c + int64_t(wrap((g >> 1) + 2, nc)) * nc, bj_blk - 2, kPfSegC, nc, bar);
    };
    if (tid == 0) {
        for (int s = 0; s < kPfNst; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8u * s) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty0 + 8u * s), "r"(blockDim.x / 32) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < kPfNst && k < nstages; ++k) issue(k);
    auto wait_full = [&](int k) { rb_mbar_wait(full0 + 8u * uint32_t(k % kPfNst), uint32_t((k / kPfNst) & 1)); };
    auto release = [&](int k) {
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8u * uint32_t(k % kPfNst)) : "memory");
    };
    auto stage = [&](int k) { return pf_sm + (k % kPfNst) * kPfStage; };
    double v[3] = {0.0, 0.0, 0.0};
    const int t2 = 2 * tid;   // the thread's fine pair in the CTA's columns; coarse column tid
    const bool edge = lane == 0 || lane == 31;
    // extra coarse columns: lane 0 -> bj - 2, bj - 1; lane 31 -> bj + 1, bj + 2 (segment offsets)
    const int oxa = lane == 0 ? tid : tid + 3, oxb = lane == 0 ? tid + 1 : tid + 4;
    double w_0, w_1, w_2, w_3, a_0 = 0.0, a_1 = 0.0, a_2 = 0.0, a_3 = 0.0, b_0 = 0.0, b_1 = 0.0, b_2 = 0.0, b_3 = 0.0;
    {
        const int xa = lane == 0 ? wrap(bj - 2, nc) : wrap(bj + 1, nc), xb = lane == 0 ? wrap(bj - 1, nc) : wrap(bj + 2, nc);
        const int a = grow(0) >> 1;
#define PF_GLOAD(K, ROW)                                              \
    {                                                                 \
        const double *cr_ = c + int64_t(wrap((ROW), nc)) * nc;        \
        w_##K = __ldg(cr_ + bj);                                      \
        if (edge) {                                                   \
            a_##K = __ldg(cr_ + xa);                                  \
            b_##K = __ldg(cr_ + xb);                                  \
        }                                                             \
    }
        PF_GLOAD(0, a - 1) PF_GLOAD(1, a) PF_GLOAD(2, a + 1) PF_GLOAD(3, a + 2)
#undef PF_GLOAD
    }
    // the window slides one coarse row when stage k's fine row is even (its coarse row is in the stage)
    auto slide = [&](int k) {
        if (grow(k) & 1) return;
        const double *cs = stage(k) + kPfOffC;
        w_0 = w_1; w_1 = w_2; w_2 = w_3; w_3 = cs[tid + 2];
        a_0 = a_1; a_1 = a_2; a_2 = a_3;
        b_0 = b_1; b_1 = b_2; b_2 = b_3;
        if (edge) { a_3 = cs[oxa]; b_3 = cs[oxb]; }
    };
    auto out_row = [&](int k, double2 &o, double &hl, double &hr) {
        const double *ss = stage(k);
        const bool odd = grow(k) & 1;
        const double2 s2 = *reinterpret_cast<const double2 *>(ss + 2 + t2);
        const double Ro = odd ? pf_vert(w_0, w_1, w_2, w_3) : w_1;
        double Ra = 0.0, Rb = 0.0;
        if (edge) {
            Ra = odd ? pf_vert(a_0, a_1, a_2, a_3) : a_1;
            Rb = odd ? pf_vert(b_0, b_1, b_2, b_3) : b_1;
        }
        const double up1 = __shfl_up_sync(0xffffffffu, Ro, 1);
        const double dn1 = __shfl_down_sync(0xffffffffu, Ro, 1);
        const double dn2 = __shfl_down_sync(0xffffffffu, Ro, 2);
        const double l31a = __shfl_sync(0xffffffffu, Ra, 31);
        const double Rm1 = lane == 0 ? Rb : up1;
        const double Rp1 = lane == 31 ? Ra : dn1;
        const double Rp2 = lane == 31 ? Rb : (lane == 30 ? l31a : dn2);
        o.x = (s2.x - bsh) + Ro;
        o.y = (s2.y - bsh) + pf_hint(Rm1, Ro, Rp1, Rp2);
        hl = __shfl_up_sync(0xffffffffu, o.y, 1);
        hr = __shfl_down_sync(0xffffffffu, o.x, 1);
        if (lane == 0) hl = (ss[1 + t2] - bsh) + pf_hint(Ra, Rb, Ro, Rp1);
        if (lane == 31) hr = (ss[4 + t2] - bsh) + Rp1;
    };
    double2 up, cur, dn;
    double hl_c, hr_c, hl_d, hr_d, tl, tr;
    wait_full(0);
    out_row(0, up, tl, tr);
    release(0);
    wait_full(1);
    slide(1);
    out_row(1, cur, hl_c, hr_c);
#pragma unroll 1
    for (int k = 1; k <= R; ++k) {
        if (tid == 0 && k >= 2 && k - 2 + kPfNst < nstages) {
            const int kr = k - 2;   // released by every warp at the end of iteration k - 2 (stage 0: before the loop)
            rb_mbar_wait(empty0 + 8u * uint32_t(kr % kPfNst), uint32_t((kr / kPfNst) & 1));
            issue(kr + kPfNst);
        }
        wait_full(k + 1);
        slide(k + 1);
        out_row(k + 1, dn, hl_d, hr_d);
        const double *st = stage(k);
        const double2 pp = *reinterpret_cast<const double2 *>(st + kPfOffP + t2);
        const double2 ff = *reinterpret_cast<const double2 *>(st + kPfOffF + t2);
        release(k);
        const double nb0 = ((up.x + dn.x) + hl_c) + cur.y;
        const double nb1 = ((up.y + dn.y) + cur.x) + hr_c;
        const double f0 = shifted ? (ff.x - sh) * fs.scale : ff.x;
        const double f1 = shifted ? (ff.y - sh) * fs.scale : ff.y;
        const double np0 = cur.x - m, np1 = cur.y - m;
        const double d0 = np0 - pp.x, d1 = np1 - pp.y;
        const double q0 = f0 - ((nb0 - 4.0 * cur.x) * inv_h2);
        const double q1 = f1 - ((nb1 - 4.0 * cur.y) * inv_h2);
        *reinterpret_cast<double2 *>(p + int64_t(grow(k)) * n + c_blk + t2) = make_double2(np0, np1);
        v[0] += d0 * d0;
        v[0] += d1 * d1;
        v[1] += q0;
        v[1] += q1;
        v[2] += q0 * q0;
        v[2] += q1 * q1;
        up = cur;
        cur = dn;
        hl_c = hl_d;
        hr_c = hr_d;
    }
    double *const outs[3] = {acc_out, acc_out + 1, acc_out + 2};
    const double inv = 1.0 / (double(n) * double(n));
    const double scales[3] = {inv, inv, inv};
    if (grid_reduce_to<3>(v, slot, outs, scales)) {
        stats[0] = sqrt(acc_out[0]);
        const double var = acc_out[2] - acc_out[1] * acc_out[1];
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
    }
}

__global__ void k_stats_sqrt(const double *acc, double *stats) {
    stats[0] = sqrt(acc[0]);
    double var = acc[2] - acc[1] * acc[1];
    stats[1] = sqrt(var > 0.0 ? var : 0.0);
}

// rms of a - b (b may be null)
__global__ void k_sqdiff(const double *__restrict__ a, const double *__restrict__ b, int64_t count, RedSlot slot,
                         double *out) {
    double v[1] = {0.0};
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count;
         t += int64_t(gridDim.x) * blockDim.x) {
        double d = b ? a[t] - b[t] : a[t];
        v[0] += d * d;
    }
    grid_reduce<1>(v, slot, out, 1.0 / double(count));
}

// ---------------------------------------------------------------------------
// launch helpers (shared with plan.cu)

// Stream-ordered scratch for the API entry points: a memory pool private to this library (one per
// device), created on first use with an unbounded release threshold, so freed blocks stay mapped for the
// next call (with threshold 0 every 4096^2 mgsr_gs_sweeps remapped 268 MB) without changing the
// process-wide default pool that torch or other libraries may use.
int scratch_alloc(void **ptr, size_t bytes, cudaStream_t st) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    MGSR_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) { set_error("device ordinal out of range"); return MGSR_E_BAD_ARG; }
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            MGSR_CUDA_TRY(cudaMemPoolCreate(&pools[dev], &props));
            uint64_t thr = UINT64_MAX;
            MGSR_CUDA_TRY(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
        }
        pool = pools[dev];
    }
    MGSR_CUDA_TRY(cudaMallocFromPoolAsync(ptr, bytes, pool, st));
    return MGSR_OK;
}

int num_sms() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

dim3 grid_2d(int rows, int cols) {
    int gx = (cols + 255) / 256;
    if (gx > 32) gx = 32;
    int gy = (148 * 8) / gx;
    if (gy > rows) gy = rows;
    if (gy < 1) gy = 1;
    return dim3(gx, gy);
}

int grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    int64_t cap = 148 * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return int(b);
}

// 2-D tensor map over an n x n fp64 row-major grid, 64 x 64 boxes, no swizzle (k_gs_rb windows)
static int make_tmap_2d(CUtensorMap *tm, const double *base, int n) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return 1;
        }
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(n)};
    const cuuint64_t strides[1] = {cuuint64_t(n) * sizeof(double)};
    const cuuint32_t box[2] = {cuuint32_t(kRbW), cuuint32_t(kRbW)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
        return 1;
    }
    return 0;
}

int launch_gs(const double *p_in, double *p_out, double *tmp, FSrc fs, int n, double h2, int sweeps,
              int zero_init, double *rc, double *rc_mean, double *mean_out, void *red_ws, cudaStream_t st) {
    // red_ws: >= 3 reduction slots.  p_in is never written (unless p_in == p_out).
    RedSlot s0 = red_slot_at(red_ws);
    RedSlot s1 = red_slot_at(static_cast<char *>(red_ws) + kRedSlotBytes);
    RedSlot s2 = red_slot_at(static_cast<char *>(red_ws) + 2 * kRedSlotBytes);
    const double inv_h2 = 1.0 / h2;
    const size_t bytes = sizeof(double) * size_t(n) * n;
    if (n <= kSmallN) {
        if (p_out != p_in && !zero_init)
            MGSR_CUDA_TRY(cudaMemcpyAsync(p_out, p_in, bytes, cudaMemcpyDeviceToDevice, st));
        size_t smem = 2 * sizeof(double) * n * n;
        cudaFuncSetAttribute(k_gs_small, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        k_gs_small<<<1, kSmallThreads, smem, st>>>(p_out, fs, n, h2, sweeps, zero_init, mean_out);
        MGSR_LAUNCH_CHECK();
        if (rc) {
            k_res_restrict<<<grid_2d(n / 2, n / 2), 256, 0, st>>>(p_out, fs, n, 2, inv_h2, rc,
                                                                                       s1, rc_mean);
            MGSR_LAUNCH_CHECK();
        }
        return MGSR_OK;
    }
    if (n >= kRbMinN && sweeps >= 1 && p_in != p_out) {
        const int chunks = (sweeps + kRbMaxK - 1) / kRbMaxK;
        if (chunks > 1 && !tmp) { set_error("gs: chunked sweeps need a scratch buffer"); return MGSR_E_BAD_ARG; }
        int done = 0;
        const double *src = p_in;
        for (int ci = 0; ci < chunks; ++ci) {
            int k = sweeps - done;
            if (k > kRbMaxK) k = kRbMaxK;
            const bool last = ci == chunks - 1;
            const bool rcl = last && rc;
            double *dst = ((chunks - 1 - ci) % 2 == 0) ? p_out : tmp;
            const int zi = (ci == 0) ? zero_init : 0;
            double *mo = last ? mean_out : nullptr;
#define MGSR_RB_LAUNCH(KK, RCV, RCP, RCM)                                                                  \
    {                                                                                                      \
        auto kern = k_gs_rb<KK, RCV>;                                                                      \
        constexpr int HE = (2 * KK + (RCV ? 1 : 0) + 1) & ~1, TX = kRbW - 2 * HE;                          \
        const int tl = ((n + TX - 1) / TX) * ((n + TX - 1) / TX);                                          \
        const size_t rsm = sizeof(double) * (2 * kRbW * kRbW + 2 * kRbWarps * 64);                         \
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rsm));                 \
        int occ = 0;                                                                                       \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kRbThreads, rsm);                        \
        int blocks = num_sms() * (occ > 0 ? occ : 1);                                                      \
        if (blocks > tl) blocks = tl;                                                                      \
        CUtensorMap tmp_, tmf_;                                                                            \
        if (make_tmap_2d(&tmp_, src ? src : fs.f, n) || make_tmap_2d(&tmf_, fs.f, n)) return MGSR_E_CUDA; \
        kern<<<blocks, kRbThreads, rsm, st>>>(tmp_, tmf_, src, dst, fs, n, h2, zi, inv_h2, RCP, s0, mo, RCM); \
    }
#define MGSR_RB_CASE(KK)                                                                                   \
    case KK:                                                                                               \
        if (rcl) MGSR_RB_LAUNCH(KK, true, rc, rc_mean)                                                     \
        else MGSR_RB_LAUNCH(KK, false, nullptr, nullptr)                                                   \
        break;
            switch (k) {
                MGSR_RB_CASE(1)
                MGSR_RB_CASE(2)
                MGSR_RB_CASE(3)
                MGSR_RB_CASE(4)
            }
#undef MGSR_RB_CASE
#undef MGSR_RB_LAUNCH
            MGSR_LAUNCH_CHECK();
            done += k;
            src = dst;
        }
        return MGSR_OK;
    }
    // generic: half-sweeps in place on p_out
    if (p_out != p_in && !zero_init)
        MGSR_CUDA_TRY(cudaMemcpyAsync(p_out, p_in, bytes, cudaMemcpyDeviceToDevice, st));
    if (zero_init) MGSR_CUDA_TRY(cudaMemsetAsync(p_out, 0, bytes, st));
    dim3 g = grid_2d(n, n / 2);
    for (int s = 0; s < sweeps; ++s)
        for (int color = 0; color < 2; ++color) {
            k_gs_half<<<g, 256, 0, st>>>(p_out, fs, n, h2, color);
            MGSR_LAUNCH_CHECK();
        }
    if (mean_out) {
        k_mean<<<grid_for(int64_t(n) * n, 256), 256, 0, st>>>(p_out, int64_t(n) * n, s0, mean_out);
        MGSR_LAUNCH_CHECK();
    }
    if (rc) {
        k_res_restrict<<<grid_2d(n / 2, n / 2), 256, 0, st>>>(p_out, fs, n, 2, inv_h2, rc, s1,
                                                                                   rc_mean);
        MGSR_LAUNCH_CHECK();
    }
    return MGSR_OK;
}

int launch_prolong_add(const double *c, int nc, int s, const double *base, const double *bshift, double *out,
                       double *mean_out, void *red_slot, cudaStream_t st) {
    RedSlot sl = red_slot_at(red_slot);
    if (s == 2 && nc >= 512) {
        const int gx = (nc + 255) / 256;
        int strips = (4 * num_sms()) / gx;
        strips = strips < 1 ? 1 : (strips > nc ? nc : strips);
        const int rows = (nc + strips - 1) / strips;
        const dim3 g(gx, (nc + rows - 1) / rows);
        k_prolong2_rows<<<g, 256, 0, st>>>(c, nc, base, bshift, out, sl, mean_out, mean_out != nullptr, rows);
        MGSR_LAUNCH_CHECK();
        return MGSR_OK;
    }
    if (s == 2) {
        k_prolong2_add<<<grid_2d(nc, nc), 256, 0, st>>>(c, nc, base, bshift, out, sl, mean_out, mean_out != nullptr);
        MGSR_LAUNCH_CHECK();
        return MGSR_OK;
    }
    if (s <= 16 && (s & (s - 1)) == 0 && nc * s <= 8192) {
        // enough row items for ~8 blocks per SM: split each coarse row's s fine rows into runs
        const int cols = (nc * s + 255) / 256;
        int ps = s;
        while (ps > 1 && int64_t(nc) * (s / ps) * cols < 148 * 8) ps >>= 1;
        k_prolong_add_pow2<<<grid_2d(nc * (s / ps), nc * s), 256, 0, st>>>(c, nc, s, __builtin_ctz(s), ps, base,
                                                                           bshift, out, sl, mean_out,
                                                                           mean_out != nullptr);
        MGSR_LAUNCH_CHECK();
        return MGSR_OK;
    }
    k_prolong_add<<<grid_2d(nc * s, nc * s), 256, 0, st>>>(c, nc, s, base, bshift, out, sl, mean_out,
                                                          mean_out != nullptr);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_add2(const double *base, const double *bshift, const double *up, const double *ushift, double *out,
                int64_t count, double *mean_out, void *red_slot, cudaStream_t st) {
    RedSlot sl = red_slot_at(red_slot);
    k_add2<<<grid_for(count, 256), 256, 0, st>>>(base, bshift, up, ushift, out, count, sl, mean_out,
                                                  mean_out != nullptr);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_res_restrict(const double *p, FSrc fs, int n, int s, double *rc, double *rc_mean, void *red_slot,
                        cudaStream_t st) {
    int nc = n / s;
    RedSlot sl = red_slot_at(red_slot);
    k_res_restrict<<<grid_2d(nc, nc), 256, 0, st>>>(p, fs, n, s, 1.0 / ((2.0 * M_PI / n) * (2.0 * M_PI / n)),
                                                                       rc, sl, rc_mean);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

// the fused finest spline prolongation + logging pass (k_prolong_finalize_rows); false when it does not apply
bool prolong_finalize_applies(int n) { return n >= 1024 && (n / 2) % 256 == 0 && !std::getenv("MGSR_NO_FUSED_TOP"); }
int launch_prolong_finalize(const double *S, const double *bshift, const double *c, int nc, const double *out_mean,
                            double *p, FSrc fs, double *acc3, double *stats2, void *red_slot, cudaStream_t st) {
    RedSlot sl = red_slot_at(red_slot);
    const int n = 2 * nc;
    const double h = 2.0 * M_PI / n;
    const int gx = nc / 256;
    int strips = (2 * num_sms()) / gx;   // one wave at 2 CTAs per SM
    strips = strips < 1 ? 1 : (strips > n ? n : strips);
    const int rows = (((n + strips - 1) / strips) + 1) & ~1;   // even: the strips start on even fine rows
    const dim3 g(gx, (n + rows - 1) / rows);
    if (int64_t(g.x) * g.y > kRedMaxBlocks) { set_error("prolong_finalize grid too large"); return MGSR_E_UNSUPPORTED; }
    // A/B: MGSR_FUSED_TOP=rows (one fine row per iteration) | tma (the bulk-copy staged form); default: row pairs
    static const char *variant = std::getenv("MGSR_FUSED_TOP");
    static const bool tma = variant && !std::strcmp(variant, "tma"), by_rows = variant && !std::strcmp(variant, "rows");
    if (!tma && !by_rows && fs.shift == nullptr) {
        k_prolong_finalize_pairs<<<g, 256, 0, st>>>(S, bshift, c, nc, out_mean, p, fs.f, 1.0 / (h * h), sl, acc3,
                                                    stats2, rows);
        MGSR_LAUNCH_CHECK();
        return MGSR_OK;
    }
    if (!tma) {
        k_prolong_finalize_rows<<<g, 256, 0, st>>>(S, bshift, c, nc, out_mean, p, fs, 1.0 / (h * h), sl, acc3, stats2,
                                                   rows);
        MGSR_LAUNCH_CHECK();
        return MGSR_OK;
    }
    static bool attr = false;
    if (!attr) {
        MGSR_CUDA_TRY(cudaFuncSetAttribute(k_prolong_finalize_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           int(kPfSmem)));
        attr = true;
    }
    k_prolong_finalize_tma<<<g, 256, kPfSmem, st>>>(S, bshift, c, nc, out_mean, p, fs, 1.0 / (h * h), sl, acc3, stats2,
                                                    rows);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_finalize(const double *out, const double *mean_ptr, double *p, FSrc fs, int n, double *acc3,
                    double *stats2, void *red_slot, cudaStream_t st) {
    RedSlot sl = red_slot_at(red_slot);
    double h = 2.0 * M_PI / n;
    // one wave: 4 CTAs per SM (the kernel's occupancy), the row strips sized to fill it
    const int gx = (n / 2 + 255) / 256;
    int strips = (4 * num_sms()) / gx;
    strips = strips < 1 ? 1 : (strips > n ? n : strips);
    const int rows = (n + strips - 1) / strips;
    const dim3 g(gx, (n + rows - 1) / rows);
    if (n % 64 == 0 && int64_t(g.x) * g.y <= kRedMaxBlocks) {
        k_finalize_rows<<<g, 256, 0, st>>>(out, mean_ptr, p, fs, n, 1.0 / (h * h), sl, acc3, stats2, rows);
        MGSR_LAUNCH_CHECK();
        return MGSR_OK;
    }
    k_finalize<<<grid_2d(n, n), 256, 0, st>>>(out, mean_ptr, p, fs, n, 1.0 / (h * h), sl, acc3);
    MGSR_LAUNCH_CHECK();
    k_stats_sqrt<<<1, 1, 0, st>>>(acc3, stats2);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_correction_small(const double *rc0, const double *rc0_mean, double *d0, const int *sides, int nlev,
                            int n_smooth, int coarse_sweeps, cudaStream_t st) {
    if (nlev < 1 || nlev > kSmallMaxLev || sides[0] > kSmallN) {
        set_error("correction_small: bad ladder");
        return MGSR_E_BAD_ARG;
    }
    SmallLadder L{};
    L.nlev = nlev;
    size_t smem = 0;
    for (int j = 0; j < nlev; ++j) {
        L.side[j] = sides[j];
        if (j > 0 && sides[j] * 2 != sides[j - 1]) { set_error("correction_small: ratio-2 ladder only"); return MGSR_E_BAD_ARG; }
        smem += 2 * sizeof(double) * size_t(sides[j]) * sides[j];
    }
    cudaFuncSetAttribute(k_correction_small, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_correction_small<<<1, kSmallThreads, smem, st>>>(rc0, rc0_mean, d0, L, n_smooth, coarse_sweeps);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_vcycle_small(double *p, const double *f, const int *sides, int nlev, int n_smooth, int coarse_sweeps,
                        double *stats, cudaStream_t st) {
    if (nlev < 2 || nlev > kSmallMaxLev || sides[0] > kSmallN) { set_error("vcycle_small: bad ladder"); return MGSR_E_BAD_ARG; }
    SmallLadder L{};
    L.nlev = nlev;
    size_t smem = 3 * sizeof(double) * size_t(sides[0]) * sides[0];
    for (int j = 0; j < nlev; ++j) {
        L.side[j] = sides[j];
        if (j > 0 && sides[j] * 2 != sides[j - 1]) { set_error("vcycle_small: ratio-2 ladder only"); return MGSR_E_BAD_ARG; }
        if (j > 0) smem += 2 * sizeof(double) * size_t(sides[j]) * sides[j];
    }
    cudaFuncSetAttribute(k_vcycle_small, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_vcycle_small<<<1, kSmallThreads, smem, st>>>(p, f, L, n_smooth, coarse_sweeps, stats);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_affine(const double *a, double *out, int64_t count, const double *shift, double scale, cudaStream_t st) {
    k_affine<<<grid_for(count, 256), 256, 0, st>>>(a, out, count, shift, scale);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

}  // namespace mgsr

// ---------------------------------------------------------------------------
// C ABI (stencil part)

using namespace mgsr;

extern "C" const char *mgsr_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *mgsr_version(void) { return "mgsr_b200 1.0 (sm_100a)"; }

// layout: [scalars 256 B][slot0][slot1][slot2][slot3]
extern "C" size_t mgsr_workspace_bytes(int64_t n) {
    (void)n;
    return 256 + 4 * kRedSlotBytes;
}

// Validate a caller's workspace and reset its reduction-slot tickets (the grid reductions need them at
// zero and return them to zero; a recycled or fresh uninitialised buffer may hold anything).
static int check_ws(void *ws, size_t bytes, cudaStream_t st) {
    if (!ws || bytes < mgsr_workspace_bytes(0)) {
        set_error("workspace too small");
        return MGSR_E_WORKSPACE;
    }
    for (int k = 0; k < 3; ++k)
        MGSR_CUDA_TRY(cudaMemsetAsync(static_cast<char *>(ws) + 256 + k * kRedSlotBytes, 0, sizeof(unsigned), st));
    return MGSR_OK;
}

extern "C" int mgsr_gs_sweeps(double *p, const double *f, int64_t n, double h2, int32_t sweeps, void *ws,
                              size_t ws_bytes, void *stream) {
    if (n < 2 || !p || !f || sweeps < 0) { set_error("sweep count must be >= 0"); return MGSR_E_BAD_ARG; }
    if (n % 2) { set_error("red-black coloring needs an even side, got " + std::to_string(n)); return MGSR_E_ODD_SIDE; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int r = check_ws(ws, ws_bytes, st)) return r;
    if (sweeps == 0) return MGSR_OK;
    double *scal = static_cast<double *>(ws);
    void *red = static_cast<char *>(ws) + 256;
    FSrc fs{f, nullptr, 1.0};
    if (n <= kSmallN)  // exact per-sweep mean subtraction inside one CTA
        return launch_gs(p, p, nullptr, fs, int(n), h2, sweeps, 0, nullptr, nullptr, nullptr, red, st);
    double *tmp = nullptr;
    if (int e = scratch_alloc(reinterpret_cast<void **>(&tmp), 2 * sizeof(double) * n * n, st)) return e;
    int rc = launch_gs(p, tmp, tmp + n * n, fs, int(n), h2, sweeps, 0, nullptr, nullptr, scal, red, st);
    if (rc == MGSR_OK) rc = launch_affine(tmp, p, n * n, scal, 1.0, st);
    cudaFreeAsync(tmp, st);
    return rc;
}

extern "C" int mgsr_laplacian(const double *p, double *out, int64_t n, double inv_h2, void *stream) {
    if (n < 2 || !p || !out) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_laplacian<<<grid_2d(int(n), int(n)), 256, 0, st>>>(p, out, int(n), inv_h2);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

extern "C" int mgsr_residual(const double *p, const double *f, double *r, int64_t n, void *ws, size_t ws_bytes,
                             void *stream) {
    if (n < 2 || !p || !f || !r) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int e = check_ws(ws, ws_bytes, st)) return e;
    double *scal = static_cast<double *>(ws);
    RedSlot sl = red_slot_at(static_cast<char *>(ws) + 256);
    double h = 2.0 * M_PI / double(n);
    k_residual_raw<<<grid_2d(int(n), int(n)), 256, 0, st>>>(p, f, r, int(n), 1.0 / (h * h), sl, scal);
    MGSR_LAUNCH_CHECK();
    return launch_affine(r, r, n * n, scal, 1.0, st);
}

extern "C" int mgsr_restrict(const double *fine, double *coarse, int64_t n, int32_t s, int32_t subtract_mean,
                             void *ws, size_t ws_bytes, void *stream) {
    if (s < 2 || (s & (s - 1))) { set_error("transfer ratio must be a power of two >= 2, got " + std::to_string(s)); return MGSR_E_RATIO; }
    if (n < 1 || !fine || !coarse) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    if (n % s) { set_error("fine side " + std::to_string(n) + " is not divisible by ratio " + std::to_string(s)); return MGSR_E_NOT_DIVISIBLE; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int e = check_ws(ws, ws_bytes, st)) return e;
    double *scal = static_cast<double *>(ws);
    RedSlot sl = red_slot_at(static_cast<char *>(ws) + 256);
    int64_t nc = n / s;
    k_inject<<<grid_2d(int(nc), int(nc)), 256, 0, st>>>(fine, coarse, int(n), s, sl, scal);
    MGSR_LAUNCH_CHECK();
    if (subtract_mean) return launch_affine(coarse, coarse, nc * nc, scal, 1.0, st);
    return MGSR_OK;
}

extern "C" int mgsr_spline_prolong(const double *c, int64_t nc, int32_t s, double *out, void *stream) {
    if (s < 2 || (s & (s - 1))) { set_error("transfer ratio must be a power of two >= 2, got " + std::to_string(s)); return MGSR_E_RATIO; }
    if (s > 16) { set_error("prolongation ratio must be one of (2, 4, 8, 16), got " + std::to_string(s)); return MGSR_E_PROLONG_RATIO; }
    if (nc < 1 || !c || !out) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    return launch_prolong_add(c, int(nc), s, nullptr, nullptr, out, nullptr, nullptr, static_cast<cudaStream_t>(stream));
}

extern "C" int mgsr_rms_diff(const double *a, const double *b, int64_t count, double *out_host, void *ws,
                             size_t ws_bytes, void *stream) {
    if (count < 1 || !a || !out_host) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int e = check_ws(ws, ws_bytes, st)) return e;
    double *scal = static_cast<double *>(ws);
    RedSlot sl = red_slot_at(static_cast<char *>(ws) + 256);
    k_sqdiff<<<grid_for(count, 256), 256, 0, st>>>(a, b, count, sl, scal);
    MGSR_LAUNCH_CHECK();
    double v = 0.0;
    MGSR_CUDA_TRY(cudaMemcpyAsync(&v, scal, sizeof(double), cudaMemcpyDeviceToHost, st));
    MGSR_CUDA_TRY(cudaStreamSynchronize(st));
    *out_host = sqrt(v);
    return MGSR_OK;
}
