// fp64 stencil kernels of the V-cycle: red-black Gauss-Seidel (temporally
// blocked in shared memory), fused residual -> half-injection restriction,
// separable Keys spline prolongation fused with the correction add, and the
// solve-loop logging pass.  Compiled with --fmad=false so every product and
// sum rounds exactly as the reference's -ffp-contract=off C loops
// (pkg/setup.py:37-39).
#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "common.cuh"
#include "stencil.cuh"

namespace mgsr {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }

__device__ __forceinline__ int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

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
    const int64_t total = int64_t(n) * half;
    const double sh = fs.load_shift();
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int i = int(t / half);
        int j = 2 * int(t % half) + ((i + color) & 1);
        int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
        int64_t c = int64_t(i) * n + j;
        double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[int64_t(i) * n + jm1]) +
                    p[int64_t(i) * n + jp1];
        p[c] = (nb - h2 * fs.at(c, sh)) * 0.25;
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

// Whole small grid in one CTA: all sweeps with the reference's per-sweep mean
// subtraction done exactly in order (block reduction), optional fused coarse
// residual.  n <= kSmallN.
__global__ void __launch_bounds__(1024) k_gs_small(double *__restrict__ p, FSrc fs, int n, double h2,
                                                   int sweeps, int zero_init, double *mean_out) {
    extern __shared__ double sm[];
    double *sp = sm, *sf = sm + n * n;
    __shared__ double sred[32];
    const int tid = threadIdx.x, nt = blockDim.x, nn = n * n;
    const double sh = fs.load_shift();
    for (int c = tid; c < nn; c += nt) {
        sp[c] = zero_init ? 0.0 : p[c];
        sf[c] = fs.at(c, sh);
    }
    __syncthreads();
    const int half = nn >> 1;
    for (int s = 0; s < sweeps; ++s) {
        for (int color = 0; color < 2; ++color) {
            for (int t = tid; t < half; t += nt) {
                int i = t / (n >> 1);
                int j = 2 * (t % (n >> 1)) + ((i + color) & 1);
                int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
                int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
                double nb = ((sp[im1 * n + j] + sp[ip1 * n + j]) + sp[i * n + jm1]) + sp[i * n + jp1];
                sp[i * n + j] = (nb - h2 * sf[i * n + j]) * 0.25;
            }
            __syncthreads();
        }
        double acc = 0.0;
        for (int c = tid; c < nn; c += nt) acc += sp[c];
        acc = warp_sum(acc);
        if ((tid & 31) == 0) sred[tid >> 5] = acc;
        __syncthreads();
        if (tid < 32) {
            double w = tid < (nt >> 5) ? sred[tid] : 0.0;
            w = warp_sum(w);
            if (tid == 0) sred[0] = w;
        }
        __syncthreads();
        const double mean = sred[0] * (1.0 / double(nn));
        for (int c = tid; c < nn; c += nt) sp[c] -= mean;
        __syncthreads();
    }
    for (int c = tid; c < nn; c += nt) p[c] = sp[c];
    if (tid == 0 && mean_out) *mean_out = 0.0;   // already gauge-fixed
}

// Temporally blocked K-sweep GS.  A TY x TX tile plus a halo of H cells is
// staged in shared memory; 2K half-sweeps run there (the invalid outer ring
// grows by one cell per half-sweep and never reaches the interior +- 1), the
// interior is written back once.  HBM traffic: read p and f once, write p
// once for K sweeps.  With RC the residual at the coarse (even, even) points
// of the interior is computed from the final values and written raw
// (half-injection input, solver.py:178-179).
template <int K, bool RC>
__global__ void __launch_bounds__(kTbThreads) k_gs_tb(const double *__restrict__ pin, double *__restrict__ pout,
                                                      FSrc fs, int n, double h2, int zero_init, double inv_h2,
                                                      double *__restrict__ rc, RedSlot slot, double *mean_out,
                                                      RedSlot rc_slot, double *rc_mean_out) {
    constexpr int H = 2 * K + (RC ? 1 : 0);
    constexpr int W = kTbTX + 2 * H, HH = kTbTY + 2 * H;
    extern __shared__ double sm[];
    double *sp = sm, *sf = sm + W * HH;
    const int tid = threadIdx.x;
    const int gx0 = blockIdx.x * kTbTX - H, gy0 = blockIdx.y * kTbTY - H;
    const double sh = fs.load_shift();
    for (int idx = tid; idx < W * HH; idx += kTbThreads) {
        int ly = idx / W, lx = idx - ly * W;
        int gi = gy0 + ly, gj = gx0 + lx;
        gi = ((gi % n) + n) % n;
        gj = ((gj % n) + n) % n;
        int64_t g = int64_t(gi) * n + gj;
        sp[idx] = zero_init ? 0.0 : pin[g];
        sf[idx] = fs.at(g, sh);
    }
    __syncthreads();
    constexpr int HW = (W - 2) / 2;
#pragma unroll 1
    for (int hs = 0; hs < 2 * K; ++hs) {
        const int color = hs & 1;
        for (int idx = tid; idx < (HH - 2) * HW; idx += kTbThreads) {
            int ly = 1 + idx / HW, k = idx - (ly - 1) * HW;
            int lx = 1 + ((color - gy0 - ly - gx0 - 1) & 1) + 2 * k;
            int c = ly * W + lx;
            double nb = ((sp[c - W] + sp[c + W]) + sp[c - 1]) + sp[c + 1];
            sp[c] = (nb - h2 * sf[c]) * 0.25;
        }
        __syncthreads();
    }
    double v[1] = {0.0};
    double r[1] = {0.0};
    for (int idx = tid; idx < kTbTX * kTbTY; idx += kTbThreads) {
        int ly = idx / kTbTX, lx = idx - ly * kTbTX;
        int gi = gy0 + H + ly, gj = gx0 + H + lx;
        if (gi >= n || gj >= n) continue;
        int c = (ly + H) * W + lx + H;
        double val = sp[c];
        pout[int64_t(gi) * n + gj] = val;
        v[0] += val;
        if (RC && !(gi & 1) && !(gj & 1)) {
            double nb = ((sp[c - W] + sp[c + W]) + sp[c - 1]) + sp[c + 1];
            double res = sf[c] - ((nb - 4.0 * val) * inv_h2);
            rc[int64_t(gi >> 1) * (n >> 1) + (gj >> 1)] = res;
            r[0] += res;
        }
    }
    grid_reduce<1>(v, slot, mean_out, 1.0 / (double(n) * double(n)));
    if (RC) {
        __syncthreads();
        grid_reduce<1>(r, rc_slot, rc_mean_out, 4.0 / (double(n) * double(n)));
    }
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
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int ic = int(t / nc), jc = int(t - int64_t(ic) * nc);
        int i = ic * s, j = jc * s;
        int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
        int64_t c = int64_t(i) * n + j;
        double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[int64_t(i) * n + jm1]) +
                    p[int64_t(i) * n + jp1];
        double res = fs.at(c, sh) - ((nb - 4.0 * p[c]) * inv_h2);
        rc[t] = res;
        v[0] += res;
    }
    grid_reduce<1>(v, slot, mean_out, 1.0 / double(total));
}

// Full-grid laplacian (API kernel; reference kernels.laplacian).
__global__ void k_laplacian(const double *__restrict__ p, double *__restrict__ out, int n, double inv_h2) {
    const int64_t total = int64_t(n) * n;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int i = int(t / n), j = int(t - int64_t(i) * n);
        int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
        double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[int64_t(i) * n + jm1]) +
                    p[int64_t(i) * n + jp1];
        out[t] = (nb - 4.0 * p[t]) * inv_h2;
    }
}

// r = f - L p (raw) and its mean; API residual then subtracts.
__global__ void k_residual_raw(const double *__restrict__ p, const double *__restrict__ f, double *__restrict__ r,
                               int n, double inv_h2, RedSlot slot, double *mean_out) {
    const int64_t total = int64_t(n) * n;
    double v[1] = {0.0};
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int i = int(t / n), j = int(t - int64_t(i) * n);
        int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
        double nb = ((p[int64_t(im1) * n + j] + p[int64_t(ip1) * n + j]) + p[int64_t(i) * n + jm1]) +
                    p[int64_t(i) * n + jp1];
        double res = f[t] - ((nb - 4.0 * p[t]) * inv_h2);
        r[t] = res;
        v[0] += res;
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
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int ic = int(t / nc), jc = int(t - int64_t(ic) * nc);
        double x = fine[int64_t(ic) * s * n + int64_t(jc) * s];
        coarse[t] = x;
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
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int I = int(t / n), J = int(t - int64_t(I) * n);
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
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int i = int(t / n), j = int(t - int64_t(i) * n);
        int im1 = i > 0 ? i - 1 : n - 1, ip1 = i < n - 1 ? i + 1 : 0;
        int jm1 = j > 0 ? j - 1 : n - 1, jp1 = j < n - 1 ? j + 1 : 0;
        double o = out[t];
        double nb = ((out[int64_t(im1) * n + j] + out[int64_t(ip1) * n + j]) + out[int64_t(i) * n + jm1]) +
                    out[int64_t(i) * n + jp1];
        double np_ = o - m;
        double d = np_ - p[t];
        double r = fs.at(t, sh) - ((nb - 4.0 * o) * inv_h2);
        p[t] = np_;
        v[0] += d * d;
        v[1] += r;
        v[2] += r * r;
    }
    grid_reduce<3>(v, slot, acc_out, 1.0 / double(total));
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

int grid_for(int64_t work, int threads) {
    int64_t b = (work + threads - 1) / threads;
    int64_t cap = 148 * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return int(b);
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
        k_gs_small<<<1, 1024, smem, st>>>(p_out, fs, n, h2, sweeps, zero_init, mean_out);
        MGSR_LAUNCH_CHECK();
        if (rc) {
            k_res_restrict<<<grid_for(int64_t(n / 2) * (n / 2), 256), 256, 0, st>>>(p_out, fs, n, 2, inv_h2, rc,
                                                                                       s1, rc_mean);
            MGSR_LAUNCH_CHECK();
        }
        return MGSR_OK;
    }
    if (n % kTbTX == 0 && n % kTbTY == 0 && sweeps >= 1 && p_in != p_out) {
        const int chunks = (sweeps + kTbMaxK - 1) / kTbMaxK;
        if (chunks > 1 && !tmp) { set_error("gs: chunked sweeps need a scratch buffer"); return MGSR_E_BAD_ARG; }
        int done = 0;
        const double *src = p_in;
        for (int ci = 0; ci < chunks; ++ci) {
            int k = sweeps - done;
            if (k > kTbMaxK) k = kTbMaxK;
            const bool last = ci == chunks - 1;
            const bool rcl = last && rc;
            double *dst = ((chunks - 1 - ci) % 2 == 0) ? p_out : tmp;
            const int zi = (ci == 0) ? zero_init : 0;
            dim3 grid(n / kTbTX, n / kTbTY);
            const int H = 2 * k + (rcl ? 1 : 0);
            size_t smem = 2 * sizeof(double) * (kTbTX + 2 * H) * (kTbTY + 2 * H);
            double *mo = last ? mean_out : nullptr;
#define MGSR_TB_CASE(KK)                                                                                   \
    case KK:                                                                                               \
        if (rcl) {                                                                                         \
            cudaFuncSetAttribute(k_gs_tb<KK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
            k_gs_tb<KK, true><<<grid, kTbThreads, smem, st>>>(src, dst, fs, n, h2, zi, inv_h2, rc, s0, mo, s1,  \
                                                              rc_mean);                                   \
        } else {                                                                                           \
            cudaFuncSetAttribute(k_gs_tb<KK, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
            k_gs_tb<KK, false><<<grid, kTbThreads, smem, st>>>(src, dst, fs, n, h2, zi, inv_h2, nullptr, s0, mo, \
                                                               s2, nullptr);                              \
        }                                                                                                  \
        break;
            switch (k) {
                MGSR_TB_CASE(1)
                MGSR_TB_CASE(2)
                MGSR_TB_CASE(3)
                MGSR_TB_CASE(4)
            }
#undef MGSR_TB_CASE
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
    int g = grid_for(int64_t(n) * n / 2, 256);
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
        k_res_restrict<<<grid_for(int64_t(n / 2) * (n / 2), 256), 256, 0, st>>>(p_out, fs, n, 2, inv_h2, rc, s1,
                                                                                   rc_mean);
        MGSR_LAUNCH_CHECK();
    }
    return MGSR_OK;
}

int launch_prolong_add(const double *c, int nc, int s, const double *base, const double *bshift, double *out,
                       double *mean_out, void *red_slot, cudaStream_t st) {
    int64_t total = int64_t(nc) * s * nc * s;
    RedSlot sl = red_slot_at(red_slot);
    k_prolong_add<<<grid_for(total, 256), 256, 0, st>>>(c, nc, s, base, bshift, out, sl, mean_out,
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
    k_res_restrict<<<grid_for(int64_t(nc) * nc, 256), 256, 0, st>>>(p, fs, n, s, 1.0 / ((2.0 * M_PI / n) * (2.0 * M_PI / n)),
                                                                       rc, sl, rc_mean);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_finalize(const double *out, const double *mean_ptr, double *p, FSrc fs, int n, double *acc3,
                    double *stats2, void *red_slot, cudaStream_t st) {
    RedSlot sl = red_slot_at(red_slot);
    double h = 2.0 * M_PI / n;
    k_finalize<<<grid_for(int64_t(n) * n, 256), 256, 0, st>>>(out, mean_ptr, p, fs, n, 1.0 / (h * h), sl, acc3);
    MGSR_LAUNCH_CHECK();
    k_stats_sqrt<<<1, 1, 0, st>>>(acc3, stats2);
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

static int check_ws(void *ws, size_t bytes) {
    if (!ws || bytes < mgsr_workspace_bytes(0)) {
        set_error("workspace too small");
        return MGSR_E_WORKSPACE;
    }
    return MGSR_OK;
}

extern "C" int mgsr_gs_sweeps(double *p, const double *f, int64_t n, double h2, int32_t sweeps, void *ws,
                              size_t ws_bytes, void *stream) {
    if (n < 2 || !p || !f || sweeps < 0) { set_error("sweep count must be >= 0"); return MGSR_E_BAD_ARG; }
    if (n % 2) { set_error("red-black coloring needs an even side, got " + std::to_string(n)); return MGSR_E_ODD_SIDE; }
    if (int r = check_ws(ws, ws_bytes)) return r;
    if (sweeps == 0) return MGSR_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double *scal = static_cast<double *>(ws);
    void *red = static_cast<char *>(ws) + 256;
    FSrc fs{f, nullptr, 1.0};
    if (n <= kSmallN)  // exact per-sweep mean subtraction inside one CTA
        return launch_gs(p, p, nullptr, fs, int(n), h2, sweeps, 0, nullptr, nullptr, nullptr, red, st);
    double *tmp = nullptr;
    MGSR_CUDA_TRY(cudaMallocAsync(&tmp, 2 * sizeof(double) * n * n, st));
    int rc = launch_gs(p, tmp, tmp + n * n, fs, int(n), h2, sweeps, 0, nullptr, nullptr, scal, red, st);
    if (rc == MGSR_OK) rc = launch_affine(tmp, p, n * n, scal, 1.0, st);
    cudaFreeAsync(tmp, st);
    return rc;
}

extern "C" int mgsr_laplacian(const double *p, double *out, int64_t n, double inv_h2, void *stream) {
    if (n < 2 || !p || !out) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_laplacian<<<grid_for(n * n, 256), 256, 0, st>>>(p, out, int(n), inv_h2);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

extern "C" int mgsr_residual(const double *p, const double *f, double *r, int64_t n, void *ws, size_t ws_bytes,
                             void *stream) {
    if (n < 2 || !p || !f || !r) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    if (int e = check_ws(ws, ws_bytes)) return e;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double *scal = static_cast<double *>(ws);
    RedSlot sl = red_slot_at(static_cast<char *>(ws) + 256);
    double h = 2.0 * M_PI / double(n);
    k_residual_raw<<<grid_for(n * n, 256), 256, 0, st>>>(p, f, r, int(n), 1.0 / (h * h), sl, scal);
    MGSR_LAUNCH_CHECK();
    return launch_affine(r, r, n * n, scal, 1.0, st);
}

extern "C" int mgsr_restrict(const double *fine, double *coarse, int64_t n, int32_t s, int32_t subtract_mean,
                             void *ws, size_t ws_bytes, void *stream) {
    if (s < 2 || (s & (s - 1))) { set_error("transfer ratio must be a power of two >= 2, got " + std::to_string(s)); return MGSR_E_RATIO; }
    if (n % s) { set_error("fine side " + std::to_string(n) + " is not divisible by ratio " + std::to_string(s)); return MGSR_E_NOT_DIVISIBLE; }
    if (int e = check_ws(ws, ws_bytes)) return e;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double *scal = static_cast<double *>(ws);
    RedSlot sl = red_slot_at(static_cast<char *>(ws) + 256);
    int64_t nc = n / s;
    k_inject<<<grid_for(nc * nc, 256), 256, 0, st>>>(fine, coarse, int(n), s, sl, scal);
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
    if (int e = check_ws(ws, ws_bytes)) return e;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
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
