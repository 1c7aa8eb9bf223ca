// Seeded initial iterate of solve() on the device, bit-exact with the reference's host draw
// (solver.py:298-300):
//     start = default_rng(seed).uniform(-p_max, p_max, (n, n));  start - start.mean()
//
// numpy's default_rng is PCG64 (128-bit LCG, XSL-RR output; the generator steps, then
// outputs), next_double = (next_uint64 >> 11) * 2^-53 and uniform = low + (high - low) * d
// (two roundings: compiled with --fmad=false).  The SeedSequence hashing stays on the host
// (bit_generator.state gives the 128-bit state and increment); the device jumps each
// thread to its own offset in the stream (LCG jump-ahead, O(log i) 128-bit products).
//
// start.mean() is numpy's pairwise sum / count.  For a C-contiguous array whose size is
// a power of two >= 128 that sum is a perfect binary tree over leaves of 128 consecutive
// values, each leaf summed with eight interleaved accumulators combined as
// ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) (numpy/_core/src/umath/loops_utils.h
// pairwise_sum; checked bitwise against numpy in tests/test_host.py).  One thread per leaf
// draws and sums its 128 values; tree kernels combine adjacent pairs level by level.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mgsr {

typedef unsigned __int128 u128;

static __device__ __forceinline__ u128 pcg_mult() {
    return (u128(0x2360ED051FC65DA4ull) << 64) | u128(0x4385DF649FCCF645ull);
}

// state after `delta` steps (pcg_advance_lcg_128)
static __device__ u128 pcg_advance(u128 state, unsigned long long delta, u128 inc) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1ull) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

static __device__ __forceinline__ uint64_t pcg_output(u128 s) {
    const uint64_t x = uint64_t(s >> 64) ^ uint64_t(s);
    const unsigned rot = unsigned(s >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int kLeaf = 128;

__global__ void k_pcg_leaves(double *__restrict__ out, double *__restrict__ leaf_sum, long long nleaves,
                             uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, double low,
                             double scale) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= nleaves) return;
    const u128 inc = (u128(inc_hi) << 64) | u128(inc_lo);
    u128 s = pcg_advance((u128(st_hi) << 64) | u128(st_lo), (unsigned long long)(t * kLeaf), inc);
    const u128 m = pcg_mult();
    double r[8];
    double2 *dst = reinterpret_cast<double2 *>(out + t * kLeaf);
#pragma unroll 1
    for (int k = 0; k < kLeaf / 8; ++k) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            s = s * m + inc;
            const double d = double(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
            v[j] = low + scale * d;
            r[j] = k == 0 ? v[j] : r[j] + v[j];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[4 * k + j] = make_double2(v[2 * j], v[2 * j + 1]);
    }
    leaf_sum[t] = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

// out[b] = perfect pairwise tree over in[b * 2048 .. b * 2048 + len), len = min(m, 2048), a power of two
__global__ void __launch_bounds__(1024) k_pair_tree(const double *__restrict__ in, long long m, double *__restrict__ out) {
    __shared__ double s[2048];
    const long long base = blockIdx.x * 2048ll;
    const int len = int(m - base < 2048 ? m - base : 2048);
    for (int i = threadIdx.x; i < len; i += blockDim.x) s[i] = in[base + i];
    __syncthreads();
    for (int w = len >> 1; w >= 1; w >>= 1) {
        double v = 0.0;
        if (int(threadIdx.x) < w) v = s[2 * threadIdx.x] + s[2 * threadIdx.x + 1];
        __syncthreads();
        if (int(threadIdx.x) < w) s[threadIdx.x] = v;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

// out[i] -= (0 + total) / count
__global__ void k_sub_mean(double *__restrict__ out, long long count, const double *total) {
    const double mean = (0.0 + *total) / double(count);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
        out[i] = out[i] - mean;
}

int grid_for(int64_t work, int threads);

}  // namespace mgsr

using namespace mgsr;

extern "C" size_t mgsr_initial_iterate_workspace_bytes(int64_t count) {
    const int64_t leaves = count / kLeaf;
    return sizeof(double) * size_t(leaves + (leaves + 2047) / 2048 + 64) + 256;
}

extern "C" int mgsr_initial_iterate(double *out, int64_t count, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                    uint64_t inc_lo, double low, double high, void *ws, size_t ws_bytes,
                                    void *stream) {
    if (!out || !ws) { set_error("initial_iterate: null buffer"); return MGSR_E_BAD_ARG; }
    if (count < kLeaf || (count & (count - 1)) != 0) {
        set_error("initial_iterate: size must be a power of two >= 128 (numpy pairwise tree)");
        return MGSR_E_UNSUPPORTED;
    }
    if (ws_bytes < mgsr_initial_iterate_workspace_bytes(count)) {
        set_error("initial_iterate: workspace too small");
        return MGSR_E_WORKSPACE;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const long long leaves = count / kLeaf;
    double *a = static_cast<double *>(ws);
    double *b = a + leaves;
    k_pcg_leaves<<<int((leaves + 127) / 128), 128, 0, st>>>(out, a, leaves, state_hi, state_lo, inc_hi, inc_lo, low,
                                                            high - low);
    MGSR_LAUNCH_CHECK();
    long long m = leaves;
    while (m > 1) {
        const long long nb = (m + 2047) / 2048;
        k_pair_tree<<<int(nb), 1024, 0, st>>>(a, m, b);
        MGSR_LAUNCH_CHECK();
        double *t = a;
        a = b;
        b = t;
        m = nb;
    }
    k_sub_mean<<<grid_for(count, 256), 256, 0, st>>>(out, count, a);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}
