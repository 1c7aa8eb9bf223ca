// Shared helpers for the mgsr_b200 CUDA library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "mgsr_b200.h"

namespace mgsr {

// Thread-local last-error text, surfaced by mgsr_last_error().
void set_error(const std::string &msg);

#define MGSR_CUDA_TRY(expr)                                                              \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            ::mgsr::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));       \
            return MGSR_E_CUDA;                                                          \
        }                                                                                \
    } while (0)

#define MGSR_LAUNCH_CHECK()                                                              \
    do {                                                                                 \
        cudaError_t _e = cudaGetLastError();                                             \
        if (_e != cudaSuccess) {                                                         \
            ::mgsr::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e));  \
            return MGSR_E_CUDA;                                                          \
        }                                                                                \
    } while (0)

constexpr int kRedMaxBlocks = 8192;   // capacity of the partial-sum array in a reduction slot
constexpr int kRedMaxVals = 4;        // values reduced together

// A reduction slot: a ticket counter plus partials.  Lives in device memory;
// the counter returns to 0 after every use, so slots are reusable across
// launches and CUDA-graph replays.
struct RedSlot {
    unsigned *counter;
    double *partials;   // kRedMaxBlocks * kRedMaxVals
};

constexpr size_t kRedSlotBytes = 256 + sizeof(double) * kRedMaxBlocks * kRedMaxVals;

__host__ __device__ inline RedSlot red_slot_at(void *base) {
    RedSlot s;
    s.counter = reinterpret_cast<unsigned *>(base);
    s.partials = reinterpret_cast<double *>(reinterpret_cast<char *>(base) + 256);
    return s;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic grid-wide sum of NV values per thread.  Every block writes its
// fixed-order partial; the last block to arrive (ticket counter) sums the
// partials in index order and writes result[k] = total_k * scale.  Bitwise
// reproducible for a fixed launch geometry.  blockDim.x must be a multiple of 32.
// grid_reduce_to: component k goes to *outs[k] * scales[k] (null outs[k] skipped;
// all null -> no-op).  One fence + one ticket per block for all NV sums.
// Returns true in thread 0 of the last block, after it wrote the outputs.
template <int NV>
__device__ bool grid_reduce_to(double (&v)[NV], RedSlot slot, double *const (&outs)[NV], const double (&scales)[NV]) {
    bool any = false;
#pragma unroll
    for (int k = 0; k < NV; ++k) any |= outs[k] != nullptr;
    if (!any) return false;   // uniform across the grid
    __shared__ double sred[NV][32];
    __shared__ bool s_last;
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthreads = blockDim.x * blockDim.y * blockDim.z;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthreads >> 5;
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblocks = gridDim.x * gridDim.y * gridDim.z;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double w = warp_sum(v[k]);
        if (lane == 0) sred[k][warp] = w;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double w = lane < nwarps ? sred[k][lane] : 0.0;
            w = warp_sum(w);
            if (lane == 0) slot.partials[bid * NV + k] = w;
        }
    }
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(slot.counter, 1u) == unsigned(nblocks - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    double acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
    for (int b = tid; b < nblocks; b += nthreads) {
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] += __ldcg(slot.partials + b * NV + k);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double w = warp_sum(acc[k]);
        if (lane == 0) sred[k][warp] = w;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double w = lane < nwarps ? sred[k][lane] : 0.0;
            w = warp_sum(w);
            if (lane == 0 && outs[k]) *outs[k] = w * scales[k];
        }
    }
    if (tid == 0) *slot.counter = 0u;
    return tid == 0;
}

template <int NV>
__device__ __forceinline__ void grid_reduce(double (&v)[NV], RedSlot slot, double *result, double scale) {
    double *outs[NV];
    double scales[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        outs[k] = result ? result + k : nullptr;
        scales[k] = scale;
    }
    grid_reduce_to<NV>(v, slot, outs, scales);
}

// Source of a right-hand side: f_eff = (f - *shift) * scale when shift != null,
// else f.  Matches the reference's materialised 0.5 * (restrict(r) - mean)
// bit for bit (solver.py:178-179, transfer.py:36-38).
struct FSrc {
    const double *f;
    const double *shift;   // device scalar or nullptr
    double scale;
    __device__ __forceinline__ double at(int64_t idx, double sh) const {
        return shift ? (f[idx] - sh) * scale : f[idx];
    }
    __device__ __forceinline__ double load_shift() const { return shift ? *shift : 0.0; }
};

}  // namespace mgsr
