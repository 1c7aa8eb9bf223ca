// Microbenchmark (bring-up tool, not part of the library): cycles per
// tcgen05.mma (cta_group::1, kind::f16, M = 128, K = 16, bf16) for several N
// and shared-memory layouts, operands resident in smem, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_bench tests/umma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(layout) << 61;
    return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

// mode: 0 = SWIZZLE_NONE K-major (8-row core matrices, 16 B rows), 1 = SWIZZLE_128B K-major,
//       2 = SWIZZLE_NONE with A start shifted by 1 row (misaligned, like the conv taps)
__global__ void __launch_bounds__(128, 1) k_bench(int n, int mode, int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (warp == 0) {
        const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm + 64 * 1024);
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
        uint64_t a0, b0;
        uint32_t a_kstep, b_kstep;
        if (mode == 1) {   // 128B swizzle: rows of 128 B (64 bf16 of K), 8-row atoms of 1 KB, SBO = 1024
            a0 = make_desc(a_base, 16, 1024, 2);
            b0 = make_desc(b_base, 16, 1024, 2);
            a_kstep = 32 / 16;   // K = 16 elements = 32 bytes within the swizzle atom
            b_kstep = 32 / 16;
        } else {           // no swizzle: planes of 8 K-elements; plane stride LBO
            const uint32_t a_lbo = 128 * 16, b_lbo = n * 16;
            a0 = make_desc(a_base + (mode == 2 ? 16 : 0), a_lbo, 128, 0);
            b0 = make_desc(b_base, b_lbo, 128, 0);
            a_kstep = 2 * a_lbo / 16;
            b_kstep = 2 * b_lbo / 16;
        }
        long long t0 = clock64();
        if (elect_one()) {
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    mma_bf16(tmem, a0 + uint64_t(ks * a_kstep), b0 + uint64_t(ks * b_kstep), idesc, (it | ks) > 0);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        }
        __syncwarp();
        asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)));
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    long long *d;
    cudaMalloc(&d, sizeof(long long) * 148);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode)
        for (int n : {16, 64, 128, 192, 256}) {
            k_bench<<<148, 128, 160 * 1024>>>(n, mode, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            const double per = avg / (iters * 4.0);
            const double ideal = 128.0 * n / 256.0;
            printf("mode %d (%s) N=%3d: %7.2f cycles/MMA  ideal %5.1f  -> %5.1f%% of peak  %s\n", mode,
                   mode == 0 ? "noswz" : (mode == 1 ? "swz128" : "noswz+1row"), n, per, ideal, 100.0 * ideal / per,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
