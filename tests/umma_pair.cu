// Microbenchmark (bring-up tool, not part of the library): cycles per tcgen05.mma.cta_group::2 (kind::f16,
// M = 256 over a CTA pair, K = 16, bf16, SWIZZLE_NONE K-major operands resident in shared memory: A 128 rows
// per CTA as planes of 8 K-elements, B split along N, N/2 rows per CTA in 8-row groups 1 KB apart -- the
// generator's layouts), one pair per two SMs, the leader issues and commits to both CTAs' barriers.
// Ideal: N / 2 cycles per MMA.  mode 1: the K-steps of consecutive MMAs walk over a 64 KB A region instead
// of re-reading the same 16 KB.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_pair tests/umma_pair.cu
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
__device__ __forceinline__ void mma2_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(128, 1) k_pair(int n, int mode, int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm + 96 * 1024);
        // D fp32, bf16 A and B, K-major, N, M = 256
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(256 >> 4) << 24);
        const uint32_t a_lbo = 128 * 16;                       // plane of 8 K-elements: 128 rows x 16 B
        const uint64_t a0 = make_desc(a_base, a_lbo, 128, 0);  // 8-row groups contiguous
        const uint64_t b0 = make_desc(b_base, 128, 1024, 0);   // per 8-row group: 8 K-chunks x 128 B
        const uint32_t a_kstep = 2 * a_lbo / 16, b_kstep = 256 / 16;
        long long t0 = clock64();
        if (rank == 0 && elect_one()) {
            for (int it = 0; it < iters; ++it) {
                const uint32_t a_off = mode == 1 ? uint32_t(it & 3) * 4 * a_kstep : 0u;   // 4 x 16 KB of A
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    mma2_bf16(tmem, a0 + uint64_t(a_off + ks * a_kstep), b0 + uint64_t(ks * b_kstep), idesc, (it | ks) > 0);
            }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(&bar)), "h"((unsigned short)3) : "memory");
        }
        __syncwarp();
        asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)));
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long *d;
    cudaMalloc(&d, sizeof(long long) * 148);
    cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 160 * 1024;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode)
        for (int n : {64, 96, 128, 192, 256}) {
            cudaLaunchKernelEx(&cfg, k_pair, n, mode, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < 148; ++i) avg += h[i];
            avg /= 148;
            const double per = avg / (iters * 4.0), ideal = n / 2.0;
            printf("cta_group::2 M=256 mode %d N=%3d: %7.2f cycles/MMA  ideal %5.1f  -> %5.1f%% of peak  %s\n", mode, n, per,
                   ideal, 100.0 * ideal / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
