// Microbenchmark (bring-up tool, not part of the library): does background shared-memory traffic slow
// tcgen05.mma?  Warp 0 issues M = 128, N = 192, K = 16 bf16 MMAs (cta_group::1, SWIZZLE_NONE K-major,
// operands resident: 96 cycles each when alone, tests/umma_bench.cu) while warps 4..19 stream LDS.128
// (and optionally STS.128) over a separate region, paced by `gap` dependent FMAs per access.  Prints
// cycles per MMA and the background bytes per clock, per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_stress tests/umma_stress.cu
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


constexpr int kStressWarps = 16;

__global__ void __launch_bounds__(128 + 32 * kStressWarps, 1)
    k_stress(int n, int iters, int gap, int stores, int conflict, long long *out, unsigned long long *bytes) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        stop = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (warp >= 4 && gap >= 0 && stores == 2) {
        // TMEM-load stress: 32 lanes x 32 columns x 4 B = 4 KB per tcgen05.ld, columns 256.. (the MMAs accumulate in 0..191)
        const uint32_t taddr = tmem + (uint32_t(32 * (warp & 3)) << 16) + 256u + 32u * uint32_t(((warp - 4) >> 2) & 3);
        unsigned long long cnt = 0;
        uint32_t sink = 0;
        float x = 0.f;
        while (!stop) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t r[32];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                      "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
                      "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
                      "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int q = 0; q < 32; ++q) sink ^= r[q];
                for (int g = 0; g < gap; ++g) x = fmaf(x, 1.0001f, 0.5f);
            }
            cnt += 4 * 32 * 4;
        }
        if (sink == 0x12345u || x == 12345.f) out[0] = 1;
        if (lane == 0) atomicAdd(bytes, cnt * 32);
    } else if (warp >= 4 && gap >= 0) {
        // 2 KB per warp: 4 LDS.128 per pass (conflict = 1: every lane's 16 bytes 128 B apart -> 8-way conflicts)
        float4 *reg = reinterpret_cast<float4 *>(sm + 160 * 1024) + (warp - 4) * 128;
        const int li = conflict ? ((lane * 8) & 127) + (lane >> 4) : lane;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned long long cnt = 0;
        while (!stop) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 v = reg[(j * 32 + li) & 127];
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                if (stores) reg[(j * 32 + li) & 127] = acc;
                for (int g = 0; g < gap; ++g) acc.x = fmaf(acc.x, 1.0001f, 0.5f);
            }
            cnt += 4 * 16 * (stores ? 2 : 1);
        }
        if (acc.x == 12345.f) out[0] = 1;
        if (lane == 0) atomicAdd(bytes, cnt * 32);
    }
    if (warp == 0) {
        const uint32_t a_base = smem_u32(sm), b_base = smem_u32(sm + 64 * 1024);
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
        const uint32_t a_lbo = 128 * 16, b_lbo = n * 16;
        const uint64_t a0 = make_desc(a_base, a_lbo, 128, 0), b0 = make_desc(b_base, b_lbo, 128, 0);
        const uint32_t a_kstep = 2 * a_lbo / 16, b_kstep = 2 * b_lbo / 16;
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
        if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    long long *d;
    unsigned long long *bytes;
    cudaMalloc(&d, sizeof(long long) * 148);
    cudaMalloc(&bytes, 8);
    cudaFuncSetAttribute(k_stress, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int iters = 4096, n = 192;
    const int gaps[] = {-1, 256, 64, 32, 16, 8, 4, 0};
    for (int conflict = 0; conflict < 2; ++conflict)
        for (int stores = 0; stores < 3; ++stores)
            for (int gap : gaps) {
                if (gap < 0 && (stores || conflict)) continue;
                if (stores == 2 && conflict) continue;
                cudaMemset(bytes, 0, 8);
                k_stress<<<148, 128 + 32 * kStressWarps, 200 * 1024>>>(n, iters, gap, stores, conflict, d, bytes);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[148];
                unsigned long long hb = 0;
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                cudaMemcpy(&hb, bytes, 8, cudaMemcpyDeviceToHost);
                double avg = 0;
                for (int i = 0; i < 148; ++i) avg += h[i];
                avg /= 148;
                printf("N=192 %s%s gap %4d: %7.2f cycles/MMA (alone 96)  background %6.1f B/clk/SM  %s\n",
                       conflict ? "8-way-conflicted " : "", stores == 2 ? "tcgen05.ld" : (stores ? "LDS+STS" : "LDS    "), gap, avg / (iters * 4.0),
                       double(hb) / 148.0 / avg, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
