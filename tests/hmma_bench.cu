// Microbenchmark (bring-up tool): mma.sync m16n8k16 bf16 latency (dependent chain) and throughput
// (independent chains) per SM on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma_16816(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int CH>
__global__ void k(int iters, long long *out, float *sink) {
    uint32_t a[4] = {threadIdx.x, 2u, 3u, 4u}, b[2] = {5u, 6u};
    float c[CH][4] = {};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < CH; ++j) mma_16816(c[j], a, b);
    long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < CH; ++j) s += c[j][0];
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; sink[blockIdx.x] = s; }
}
template <int CH>
void run(int warps) {
    long long *d; float *sk; cudaMalloc(&d, 8 * 148); cudaMalloc(&sk, 4 * 148);
    const int iters = 2048;
    k<CH><<<148, 32 * warps>>>(iters, d, sk);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = double(h[0]) / (iters * CH);
    printf("chains/warp %d warps/SM %2d: %6.2f cycles per mma per warp  -> %6.1f MACs/cycle/SM\n", CH, warps, cyc,
           2048.0 * warps / cyc);
}
int main() { run<1>(1); run<4>(1); run<8>(1); run<4>(4); run<4>(8); run<4>(16); run<8>(16); return 0; }
