// Generator inference on CUDA cores in fp32 (precision mode MGSR_PREC_FP32)
// and the windowed SR-prolongation glue (gather / stitch / denormalise).
//
// Reference: srmodel.py:285-344 (replicate-padded same-size correlation,
// PReLU, BN eps=1e-5, pixel shuffle c*4+i*2+j -> (i,j), tail bias + s*tanh(x/s)),
// srmodel.py:414-487 (6x6 windows at stride 2, central-band stitch, channel
// mean, sign-preserving log map).  General window side (the second generator
// application of a x4 pass runs on 12x12); this is the reference-precision
// path, the tensor-core path lives in generator_tc.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "generator.cuh"
#include "stencil.cuh"

namespace mgsr {

enum { OP_PRELU = 0, OP_BN_PRELU = 1, OP_BN_RES = 2, OP_SHUF_PRELU = 3, OP_TAIL = 4 };

struct Epi {
    const float *scale, *shift, *alpha, *bias;
    const float *res;   // OP_BN_RES residual input (may alias out)
    float tanh_s;
};

constexpr int kConvThreads = 256, kConvOB = 16;

// Same-size correlation with replicate padding, CTA = (sample, 16 output
// channels); input channels staged through shared memory in chunks.
template <int K, int MAXP, int OP>
__global__ void __launch_bounds__(kConvThreads) k_conv_simt(const float *__restrict__ in, int C, int H,
                                                            const float *__restrict__ w, int O,
                                                            float *__restrict__ out, Epi ep, int cc_max) {
    extern __shared__ float s_in[];
    constexpr int P = K / 2;
    const int n = blockIdx.x, ob = blockIdx.y * kConvOB, tid = threadIdx.x;
    const int HW = H * H, HP = H + K - 1;
    const int nout = kConvOB * HW;
    float acc[MAXP];
#pragma unroll
    for (int k = 0; k < MAXP; ++k) acc[k] = 0.f;
    for (int c0 = 0; c0 < C; c0 += cc_max) {
        const int cc = min(cc_max, C - c0);
        __syncthreads();
        for (int idx = tid; idx < cc * HP * HP; idx += kConvThreads) {
            int c = idx / (HP * HP), r = idx - c * HP * HP;
            int yy = min(max(r / HP - P, 0), H - 1), xx = min(max(r % HP - P, 0), H - 1);
            s_in[idx] = in[((int64_t(n) * C + c0 + c) * H + yy) * H + xx];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MAXP; ++k) {
            const int idx = tid + k * kConvThreads;
            if (idx >= nout) break;
            const int o = ob + idx / HW, pix = idx % HW, y = pix / H, x = pix % H;
            if (o >= O) continue;
            const float *wo = w + (int64_t(o) * C + c0) * K * K;
            float a = acc[k];
            for (int c = 0; c < cc; ++c) {
                const float *si = s_in + (c * HP + y) * HP + x;
                const float *wc = wo + c * K * K;
#pragma unroll
                for (int dy = 0; dy < K; ++dy)
#pragma unroll
                    for (int dx = 0; dx < K; ++dx) a = fmaf(si[dy * HP + dx], __ldg(wc + dy * K + dx), a);
            }
            acc[k] = a;
        }
    }
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
        const int idx = tid + k * kConvThreads;
        if (idx >= nout) break;
        const int o = ob + idx / HW, pix = idx % HW, y = pix / H, x = pix % H;
        if (o >= O) continue;
        float v = acc[k];
        if (OP == OP_PRELU) {
            out[(int64_t(n) * O + o) * HW + pix] = v > 0.f ? v : ep.alpha[o] * v;
        } else if (OP == OP_BN_PRELU) {
            v = fmaf(v, ep.scale[o], ep.shift[o]);
            out[(int64_t(n) * O + o) * HW + pix] = v > 0.f ? v : ep.alpha[o] * v;
        } else if (OP == OP_BN_RES) {
            int64_t oi = (int64_t(n) * O + o) * HW + pix;
            out[oi] = ep.res[oi] + fmaf(v, ep.scale[o], ep.shift[o]);
        } else if (OP == OP_SHUF_PRELU) {
            const int c = o >> 2, i = (o >> 1) & 1, j = o & 1, W2 = 2 * H;
            v = v > 0.f ? v : ep.alpha[c] * v;
            out[((int64_t(n) * (O >> 2) + c) * W2 + 2 * y + i) * W2 + 2 * x + j] = v;
        } else {
            const float s = ep.tanh_s;
            out[(int64_t(n) * O + o) * HW + pix] = s * tanhf((v + ep.bias[o]) / s);
        }
    }
}

// Register-tiled form: CTA = (NW windows, a block of OB <= 16 output channels); thread = one
// pixel (or MAXP pixels when a window has more than 256) of one window, accumulating all OB
// channels, so each staged input value feeds OB FMAs and the block's weights ([c][tap][oc] in
// shared memory, read as float4 broadcasts) feed every pixel.  Per output the accumulation order
// (c ascending, dy, dx, fmaf) is k_conv_simt's, so results are bitwise identical.
constexpr int kConv2Threads = 256, kConv2OB = 16, kConv2CC = 16;

template <int K, int MAXP, int OP, int OB>
__global__ void __launch_bounds__(kConv2Threads) k_conv_rt(const float *__restrict__ in, int N, int C, int H,
                                                          const float *__restrict__ w, int O,
                                                          float *__restrict__ out, Epi ep, int nw) {
    extern __shared__ __align__(16) float sm2[];
    constexpr int P = K / 2, KK = K * K;
    const int HW = H * H, HP = H + K - 1, HP2 = HP * HP;
    const int n0 = blockIdx.x * nw, ob = blockIdx.y * OB;
    const int OBn = min(OB, O - ob);
    float *s_w = sm2;                                   // [cc][KK][16]
    float *s_in = sm2 + kConv2CC * KK * OB;       // [nw][cc][HP][HP]
    const int tid = threadIdx.x;
    float acc[MAXP][OB];
#pragma unroll
    for (int k = 0; k < MAXP; ++k)
#pragma unroll
        for (int o = 0; o < OB; ++o) acc[k][o] = 0.f;
    int wl[MAXP], py[MAXP], px[MAXP];
    bool act[MAXP];
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
        const int slot = tid + k * kConv2Threads;
        wl[k] = slot / HW;
        const int pix = slot - wl[k] * HW;
        py[k] = pix / H;
        px[k] = pix - py[k] * H;
        act[k] = wl[k] < nw && n0 + wl[k] < N;
    }
    for (int c0 = 0; c0 < C; c0 += kConv2CC) {
        const int cc = min(kConv2CC, C - c0);
        __syncthreads();
        for (int idx = tid; idx < nw * cc * HP2; idx += kConv2Threads) {
            const int wi = idx / (cc * HP2), r0 = idx - wi * cc * HP2, c = r0 / HP2, r = r0 - c * HP2;
            const int yy = min(max(r / HP - P, 0), H - 1), xx = min(max(r % HP - P, 0), H - 1);
            const int n = n0 + wi;
            s_in[idx] = n < N ? in[((int64_t(n) * C + c0 + c) * H + yy) * H + xx] : 0.f;
        }
        for (int idx = tid; idx < cc * KK * OB; idx += kConv2Threads) {
            const int o = idx % OB, t = (idx / OB) % KK, c = idx / (OB * KK);
            s_w[idx] = o < OBn ? __ldg(w + (int64_t(ob + o) * C + c0 + c) * KK + t) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < MAXP; ++k) {
            if (!act[k]) continue;
            for (int c = 0; c < cc; ++c) {
                const float *si = s_in + ((wl[k] * cc + c) * HP + py[k]) * HP + px[k];
                const float4 *wc = reinterpret_cast<const float4 *>(s_w + c * KK * OB);
#pragma unroll
                for (int dy = 0; dy < K; ++dy)
#pragma unroll
                    for (int dx = 0; dx < K; ++dx) {
                        const float v = si[dy * HP + dx];
                        const float4 *wt = wc + (dy * K + dx) * (OB / 4);
#pragma unroll
                        for (int q = 0; q < OB / 4; ++q) {
                            const float4 w4 = wt[q];
                            acc[k][4 * q] = fmaf(v, w4.x, acc[k][4 * q]);
                            acc[k][4 * q + 1] = fmaf(v, w4.y, acc[k][4 * q + 1]);
                            acc[k][4 * q + 2] = fmaf(v, w4.z, acc[k][4 * q + 2]);
                            acc[k][4 * q + 3] = fmaf(v, w4.w, acc[k][4 * q + 3]);
                        }
                    }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < MAXP; ++k) {
        if (!act[k]) continue;
        const int n = n0 + wl[k], pix = py[k] * H + px[k], y = py[k], x = px[k];
#pragma unroll
        for (int oo = 0; oo < OB; ++oo) {
            if (oo >= OBn) break;
            const int o = ob + oo;
            float v = acc[k][oo];
            if (OP == OP_PRELU) {
                out[(int64_t(n) * O + o) * HW + pix] = v > 0.f ? v : ep.alpha[o] * v;
            } else if (OP == OP_BN_PRELU) {
                v = fmaf(v, ep.scale[o], ep.shift[o]);
                out[(int64_t(n) * O + o) * HW + pix] = v > 0.f ? v : ep.alpha[o] * v;
            } else if (OP == OP_BN_RES) {
                const int64_t oi = (int64_t(n) * O + o) * HW + pix;
                out[oi] = ep.res[oi] + fmaf(v, ep.scale[o], ep.shift[o]);
            } else if (OP == OP_SHUF_PRELU) {
                const int c = o >> 2, i = (o >> 1) & 1, j = o & 1, W2 = 2 * H;
                v = v > 0.f ? v : ep.alpha[c] * v;
                out[((int64_t(n) * (O >> 2) + c) * W2 + 2 * y + i) * W2 + 2 * x + j] = v;
            } else {
                const float sc = ep.tanh_s;
                out[(int64_t(n) * O + o) * HW + pix] = sc * tanhf((v + ep.bias[o]) / sc);
            }
        }
    }
}

// Row-tiled form for the window sides the SR passes use (H = 6 and 12) and 64-wide output blocks:
// thread = one 6-pixel row segment of one window x 8 output channels (48 accumulators).  Per input
// channel and kernel row it reads <= 12 staged inputs and K x 8 weights for K x 48 FMAs (~0.22 shared-
// memory words per FMA; k_conv_rt's one pixel x 16 channels needed 1.06 and was LSU-bound).
//   * The input planes are staged RAW (a window's cc channels are contiguous in (N, C, H, H): straight
//     16-byte copies, no index arithmetic); the replicate padding is resolved when a row is read: the
//     clamped row index per dy, and a compile-time column map per segment (rows_load).
//   * Weights come pre-transposed ([c][tap][O], mgsr_gen::*_t): staging is 16-byte copies and a warp's
//     weight read is one conflict-free 128-byte line.
//   * The epilogue goes through shared memory: every value is placed at its offset inside the CTA's
//     contiguous output block (64 channels x H x H per window; for the pixel shuffle 16 planes of
//     2H x 2H), then the block is written (and the residual read) with coalesced 16-byte accesses.
// Per output the accumulation order is unchanged (c ascending, dy, dx, fmaf) and so are the epilogue
// expressions: bitwise identical to k_conv_simt / k_conv_rt.  One 384-thread CTA per SM (12 warps = 3 per
// scheduler, evenly; three 192-thread CTAs left two schedulers a warp short and measured 8% slower), 16 input
// channels per stage.
#ifndef MGSR_ROW_THREADS
#define MGSR_ROW_THREADS 384
#endif
#ifndef MGSR_ROW_REGS
#define MGSR_ROW_REGS 168
#endif
constexpr int kRowThreads = MGSR_ROW_THREADS;
#ifndef MGSR_ROW_CC
#define MGSR_ROW_CC 16
#endif
template <int K> struct RowCfg { static constexpr int CC = K == 3 ? MGSR_ROW_CC : 1; };   // C must be a multiple

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(uint32_t(__cvta_generic_to_shared(smem))), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

#ifndef MGSR_ROW_FFMA2
#define MGSR_ROW_FFMA2 1
#endif
#ifndef MGSR_TAIL_FFMA2
#define MGSR_TAIL_FFMA2 1
#endif
__device__ __forceinline__ unsigned long long pack2f(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
// (lo, hi) = a * b + (lo, hi) on packed pairs
__device__ __forceinline__ void ffma2(float &lo, float &hi, unsigned long long a, unsigned long long b) {
    unsigned long long d = pack2f(lo, hi);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(d));
}

// v[j] = row[clamp(6 * SEG + j - P, 0, H - 1)], j < K + 5, from the fewest aligned vector loads
template <int K, int H, int SEG>
__device__ __forceinline__ void rows_load(const float *row, float (&v)[K + 5]) {
    constexpr int P = K / 2;
    constexpr int BASE = (H == 12 && K == 3) ? 4 * SEG : 0;
    constexpr int L = H == 6 ? 6 : (K == 3 ? 8 : 12);
    float b[L];
    if constexpr (H == 6) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float2 t = *reinterpret_cast<const float2 *>(row + 2 * j);
            b[2 * j] = t.x;
            b[2 * j + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < L / 4; ++j) {
            const float4 t = *reinterpret_cast<const float4 *>(row + BASE + 4 * j);
            b[4 * j] = t.x;
            b[4 * j + 1] = t.y;
            b[4 * j + 2] = t.z;
            b[4 * j + 3] = t.w;
        }
    }
#pragma unroll
    for (int j = 0; j < K + 5; ++j) {
        int col = 6 * SEG + j - P;
        col = col < 0 ? 0 : (col > H - 1 ? H - 1 : col);
        v[j] = b[col - BASE];
    }
}

template <int K, int H, int SEG>
__device__ __forceinline__ void rows_chunk(const float *s_win, const float *sw, int cc, int y, float (&acc)[6][8]) {
    constexpr int P = K / 2, HW = H * H;
    int yo[K];
#pragma unroll
    for (int dy = 0; dy < K; ++dy) yo[dy] = min(max(y + dy - P, 0), H - 1) * H;
    for (int c = 0; c < cc; ++c) {
        const float *si = s_win + c * HW;
#pragma unroll
        for (int dy = 0; dy < K; ++dy) {
            float v[K + 5];
            rows_load<K, H, SEG>(si + yo[dy], v);
#pragma unroll
            for (int dx = 0; dx < K; ++dx) {
                const float4 wa = *reinterpret_cast<const float4 *>(sw + ((c * K + dy) * K + dx) * 64);
                const float4 wb = *reinterpret_cast<const float4 *>(sw + ((c * K + dy) * K + dx) * 64 + 32);
#if MGSR_ROW_FFMA2
                // two FMAs per instruction (sm_100 FFMA2, each half an IEEE fma: bitwise the scalar result); the
                // activation is the scalar-broadcast operand, a weight pair and an accumulator pair the packed ones
                const unsigned long long w0 = pack2f(wa.x, wa.y), w1 = pack2f(wa.z, wa.w), w2 = pack2f(wb.x, wb.y),
                                         w3 = pack2f(wb.z, wb.w);
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const unsigned long long a2 = pack2f(v[i + dx], v[i + dx]);
                    ffma2(acc[i][0], acc[i][1], a2, w0);
                    ffma2(acc[i][2], acc[i][3], a2, w1);
                    ffma2(acc[i][4], acc[i][5], a2, w2);
                    ffma2(acc[i][6], acc[i][7], a2, w3);
                }
#else
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    const float a = v[i + dx];
                    acc[i][0] = fmaf(a, wa.x, acc[i][0]);
                    acc[i][1] = fmaf(a, wa.y, acc[i][1]);
                    acc[i][2] = fmaf(a, wa.z, acc[i][2]);
                    acc[i][3] = fmaf(a, wa.w, acc[i][3]);
                    acc[i][4] = fmaf(a, wb.x, acc[i][4]);
                    acc[i][5] = fmaf(a, wb.y, acc[i][5]);
                    acc[i][6] = fmaf(a, wb.z, acc[i][6]);
                    acc[i][7] = fmaf(a, wb.w, acc[i][7]);
                }
#endif
            }
        }
    }
}

template <int K, int OP, int H>
__global__ void __maxnreg__(MGSR_ROW_REGS) k_conv_rows(const float *__restrict__ in, int N, int C,
                                                              const float *__restrict__ wt, int O,
                                                              float *__restrict__ out, Epi ep) {
    extern __shared__ __align__(16) float smr[];
    constexpr int KK = K * K, CC = RowCfg<K>::CC, HW = H * H, NSEG = H / 6;
    constexpr int NW = kRowThreads / 8 / (H * NSEG);   // windows per CTA: 4 (H = 6), 1 (H = 12)
    constexpr int RPS = NW * H;                        // row slots per segment (a multiple of 4: warp-uniform SEG)
    constexpr int STAGE = CC * KK * 64 + NW * CC * HW;   // floats per stage: weights [cc][KK][64] + raw planes [NW][cc][H][H]
    const int tid = threadIdx.x, o8 = tid & 7, rs = tid >> 3;
    const int seg = rs / RPS, r2 = rs - seg * RPS, wl = r2 / H, y = r2 - wl * H, x0 = 6 * seg;
    const int n0 = blockIdx.x * NW, ob = blockIdx.y * 64;
    const bool act = n0 + wl < N;
    float acc[6][8];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int o = 0; o < 8; ++o) acc[i][o] = 0.f;
    // chunk c0 of the input channels -> stage buffer `st` (asynchronous 16-byte copies; windows past N are skipped:
    // their threads never compute)
    // The address arithmetic is hoisted: a thread's weight pieces sit (tid & 15) + 16 * ((tid >> 4) + (threads / 16) j) apart,
    // its plane pieces are window-contiguous.
    const float4 *w_src = reinterpret_cast<const float4 *>(wt) + ob / 4 + (tid & 15) + int64_t(tid >> 4) * (O / 4);
    const int w_step = (kRowThreads / 16) * (O / 4);
    auto stage = [&](int c0, int st) {
        float *s_w = smr + st * STAGE, *s_in = s_w + CC * KK * 64;
        constexpr int per = CC * HW / 4;   // 16-byte pieces per window (HW is a multiple of 4)
#pragma unroll
        for (int j = 0; j < (NW * per + kRowThreads - 1) / kRowThreads; ++j) {
            const int idx = tid + j * kRowThreads;
            const int wi = idx / per, k = idx - wi * per, n = n0 + wi;
            if (idx < NW * per && n < N)
                cp_async16(reinterpret_cast<float4 *>(s_in) + idx,
                           reinterpret_cast<const float4 *>(in + (int64_t(n) * C + c0) * HW) + k);
        }
        const float4 *src = w_src + int64_t(c0) * KK * (O / 4);
#pragma unroll
        for (int j = 0; j < (CC * KK * 16 + kRowThreads - 1) / kRowThreads; ++j) {
            const int idx = tid + j * kRowThreads;
            if (idx < CC * KK * 16) cp_async16(reinterpret_cast<float4 *>(s_w) + idx, src + j * w_step);
        }
        cp_async_commit();
    };
    stage(0, 0);
    int st = 0;
    for (int c0 = 0; c0 < C; c0 += CC, st ^= 1) {
        constexpr int cc = CC;
        cp_async_wait_all();
        __syncthreads();   // chunk c0 landed for every thread; everyone is done with the other buffer
        if (c0 + CC < C) stage(c0 + CC, st ^ 1);
        if (act) {
            const float *s_w = smr + st * STAGE, *s_win = s_w + CC * KK * 64 + wl * cc * HW;
            if (NSEG == 1 || seg == 0) rows_chunk<K, H, 0>(s_win, s_w + o8 * 4, cc, y, acc);
            else rows_chunk<K, H, NSEG - 1>(s_win, s_w + o8 * 4, cc, y, acc);
        }
    }
    // epilogue through shared memory: tile[w][offset inside the window's contiguous output block]
    __syncthreads();
    float *tile = smr;
    if (act) {
#pragma unroll
        for (int oo = 0; oo < 8; ++oo) {
            const int ol = (oo >> 2) * 32 + o8 * 4 + (oo & 3), o = ob + ol;
            float sc = 1.f, sh = 0.f, al = 0.f;
            if (OP == OP_BN_PRELU || OP == OP_BN_RES) { sc = ep.scale[o]; sh = ep.shift[o]; }
            if (OP == OP_PRELU || OP == OP_BN_PRELU) al = ep.alpha[o];
            if (OP == OP_SHUF_PRELU) al = ep.alpha[o >> 2];
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                const int x = x0 + i;
                float v = acc[i][oo];
                int off;
                if (OP == OP_SHUF_PRELU) {
                    v = v > 0.f ? v : al * v;
                    off = (ol >> 2) * 4 * HW + (2 * y + ((ol >> 1) & 1)) * 2 * H + 2 * x + (ol & 1);
                } else {
                    if (OP != OP_PRELU) v = fmaf(v, sc, sh);
                    if (OP != OP_BN_RES) v = v > 0.f ? v : al * v;
                    off = ol * HW + y * H + x;
                }
                tile[wl * 64 * HW + off] = v;
            }
        }
    }
    {
        // non-shuffle: channels ob .. ob + 63 of (N, O, H, H); shuffle: planes ob/4 .. ob/4 + 15 of (N, O/4, 2H, 2H):
        // either way the window's block starts at (n O + ob) H H.  The residual is requested before the barrier.
        constexpr int per = 16 * HW, NP = NW * per / kRowThreads;   // 16-byte pieces per window block / per thread
        static_assert(NW * per % kRowThreads == 0, "whole pieces per thread");
        float4 r[OP == OP_BN_RES ? NP : 1];
        if (OP == OP_BN_RES) {
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                const int idx = tid + j * kRowThreads, wi = idx / per, k = idx - wi * per, n = n0 + wi;
                if (n < N) r[j] = *(reinterpret_cast<const float4 *>(ep.res + (int64_t(n) * O + ob) * HW) + k);
            }
        }
        __syncthreads();
        const float4 *t4 = reinterpret_cast<const float4 *>(tile);
#pragma unroll
        for (int j = 0; j < NP; ++j) {
            const int idx = tid + j * kRowThreads, wi = idx / per, k = idx - wi * per, n = n0 + wi;
            if (n >= N) break;
            float4 t = t4[idx];
            if (OP == OP_BN_RES) {
                t.x = r[j].x + t.x;
                t.y = r[j].y + t.y;
                t.z = r[j].z + t.z;
                t.w = r[j].w + t.w;
            }
            *(reinterpret_cast<float4 *>(out + (int64_t(n) * O + ob) * HW) + k) = t;
        }
    }
}

// The 9x9 64 -> 3 tail on 12- or 24-wide images: thread = one 12-pixel row segment x the 3 outputs
// (36 accumulators); per input channel and kernel row 12 or 16 staged inputs (raw planes, replicate
// padding resolved by the compile-time column map) and 9 x 4 weights ([c][tap][4], one broadcast float4
// per tap) for 324 FMAs.  Same accumulation order and epilogue expression as the other forms.
constexpr int kTailCC = 2;

template <int H, int SEG>
__device__ __forceinline__ void tail_chunk(const float *s_win, const float4 *sw, int cc, int y, float (&acc)[12][3]) {
    constexpr int K = 9, P = 4, HW = H * H;
    constexpr int BASE = H == 12 ? 0 : 8 * SEG, L = H == 12 ? 12 : 16;
    for (int c = 0; c < cc; ++c) {
        const float *si = s_win + c * HW;
#pragma unroll 3
        for (int dy = 0; dy < K; ++dy) {
            float b[L], v[20];
            const int yo = min(max(y + dy - P, 0), H - 1) * H;
#pragma unroll
            for (int j = 0; j < L / 4; ++j) {
                const float4 t = *reinterpret_cast<const float4 *>(si + yo + BASE + 4 * j);
                b[4 * j] = t.x;
                b[4 * j + 1] = t.y;
                b[4 * j + 2] = t.z;
                b[4 * j + 3] = t.w;
            }
#pragma unroll
            for (int j = 0; j < 20; ++j) {
                int col = 12 * SEG + j - P;
                col = col < 0 ? 0 : (col > H - 1 ? H - 1 : col);
                v[j] = b[col - BASE];
            }
#pragma unroll
            for (int dx = 0; dx < K; ++dx) {
                const float4 w4 = sw[(c * K + dy) * K + dx];
#if MGSR_TAIL_FFMA2
                // outputs 0 and 1 as a packed pair (weights (w.x, w.y) as loaded, the pixel as the broadcast operand),
                // output 2 scalar
                const unsigned long long w01 = pack2f(w4.x, w4.y);
#pragma unroll
                for (int i = 0; i < 12; ++i) {
                    ffma2(acc[i][0], acc[i][1], pack2f(v[i + dx], v[i + dx]), w01);
                    acc[i][2] = fmaf(v[i + dx], w4.z, acc[i][2]);
                }
#else
#pragma unroll
                for (int i = 0; i < 12; ++i) {
                    acc[i][0] = fmaf(v[i + dx], w4.x, acc[i][0]);
                    acc[i][1] = fmaf(v[i + dx], w4.y, acc[i][1]);
                    acc[i][2] = fmaf(v[i + dx], w4.z, acc[i][2]);
                }
#endif
            }
        }
    }
}

template <int H>
__global__ void __maxnreg__(MGSR_ROW_REGS) k_conv_tail_rows(const float *__restrict__ in, int N, int C,
                                                                   const float *__restrict__ wt,
                                                                   float *__restrict__ out, Epi ep) {
    extern __shared__ __align__(16) float smr[];
    constexpr int KK = 81, HW = H * H, NSEG = H / 12, NW = kRowThreads / (H * NSEG), RPS = NW * H;
    constexpr int STAGE = kTailCC * KK * 4 + NW * kTailCC * HW;   // weights [cc][81][4] + raw planes [NW][cc][H][H]
    const int tid = threadIdx.x;
    const int seg = tid / RPS, r2 = tid - seg * RPS, wl = r2 / H, y = r2 - wl * H, x0 = 12 * seg;
    const int n0 = blockIdx.x * NW;
    const bool act = n0 + wl < N;
    float acc[12][3];
#pragma unroll
    for (int i = 0; i < 12; ++i) acc[i][0] = acc[i][1] = acc[i][2] = 0.f;
    auto stage = [&](int c0, int st) {
        const int cc = min(kTailCC, C - c0);
        float *s_w = smr + st * STAGE, *s_in = s_w + kTailCC * KK * 4;
        const int per = cc * HW / 4;
        for (int idx = tid; idx < NW * per; idx += kRowThreads) {
            const int wi = idx / per, k = idx - wi * per, n = n0 + wi;
            if (n < N) cp_async16(reinterpret_cast<float4 *>(s_in) + idx,
                                  reinterpret_cast<const float4 *>(in + (int64_t(n) * C + c0) * HW) + k);
        }
        for (int idx = tid; idx < cc * KK; idx += kRowThreads)
            cp_async16(reinterpret_cast<float4 *>(s_w) + idx, reinterpret_cast<const float4 *>(wt) + int64_t(c0) * KK + idx);
        cp_async_commit();
    };
    stage(0, 0);
    int st = 0;
    for (int c0 = 0; c0 < C; c0 += kTailCC, st ^= 1) {
        const int cc = min(kTailCC, C - c0);
        cp_async_wait_all();
        __syncthreads();
        if (c0 + kTailCC < C) stage(c0 + kTailCC, st ^ 1);
        if (act) {
            const float *s_w = smr + st * STAGE, *s_win = s_w + kTailCC * KK * 4 + wl * cc * HW;
            const float4 *sw = reinterpret_cast<const float4 *>(s_w);
            if (NSEG == 1 || seg == 0) tail_chunk<H, 0>(s_win, sw, cc, y, acc);
            else tail_chunk<H, NSEG - 1>(s_win, sw, cc, y, acc);
        }
    }
    if (!act) return;
    const int n = n0 + wl;
    const float sc = ep.tanh_s;
#pragma unroll
    for (int o = 0; o < 3; ++o) {
        float4 *dst = reinterpret_cast<float4 *>(out + (int64_t(n) * 3 + o) * HW + y * H + x0);
#pragma unroll
        for (int q = 0; q < 3; ++q)
            dst[q] = make_float4(sc * tanhf((acc[4 * q][o] + ep.bias[o]) / sc), sc * tanhf((acc[4 * q + 1][o] + ep.bias[o]) / sc),
                                 sc * tanhf((acc[4 * q + 2][o] + ep.bias[o]) / sc), sc * tanhf((acc[4 * q + 3][o] + ep.bias[o]) / sc));
    }
}

// Direct form for large images (generator_forward on sides whose per-CTA tiles exceed shared memory):
// one thread per output value, replicate-clamped taps read through the read-only cache, the same
// accumulation order (c ascending, dy, dx, fmaf) and epilogues as k_conv_simt.
template <int K, int OP>
__global__ void __launch_bounds__(256) k_conv_direct(const float *__restrict__ in, int N, int C, int H,
                                                     const float *__restrict__ w, int O, float *__restrict__ out,
                                                     Epi ep) {
    constexpr int P = K / 2;
    const int64_t HW = int64_t(H) * H, total = int64_t(N) * O * HW;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t n = t / (O * HW);
        const int o = int((t / HW) % O);
        const int pix = int(t % HW), y = pix / H, x = pix % H;
        float v = 0.f;
        for (int c = 0; c < C; ++c) {
            const float *ic = in + (n * C + c) * HW;
            const float *wc = w + (int64_t(o) * C + c) * K * K;
            for (int dy = 0; dy < K; ++dy) {
                const int yy = min(max(y + dy - P, 0), H - 1);
                for (int dx = 0; dx < K; ++dx) {
                    const int xx = min(max(x + dx - P, 0), H - 1);
                    v = fmaf(__ldg(ic + yy * H + xx), __ldg(wc + dy * K + dx), v);
                }
            }
        }
        if (OP == OP_PRELU) {
            out[t] = v > 0.f ? v : ep.alpha[o] * v;
        } else if (OP == OP_BN_PRELU) {
            v = fmaf(v, ep.scale[o], ep.shift[o]);
            out[t] = v > 0.f ? v : ep.alpha[o] * v;
        } else if (OP == OP_BN_RES) {
            out[t] = ep.res[t] + fmaf(v, ep.scale[o], ep.shift[o]);
        } else if (OP == OP_SHUF_PRELU) {
            const int cc = o >> 2, i = (o >> 1) & 1, j = o & 1, W2 = 2 * H;
            v = v > 0.f ? v : ep.alpha[cc] * v;
            out[((n * (O >> 2) + cc) * W2 + 2 * y + i) * W2 + 2 * x + j] = v;
        } else {
            const float sc = ep.tanh_s;
            out[t] = sc * tanhf((v + ep.bias[o]) / sc);
        }
    }
}

template <int K, int OP>
static int conv(const float *in, int N, int C, int H, const float *w, const float *wt, int O, float *out,
                const Epi &ep, cudaStream_t st) {
    // MGSR_F32_LEGACY=1 keeps the one-pixel kernels below for every shape (the bitwise cross-check of the tests)
    if (std::getenv("MGSR_F32_LEGACY")) wt = nullptr;
    if constexpr (OP == OP_TAIL) {
        if (wt && K == 9 && O == 3 && (H == 12 || H == 24)) {
            auto go = [&](auto kern, int nw) {
                const size_t smem = 2 * sizeof(float) * (size_t(kTailCC) * 81 * 4 + size_t(nw) * kTailCC * H * H);
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
                kern<<<(N + nw - 1) / nw, kRowThreads, smem, st>>>(in, N, C, wt, out, ep);
            };
            if (H == 12) go(k_conv_tail_rows<12>, kRowThreads / 12);
            else go(k_conv_tail_rows<24>, kRowThreads / 48);
            MGSR_LAUNCH_CHECK();
            return MGSR_OK;
        }
    } else {
        if (wt && O % 64 == 0 && C % RowCfg<K>::CC == 0 && (H == 6 || H == 12)) {
            constexpr int CC = RowCfg<K>::CC;
            auto go = [&](auto kern, int nw) {
                // main loop: two stages of (weights + raw planes of a chunk); epilogue: the 64-channel output blocks
                size_t smem = 2 * sizeof(float) * (size_t(CC) * K * K * 64 + size_t(nw) * CC * H * H);
                const size_t epi = sizeof(float) * size_t(nw) * 64 * H * H;
                if (epi > smem) smem = epi;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
                kern<<<dim3((N + nw - 1) / nw, O / 64), kRowThreads, smem, st>>>(in, N, C, wt, O, out, ep);
            };
            if (H == 6) go(k_conv_rows<K, OP, 6>, kRowThreads / 8 / 6);
            else go(k_conv_rows<K, OP, 12>, kRowThreads / 8 / 24);
            MGSR_LAUNCH_CHECK();
            return MGSR_OK;
        }
    }
    {
        const int HW = H * H, HP = H + K - 1;
        const int nw = HW <= kConv2Threads ? kConv2Threads / HW : 1;
        const int per = (HW + kConv2Threads - 1) / kConv2Threads;
        // output-channel block: 16, or 4 for the 3-channel tail (no FMAs on padding channels)
        const int ob = O >= 16 ? kConv2OB : 4;
        const size_t smem = sizeof(float) * (size_t(kConv2CC) * K * K * ob + size_t(nw) * kConv2CC * HP * HP);
        if (per <= 3 && smem <= 200 * 1024) {
            dim3 grid((N + nw - 1) / nw, (O + ob - 1) / ob);
            auto go = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
                kern<<<grid, kConv2Threads, smem, st>>>(in, N, C, H, w, O, out, ep, nw);
            };
            if (ob == kConv2OB) {
                if (per == 1) go(k_conv_rt<K, 1, OP, kConv2OB>);
                else go(k_conv_rt<K, 3, OP, kConv2OB>);
            } else {
                if (per == 1) go(k_conv_rt<K, 1, OP, 4>);
                else go(k_conv_rt<K, 3, OP, 4>);
            }
            MGSR_LAUNCH_CHECK();
            return MGSR_OK;
        }
    }
    const int HP = H + K - 1;
    int cc = 12288 / (HP * HP);
    if (cc > C) cc = C;
    const size_t smem = sizeof(float) * (cc > 0 ? cc : 1) * HP * HP;
    const int per = (kConvOB * H * H + kConvThreads - 1) / kConvThreads;
    if (cc < 1 || per > 36) {
        k_conv_direct<K, OP><<<grid_for(int64_t(N) * O * H * H, 256), 256, 0, st>>>(in, N, C, H, w, O, out, ep);
        MGSR_LAUNCH_CHECK();
        return MGSR_OK;
    }
    dim3 grid(N, (O + kConvOB - 1) / kConvOB);
    if (per <= 3)
        k_conv_simt<K, 3, OP><<<grid, kConvThreads, smem, st>>>(in, C, H, w, O, out, ep, cc);
    else if (per <= 9)
        k_conv_simt<K, 9, OP><<<grid, kConvThreads, smem, st>>>(in, C, H, w, O, out, ep, cc);
    else
        k_conv_simt<K, 36, OP><<<grid, kConvThreads, smem, st>>>(in, C, H, w, O, out, ep, cc);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

// Per-window scratch floats for a forward at side H (buffers S, Y, Z, U, out).
static size_t gen_scratch_floats(int H) { return size_t(64) * H * H * 3 + size_t(64) * 4 * H * H + 3 * 4 * H * H; }

// Generator forward on N samples (N,3,H,H) fp32 -> (N,3,2H,2H) fp32 (srmodel.py:330-344).
static int gen_forward_f32(const mgsr_gen *g, const float *x, int N, int H, float *y, float *scratch,
                           cudaStream_t st) {
    const size_t t64 = size_t(N) * 64 * H * H;
    float *S = scratch, *Y = S + t64, *Z = Y + t64, *U = Z + t64;
    Epi ep{};
    int r;
    ep.alpha = g->head_a;
    if ((r = conv<9, OP_PRELU>(x, N, 3, H, g->head_w, g->head_t, 64, S, ep, st))) return r;
    MGSR_CUDA_TRY(cudaMemcpyAsync(Y, S, sizeof(float) * t64, cudaMemcpyDeviceToDevice, st));
    for (int b = 0; b < g->blocks; ++b) {
        Epi e1{g->bn1s[b], g->bn1b[b], g->pa[b], nullptr, nullptr, 1.f};
        if ((r = conv<3, OP_BN_PRELU>(Y, N, 64, H, g->c1[b], g->c1_t[b], 64, Z, e1, st))) return r;
        Epi e2{g->bn2s[b], g->bn2b[b], nullptr, nullptr, Y, 1.f};
        if ((r = conv<3, OP_BN_RES>(Z, N, 64, H, g->c2[b], g->c2_t[b], 64, Y, e2, st))) return r;
    }
    Epi ep_post{g->post_s, g->post_b, nullptr, nullptr, S, 1.f};
    if ((r = conv<3, OP_BN_RES>(Y, N, 64, H, g->post_w, g->post_t, 64, Z, ep_post, st))) return r;
    Epi ep_up{nullptr, nullptr, g->up_a, nullptr, nullptr, 1.f};
    if ((r = conv<3, OP_SHUF_PRELU>(Z, N, 64, H, g->up_w, g->up_t, 256, U, ep_up, st))) return r;
    Epi ep_t{nullptr, nullptr, nullptr, g->tail_b, nullptr, float(g->tanh_scale)};
    return conv<9, OP_TAIL>(U, N, 64, 2 * H, g->tail_w, g->tail_t, 3, y, ep_t, st);
}

// ---------------------------------------------------------------------------
// windowed pass glue

// q = clip((log10|v| - log_lo)/span, 0, 1) * sign(v) in fp64 (grid.py:103-109)
__device__ __forceinline__ double normalize_q(double v, double log_lo, double span) {
    if (v == 0.0) return 0.0;
    double t = (log10(fabs(v)) - log_lo) / span;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    return v > 0.0 ? t : -t;
}

__device__ __forceinline__ double denormalize_q(double q, double log_lo, double span) {
    if (q == 0.0) return 0.0;   // sign 0 annihilates (grid.py:112-114)
    double m = pow(10.0, log_lo + fabs(q) * span);
    return q > 0.0 ? m : -m;
}

// windows [k0, k0+cnt) of the plan (srmodel.py:423-440) -> X (cnt, 3, 6, 6) fp32
__global__ void k_sr_gather(const double *__restrict__ c, const double *shift, int nc, int npos, int64_t k0,
                            int cnt, double log_lo, double span, float *__restrict__ X) {
    const double sh = shift ? *shift : 0.0;
    const int64_t total = int64_t(cnt) * 36;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int64_t kw = t / 36;
        int pix = int(t - kw * 36), y = pix / 6, x = pix % 6;
        int64_t k = k0 + kw;
        int iw = 2 * int(k / npos), jw = 2 * int(k % npos);
        float q = float(normalize_q(c[int64_t(iw + y) * nc + jw + x] - sh, log_lo, span));
        X[(kw * 3 + 0) * 36 + pix] = q;
        X[(kw * 3 + 1) * 36 + pix] = q;
        X[(kw * 3 + 2) * 36 + pix] = q;
    }
}

// general gather for a pass whose input is a (nc, nc) grid and windows 6x6
// (also used for the 12x12 second application input? no: that is the
// generator's own output, fed directly).  Stitch: channel mean, keep band,
// denormalise.  Yout (cnt, 3, 6*sc, 6*sc).
__global__ void k_sr_stitch(const float *__restrict__ Y, int npos, int64_t k0, int cnt, int sc, int nc,
                            double log_lo, double span, double *__restrict__ fine) {
    const int side = 6 * sc;
    const int64_t per = int64_t(side) * side;
    const int64_t total = int64_t(cnt) * per;
    const int nf = nc * sc;
    const int last = 2 * (npos - 1);
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total;
         t += int64_t(gridDim.x) * blockDim.x) {
        int64_t kw = t / per;
        int pix = int(t - kw * per), fy = pix / side, fx = pix % side;
        int64_t k = k0 + kw;
        int iw = 2 * int(k / npos), jw = 2 * int(k % npos);
        int lo_i = iw == 0 ? 0 : 2, hi_i = iw == last ? 6 : 4;
        int lo_j = jw == 0 ? 0 : 2, hi_j = jw == last ? 6 : 4;
        if (fy < lo_i * sc || fy >= hi_i * sc || fx < lo_j * sc || fx >= hi_j * sc) continue;
        const float *yw = Y + kw * 3 * per + pix;
        double m = ((double(yw[0]) + double(yw[per])) + double(yw[2 * per])) / 3.0;
        fine[int64_t(iw * sc + fy) * nf + jw * sc + fx] = denormalize_q(m, log_lo, span);
    }
}

__global__ void k_mean_f64(const double *__restrict__ a, int64_t count, RedSlot slot, double *result) {
    double v[1] = {0.0};
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count;
         t += int64_t(gridDim.x) * blockDim.x)
        v[0] += a[t];
    grid_reduce<1>(v, slot, result, 1.0 / double(count));
}

int launch_mean_f64(const double *a, int64_t count, void *red_slot, double *result, cudaStream_t st) {
    k_mean_f64<<<grid_for(count, 256), 256, 0, st>>>(a, count, red_slot_at(red_slot), result);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

__global__ void k_f64_to_f32(const double *__restrict__ a, float *__restrict__ b, int64_t count) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count;
         t += int64_t(gridDim.x) * blockDim.x)
        b[t] = float(a[t]);
}

__global__ void k_f32_to_f64(const float *__restrict__ a, double *__restrict__ b, int64_t count) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < count;
         t += int64_t(gridDim.x) * blockDim.x)
        b[t] = double(a[t]);
}

// windows per fp32 chunk: a multiple of 148 x 8 (one resident 384-thread CTA of the row-tiled kernels per SM,
// 8 windows per CTA at side 6), so a full chunk's launches are whole waves
constexpr int kSrChunk = 3552;

static size_t pass_ws_floats(int apps) {
    // input X (3*36) + generator scratch for the largest application + outputs
    int H = 6, Hmax = 6 * (1 << (apps - 1));
    size_t per = 3 * 36 + gen_scratch_floats(Hmax) + 3 * 4 * Hmax * Hmax + 3 * 4 * H * H * 4;
    return per * kSrChunk;
}

size_t sr_workspace_bytes(int64_t nc, int s, int precision) {
    // intermediate fine grid for two-pass ratios + fp32 chunk buffers + scalars
    size_t inter = (s == 8 || s == 16) ? sizeof(double) * size_t(nc * 4) * size_t(nc * 4) : 0;
    // the fp32 CUDA-core chunk buffers only for the passes that run in fp32 (the tensor-core passes never fall
    // back to them): fp32 everywhere, or MIXED's first pass of a two-pass ratio (two applications)
    const bool simt_pass = !tensor_core_precision(precision) || (precision == MGSR_PREC_MIXED && (s == 8 || s == 16));
    size_t simt = simt_pass ? sizeof(float) * pass_ws_floats(s == 2 ? 1 : 2) + 4096 : 0;
    size_t tc = 0;
    if (tensor_core_precision(precision)) {   // the largest pass of the plan: (ratio, coarse side) per pass
        tc = s == 2 ? tc_workspace_bytes(nc) : tc4_workspace_bytes(nc);
        if (s == 8 && tc_workspace_bytes(4 * nc) > tc) tc = tc_workspace_bytes(4 * nc);
        if (s == 16 && tc4_workspace_bytes(4 * nc) > tc) tc = tc4_workspace_bytes(4 * nc);
    }
    return inter + (simt > tc ? simt : tc) + 512;
}

static const int *pass_plan(int s, int *count) {
    static const int p2[] = {1}, p4[] = {2}, p8[] = {2, 1}, p16[] = {2, 2};
    switch (s) {
        case 2: *count = 1; return p2;
        case 4: *count = 1; return p4;
        case 8: *count = 2; return p8;
        case 16: *count = 2; return p16;
    }
    *count = 0;
    return nullptr;
}

// One windowed pass (srmodel.py:443-463) with `apps` applications, fp32 generator.
static int sr_pass_simt(const mgsr_gen *g, const double *c, const double *c_shift, int nc, int apps,
                        double log_lo, double span, double *fine, float *fws, cudaStream_t st) {
    const int npos = nc / 2 - 2;
    const int64_t nw = int64_t(npos) * npos;
    const int Hmax = 6 * (1 << (apps - 1));
    float *X = fws;
    float *Y1 = X + size_t(kSrChunk) * 3 * 36;                 // (chunk,3,12,12)
    float *Y2 = Y1 + size_t(kSrChunk) * 3 * 144;               // (chunk,3,24,24) if apps == 2
    float *scratch = Y2 + (apps == 2 ? size_t(kSrChunk) * 3 * 576 : 0);
    (void)Hmax;
    for (int64_t k0 = 0; k0 < nw; k0 += kSrChunk) {
        int cnt = int(nw - k0 < kSrChunk ? nw - k0 : kSrChunk);
        k_sr_gather<<<grid_for(int64_t(cnt) * 36, 256), 256, 0, st>>>(c, c_shift, nc, npos, k0, cnt, log_lo, span, X);
        MGSR_LAUNCH_CHECK();
        int r = gen_forward_f32(g, X, cnt, 6, Y1, scratch, st);
        if (r) return r;
        const float *Yout = Y1;
        if (apps == 2) {
            r = gen_forward_f32(g, Y1, cnt, 12, Y2, scratch, st);
            if (r) return r;
            Yout = Y2;
        }
        int sc = 1 << apps;
        k_sr_stitch<<<grid_for(int64_t(cnt) * 36 * sc * sc, 256), 256, 0, st>>>(Yout, npos, k0, cnt, sc, nc, log_lo,
                                                                                span, fine);
        MGSR_LAUNCH_CHECK();
    }
    return MGSR_OK;
}

int launch_sr_prolong(const mgsr_gen *g, const double *c, const double *c_shift, int nc, int s, double p_min,
                      double p_max, int precision, double *out, double *out_mean, void *ws, size_t ws_bytes,
                      void *red_slot, cudaStream_t st, cudaEvent_t *gen_markers) {
    if (!valid_precision(precision)) { set_error("precision must be one of fp32, bf16, fp16, mixed"); return MGSR_E_BAD_ARG; }
    int npass = 0;
    const int *plan = pass_plan(s, &npass);
    if (!plan) { set_error("unsupported SR ratio " + std::to_string(s) + "; expected one of [2, 4, 8, 16]"); return MGSR_E_SR_RATIO; }
    if (nc < 6) { set_error("coarse side must be >= 6, got " + std::to_string(nc)); return MGSR_E_WINDOW; }
    if (nc % 2) { set_error("coarse side must be even, got " + std::to_string(nc)); return MGSR_E_WINDOW; }
    if (ws_bytes < sr_workspace_bytes(nc, s, precision)) { set_error("sr workspace too small"); return MGSR_E_WORKSPACE; }
    const double log_lo = std::log10(p_min), span = std::log10(p_max) - std::log10(p_min);
    char *w = static_cast<char *>(ws);
    double *scal = reinterpret_cast<double *>(w);     // [0] intermediate mean
    w += 512;
    double *inter = nullptr;
    if (npass == 2) {
        inter = reinterpret_cast<double *>(w);
        w += sizeof(double) * size_t(nc * 4) * size_t(nc * 4);
    }
    RedSlot sl = red_slot_at(red_slot);
    const double *src = c;
    const double *src_shift = c_shift;
    int n_in = nc;
    for (int ip = 0; ip < npass; ++ip) {
        const int apps = plan[ip];
        double *dst = (ip == npass - 1) ? out : inter;
        int r;
        const bool mark = gen_markers && ip == npass - 1;
        if (mark) MGSR_CUDA_TRY(cudaEventRecordWithFlags(gen_markers[0], st, cudaEventRecordExternal));
        const int pprec = pass_precision(precision, ip, npass);
        if (tensor_core_precision(pprec)) {
            // tensor-core path only; no silent fallback to the fp32 CUDA-core path
            if (!g->tc_blob) { set_error("tensor-core weights not packed"); return MGSR_E_UNSUPPORTED; }
            const size_t left = ws_bytes - size_t(w - static_cast<char *>(ws));
            r = apps == 1 ? launch_sr_pass_tc(g, src, src_shift, n_in, log_lo, span, dst, w, left, st,
                                              pprec != MGSR_PREC_BF16)
                          : launch_sr_pass4_tc(g, src, src_shift, n_in, log_lo, span, dst, w, left, st,
                                               pprec != MGSR_PREC_BF16);
        } else {
            r = sr_pass_simt(g, src, src_shift, n_in, apps, log_lo, span, dst, reinterpret_cast<float *>(w), st);
        }
        if (r) return r;
        if (mark) MGSR_CUDA_TRY(cudaEventRecordWithFlags(gen_markers[1], st, cudaEventRecordExternal));
        const int n_out = n_in << apps;
        double *mean_dst = (ip == npass - 1) ? out_mean : scal;
        k_mean_f64<<<grid_for(int64_t(n_out) * n_out, 256), 256, 0, st>>>(dst, int64_t(n_out) * n_out, sl, mean_dst);
        MGSR_LAUNCH_CHECK();
        src = dst;
        src_shift = scal;
        n_in = n_out;
    }
    return MGSR_OK;
}

}  // namespace mgsr

// ---------------------------------------------------------------------------
// C ABI (generator part)

using namespace mgsr;

namespace {

int upload(mgsr_gen *g, const float *host, size_t count, float **dst) {
    float *d = nullptr;
    MGSR_CUDA_TRY(cudaMalloc(&d, sizeof(float) * count));
    MGSR_CUDA_TRY(cudaMemcpy(d, host, sizeof(float) * count, cudaMemcpyHostToDevice));
    g->allocations.push_back(d);
    *dst = d;
    return MGSR_OK;
}

// OIHW weights -> [C][taps][Opad] for the row-tiled kernels (zero-filled pad channels)
int upload_transposed(mgsr_gen *g, const float *host, int O, int C, int KK, int Opad, float **dst) {
    std::vector<float> t(size_t(C) * KK * Opad, 0.f);
    for (int o = 0; o < O; ++o)
        for (int c = 0; c < C; ++c)
            for (int k = 0; k < KK; ++k) t[(size_t(c) * KK + k) * Opad + o] = host[(size_t(o) * C + c) * KK + k];
    return upload(g, t.data(), t.size(), dst);
}

// BN(x) = gamma (x - mean)/sqrt(var + 1e-5) + beta  ->  x*scale + shift (srmodel.py:313-318)
int upload_bn(mgsr_gen *g, const float *gamma, const float *beta, const float *mean, const float *var, float **s,
              float **b) {
    std::vector<float> sc(64), sh(64);
    for (int i = 0; i < 64; ++i) {
        double k = double(gamma[i]) / std::sqrt(double(var[i]) + 1e-5);
        sc[i] = float(k);
        sh[i] = float(double(beta[i]) - double(mean[i]) * k);
    }
    if (int r = upload(g, sc.data(), 64, s)) return r;
    return upload(g, sh.data(), 64, b);
}

}  // namespace

extern "C" int mgsr_generator_create(const float *const *t, int32_t num_tensors, int32_t blocks, double tanh_scale,
                                     mgsr_gen **out) {
    if (blocks < 1 || num_tensors != 2 + 11 * blocks + 5 + 2 + 2) {
        set_error("missing tensors: tensor count does not match expected_tensor_shapes(" + std::to_string(blocks) + ")");
        return MGSR_E_BAD_ARG;
    }
    if (!(tanh_scale >= 1.0)) { set_error("tanh scale must be >= 1"); return MGSR_E_BAD_ARG; }
    mgsr_gen *g = new mgsr_gen();
    g->blocks = blocks;
    g->tanh_scale = tanh_scale;
    int i = 0, r = 0;
#define UP(cnt, dst) if ((r = upload(g, t[i++], (cnt), (dst)))) goto fail;
    if ((r = upload_transposed(g, t[i], 64, 3, 81, 64, &g->head_t))) goto fail;
    UP(64 * 3 * 81, &g->head_w);
    UP(64, &g->head_a);
    g->c1.resize(blocks); g->c2.resize(blocks); g->bn1s.resize(blocks); g->bn1b.resize(blocks);
    g->bn2s.resize(blocks); g->bn2b.resize(blocks); g->pa.resize(blocks);
    g->c1_t.resize(blocks); g->c2_t.resize(blocks);
    for (int b = 0; b < blocks; ++b) {
        if ((r = upload_transposed(g, t[i], 64, 64, 9, 64, &g->c1_t[b]))) goto fail;
        UP(64 * 64 * 9, &g->c1[b]);
        if ((r = upload_bn(g, t[i], t[i + 1], t[i + 2], t[i + 3], &g->bn1s[b], &g->bn1b[b]))) goto fail;
        i += 4;
        UP(64, &g->pa[b]);
        if ((r = upload_transposed(g, t[i], 64, 64, 9, 64, &g->c2_t[b]))) goto fail;
        UP(64 * 64 * 9, &g->c2[b]);
        if ((r = upload_bn(g, t[i], t[i + 1], t[i + 2], t[i + 3], &g->bn2s[b], &g->bn2b[b]))) goto fail;
        i += 4;
    }
    if ((r = upload_transposed(g, t[i], 64, 64, 9, 64, &g->post_t))) goto fail;
    UP(64 * 64 * 9, &g->post_w);
    if ((r = upload_bn(g, t[i], t[i + 1], t[i + 2], t[i + 3], &g->post_s, &g->post_b))) goto fail;
    i += 4;
    if ((r = upload_transposed(g, t[i], 256, 64, 9, 256, &g->up_t))) goto fail;
    UP(256 * 64 * 9, &g->up_w);
    UP(64, &g->up_a);
    if ((r = upload_transposed(g, t[i], 3, 64, 81, 4, &g->tail_t))) goto fail;
    UP(3 * 64 * 81, &g->tail_w);
    UP(3, &g->tail_b);
#undef UP
    if ((r = tc_pack_weights(g, t))) goto fail;
    *out = g;
    return MGSR_OK;
fail:
    mgsr_generator_destroy(g);
    return r;
}

extern "C" int mgsr_generator_destroy(mgsr_gen *g) {
    if (!g) return MGSR_OK;
    for (void *p : g->allocations) cudaFree(p);
    if (g->tc_blob) cudaFree(g->tc_blob);
    delete g;
    return MGSR_OK;
}

extern "C" int mgsr_generator_forward(const mgsr_gen *g, const double *x, int64_t batch, int64_t side, double *y,
                                      void *stream) {
    if (!g || !x || !y || batch < 1 || side < 1) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int H = int(side);
    size_t nx = size_t(batch) * 3 * H * H, ny = size_t(batch) * 3 * 4 * H * H;
    size_t bytes = sizeof(float) * (nx + ny + gen_scratch_floats(H) * size_t(batch));
    float *buf = nullptr;
    if (int e = scratch_alloc(reinterpret_cast<void **>(&buf), bytes, st)) return e;
    k_f64_to_f32<<<grid_for(nx, 256), 256, 0, st>>>(x, buf, nx);
    int r = gen_forward_f32(g, buf, int(batch), H, buf + nx, buf + nx + ny, st);
    if (!r) k_f32_to_f64<<<grid_for(ny, 256), 256, 0, st>>>(buf + nx, y, ny);
    cudaFreeAsync(buf, st);
    if (!r) MGSR_LAUNCH_CHECK();
    return r;
}

extern "C" size_t mgsr_sr_workspace_bytes(int64_t nc, int32_t s) {
    const size_t a = sr_workspace_bytes(nc, s, MGSR_PREC_FP32), b = sr_workspace_bytes(nc, s, MGSR_PREC_BF16);
    return (a > b ? a : b) + kRedSlotBytes + 256;
}

extern "C" int mgsr_sr_prolong(const mgsr_gen *g, const double *c, int64_t nc, int32_t s, double p_min,
                               double p_max, int32_t precision, double *out, void *ws, size_t ws_bytes,
                               void *stream) {
    if (!g || !c || !out) { set_error("SR prolongation requires generator weights"); return MGSR_E_BAD_ARG; }
    if (!valid_precision(precision)) { set_error("precision must be one of fp32, bf16, fp16, mixed"); return MGSR_E_BAD_ARG; }
    if (ws_bytes < mgsr_sr_workspace_bytes(nc, s)) { set_error("workspace too small"); return MGSR_E_WORKSPACE; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char *w = static_cast<char *>(ws);
    double *mean = reinterpret_cast<double *>(w);
    void *red = w + 256;
    MGSR_CUDA_TRY(cudaMemsetAsync(red, 0, sizeof(unsigned), st));   // the slot's ticket starts at zero
    w += 256 + kRedSlotBytes;
    int r = launch_sr_prolong(g, c, nullptr, int(nc), s, p_min, p_max, precision, out, mean, w,
                              ws_bytes - 256 - kRedSlotBytes, red, st);
    if (r) return r;
    return launch_affine(out, out, int64_t(nc) * s * nc * s, mean, 1.0, st);
}
