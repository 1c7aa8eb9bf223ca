// Tensor-core (tcgen05/TMEM) generator megakernel for ratio-2 SR passes.
//
// Reference semantics: srmodel.py:285-344 (generator), 414-463 (windowed
// pass), grid.py:103-114 (log normalisation).  One persistent CTA per SM
// walks groups of 6 windows; all 20 layers of a window group stay on chip:
//
//   * activations: bf16 in shared memory, each 6x6 window stored as an 8x8
//     replicate-padded tile (64 rows) so that every 3x3 tap of a same-size
//     replicate-padded correlation is the SAME matrix shifted by a constant
//     row offset: the UMMA A-descriptor start address moves by 16 B per row
//     (K-major, no swizzle), no im2col.  Two windows = one 128-row M tile,
//     three tiles per group.
//   * accumulators and the fp32 residual stream live in TMEM (512 columns:
//     per tile 64 accumulator + 64 residual columns; the 256-wide
//     up-convolution runs as two N=128 halves in the same 128 columns).
//   * weights (bf16, pre-packed in the UMMA core-matrix layout) stream from
//     L2 through a 3-stage ring with cp.async.bulk + mbarrier complete_tx.
//   * head 9x9 conv: tf32 MMA (K = 81 taps, the 3 identical input channels
//     folded) on an im2col built per tile; PReLU in the epilogue.
//   * body: 2B+1 3x3 convs (bf16 x bf16 -> fp32) with BN folded into a
//     per-channel affine, PReLU / residual add / global skip fused into the
//     epilogue (TMEM -> registers -> smem).
//   * up conv 64->256 + pixel shuffle + PReLU fused into the epilogue, which
//     writes the 12x12 shuffled field (fp32) for the tail.
//   * tail 9x9 conv 64->3 + bias + s*tanh(x/s) + channel mean + denormalise,
//     evaluated in fp32 on CUDA cores ONLY at the stitched (kept) pixels, and
//     written straight into the fine fp64 grid.
//
// Warp roles: warp 0 = weight producer (1 lane), warp 1 = MMA issuer (1 lane,
// also TMEM allocator), warps 2..9 = epilogue (256 threads; warp w reads TMEM
// lane quadrant w%4, column half (w-2)/4).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "generator.cuh"
#include "stencil.cuh"

namespace mgsr {
namespace tc {

constexpr int T = 3;                 // M tiles per group
constexpr int WPT = 2;               // windows per tile
constexpr int WPG = T * WPT;         // windows per group
constexpr int ROWS = 128;            // rows per tile (2 x 8x8 padded windows)
constexpr int GUARD = 16;            // guard rows around the act planes (tap shifts are within +-9)
constexpr int PLANE_ROWS = GUARD + T * ROWS + GUARD;
constexpr int ACT_PLANE = PLANE_ROWS * 16;            // bytes per 8-channel plane
constexpr int ACT_BYTES = 8 * ACT_PLANE;              // 53248
constexpr int SKIP_TILE = 8 * ROWS * 16;              // 16384
constexpr int SKIP_BYTES = T * SKIP_TILE;             // 49152
constexpr int STAGES = 3;
constexpr int STAGE_BYTES = 16384;
constexpr int RING_BYTES = STAGES * STAGE_BYTES;      // 49152
constexpr int UNION_BYTES = 69632;
constexpr int MISC_BYTES = 2048;                      // q table (3 tiles x 72 floats) etc.
constexpr int BAR_BYTES = 256;
constexpr int OFF_ACT = 0;
constexpr int OFF_SKIP = OFF_ACT + ACT_BYTES;
constexpr int OFF_RING = OFF_SKIP + SKIP_BYTES;
constexpr int OFF_UNION = OFF_RING + RING_BYTES;
constexpr int OFF_MISC = OFF_UNION + UNION_BYTES;
constexpr int OFF_BAR = OFF_MISC + MISC_BYTES;
constexpr int SMEM_BYTES = OFF_BAR + BAR_BYTES + 1024;   // +1024 alignment slack
// union sub-layout
constexpr int U_PIX = 33;                                // floats per pixel (32 channels + 1 pad)
constexpr int U_BYTES = WPT * 144 * U_PIX * 4;           // 38016
constexpr int TW_OFF = U_BYTES;                          // tail weights [dy][dx][o][32]
constexpr int TW_BYTES = 81 * 3 * 32 * 4;                // 31104
constexpr int HK = 88;                                   // head K (81 taps padded to tf32 K multiple)
constexpr int HPLANES = HK / 4;                          // 22 planes of 4 tf32
constexpr int I2C_BYTES = HPLANES * ROWS * 16;           // 45056
constexpr int HB_OFF = I2C_BYTES;
constexpr int HB_BYTES = HPLANES * 64 * 16;              // 22528
static_assert(U_BYTES + TW_BYTES <= UNION_BYTES, "union");
static_assert(HB_OFF + HB_BYTES <= UNION_BYTES, "union");
static_assert(SMEM_BYTES <= 232448, "smem");

constexpr int NTHREADS = 320;
constexpr int BODY_TAP_BYTES = 8192;   // 64 oc x 64 ic bf16
constexpr int UP_TAP_BYTES = 16384;    // 128 oc x 64 ic bf16

// blob layout (bytes); body layer count NL = 2B + 1
struct BlobLayout {
    size_t head_b, body, up, tail, consts, total;
    int nl;
};

__host__ __device__ inline BlobLayout blob_layout(int blocks) {
    BlobLayout L;
    L.nl = 2 * blocks + 1;
    L.head_b = 0;
    L.body = L.head_b + HB_BYTES;
    L.up = L.body + size_t(L.nl) * 9 * BODY_TAP_BYTES;
    L.tail = L.up + 2 * 9 * UP_TAP_BYTES;
    L.consts = L.tail + 2 * TW_BYTES;
    L.total = L.consts + sizeof(float) * (64 + 192 * L.nl + 64 + 4);
    return L;
}
// consts (floats): [0,64) head alpha; layer L: 64 + 192 L + {0: scale, 64: shift, 128: alpha};
// up alpha at 64 + 192 NL; tail bias (3) after that.

// ---------------------------------------------------------------------------
// PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFFu);
    d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
    d |= uint64_t(1) << 46;   // descriptor version 1 (sm_100); base offset 0; SWIZZLE_NONE
    return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

#define TMEM_LD32(taddr, v)                                                                                   \
    asm volatile(                                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"      \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                            \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),     \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),            \
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),          \
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),          \
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                                                               \
        : "r"(taddr))

#define TMEM_ST32(taddr, v)                                                                                   \
    asm volatile(                                                                                             \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"   \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                 \
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),    \
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),        \
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),       \
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])                    \
        : "memory")

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// instruction descriptors: D fp32, K-major A and B, M = 128
__host__ __device__ constexpr uint32_t idesc_bf16(int n) { return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24); }
__host__ __device__ constexpr uint32_t idesc_tf32(int n) { return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24); }

struct Params {
    const double *c;
    const double *c_shift;
    int nc, npos;
    long long nwin;
    int ngroups;
    double log_lo, span;
    double *fine;
    int nf;
    const uint8_t *blob;
    int nl;
    float tanh_s;
    float *dbg;
    int dbg_layer;
};

// window geometry of a global window index
struct Win {
    int iw, jw, lo_i, hi_i, lo_j, hi_j;
    bool valid;
};
__device__ __forceinline__ Win window_of(const Params &P, long long k) {
    Win w;
    w.valid = k < P.nwin;
    long long kk = w.valid ? k : P.nwin - 1;
    w.iw = 2 * int(kk / P.npos);
    w.jw = 2 * int(kk % P.npos);
    const int last = 2 * (P.npos - 1);
    w.lo_i = w.iw == 0 ? 0 : 2;
    w.hi_i = w.iw == last ? 6 : 4;
    w.lo_j = w.jw == 0 ? 0 : 2;
    w.hi_j = w.jw == last ? 6 : 4;
    return w;
}

__device__ __forceinline__ double normalize_q(double v, double log_lo, double span) {
    if (v == 0.0) return 0.0;
    double t = (log10(fabs(v)) - log_lo) / span;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    return v > 0.0 ? t : -t;
}

// Write one row's 32 channels (bf16) of tile t into the act planes at row `row`
// plus its replicate-padding images.  kc0 = first 8-channel plane (4 planes).
__device__ __forceinline__ void store_act_row(uint8_t *act, int t, int row, int kc0, const uint32_t (&pk)[16]) {
    const int w = row >> 6, pix = row & 63, py = pix >> 3, px = pix & 7;
    if (py < 1 || py > 6 || px < 1 || px > 6) return;   // border rows hold replicas written by interior rows
    int ty[2] = {py, py == 1 ? 0 : (py == 6 ? 7 : -1)};
    int tx[2] = {px, px == 1 ? 0 : (px == 6 ? 7 : -1)};
#pragma unroll
    for (int a = 0; a < 2; ++a) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            if (ty[a] < 0 || tx[b] < 0) continue;
            const int r = GUARD + t * ROWS + w * 64 + ty[a] * 8 + tx[b];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint4 v = make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
                *reinterpret_cast<uint4 *>(act + (kc0 + k) * ACT_PLANE + r * 16) = v;
            }
        }
    }
}

__global__ void __launch_bounds__(NTHREADS, 1) k_gen_tc(Params P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *act = smem + OFF_ACT;
    uint8_t *skip = smem + OFF_SKIP;
    uint8_t *ring = smem + OFF_RING;
    uint8_t *uni = smem + OFF_UNION;
    float *misc = reinterpret_cast<float *>(smem + OFF_MISC);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + OFF_BAR + 200);
    const uint32_t b_full = smem_u32(bars + 0);      // [STAGES]
    const uint32_t b_empty = smem_u32(bars + 3);     // [STAGES]
    const uint32_t b_i2c_full = smem_u32(bars + 6);
    const uint32_t b_i2c_empty = smem_u32(bars + 7);
    const uint32_t b_acc_full = smem_u32(bars + 8);  // [T]
    const uint32_t b_act_ready = smem_u32(bars + 11);  // [T]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const BlobLayout BL = blob_layout((P.nl - 1) / 2);
    const float *consts = reinterpret_cast<const float *>(P.blob + BL.consts);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(b_full + 8 * s, 1);
            mbar_init(b_empty + 8 * s, 1);
        }
        mbar_init(b_i2c_full, 1);
        mbar_init(b_i2c_empty, 1);
        for (int t = 0; t < T; ++t) {
            mbar_init(b_acc_full + 8 * t, 1);
            mbar_init(b_act_ready + 8 * t, 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ================= weight producer =================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int g = blockIdx.x; g < P.ngroups; g += gridDim.x) {
                for (int L = 0; L < P.nl + 2; ++L) {
                    const bool up = L >= P.nl;
                    const uint32_t bytes = up ? UP_TAP_BYTES : BODY_TAP_BYTES;
                    const uint8_t *src = up ? P.blob + BL.up + size_t(L - P.nl) * 9 * UP_TAP_BYTES
                                            : P.blob + BL.body + size_t(L) * 9 * BODY_TAP_BYTES;
                    for (int tap = 0; tap < 9; ++tap) {
                        mbar_wait(b_empty + 8 * stage, phase ^ 1);
                        mbar_expect_tx(b_full + 8 * stage, bytes);
                        bulk_g2s(smem_u32(ring + stage * STAGE_BYTES), src + size_t(tap) * bytes, bytes,
                                 b_full + 8 * stage);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0, i2c_ph = 0;
            uint32_t ar_ph[T] = {0, 0, 0};
            const uint32_t act_base = smem_u32(act);
            const uint32_t ring_base = smem_u32(ring);
            const uint32_t i2c_base = smem_u32(uni);
            const uint32_t hb_base = smem_u32(uni + HB_OFF);
            for (int g = blockIdx.x; g < P.ngroups; g += gridDim.x) {
                // head: D[t] = im2col(q) (128 x 88, tf32) x Wh^T (88 x 64)
                for (int t = 0; t < T; ++t) {
                    mbar_wait(b_act_ready + 8 * t, ar_ph[t]);
                    ar_ph[t] ^= 1;
                    mbar_wait(b_i2c_full, i2c_ph);
                    i2c_ph ^= 1;
                    tc_fence_after();
                    const uint32_t d = tmem + 128 * t;
                    for (int ks = 0; ks < HK / 8; ++ks) {
                        uint64_t a = make_desc(i2c_base + 2 * ks * (ROWS * 16), ROWS * 16, 128);
                        uint64_t b = make_desc(hb_base + 2 * ks * (64 * 16), 64 * 16, 128);
                        mma_tf32(d, a, b, idesc_tf32(64), ks > 0);
                    }
                    umma_commit(b_acc_full + 8 * t);
                    umma_commit(b_i2c_empty);
                }
                // body + post (N = 64) and the two up-conv halves (N = 128)
                for (int L = 0; L < P.nl + 2; ++L) {
                    const bool up = L >= P.nl;
                    const uint32_t idesc = up ? idesc_bf16(128) : idesc_bf16(64);
                    const uint32_t bplane = up ? 128 * 16 : 64 * 16;
                    for (int tap = 0; tap < 9; ++tap) {
                        mbar_wait(b_full + 8 * stage, phase);
                        tc_fence_after();
                        const int shift = (tap / 3 - 1) * 8 + (tap % 3 - 1);
                        const uint32_t bbase = ring_base + stage * STAGE_BYTES;
                        for (int t = 0; t < T; ++t) {
                            if (tap == 0) {
                                mbar_wait(b_act_ready + 8 * t, ar_ph[t]);
                                ar_ph[t] ^= 1;
                                tc_fence_after();
                            }
                            const uint32_t d = tmem + 128 * t;
                            const uint32_t arow = act_base + uint32_t(GUARD + t * ROWS + shift) * 16;
#pragma unroll
                            for (int ks = 0; ks < 4; ++ks) {
                                uint64_t a = make_desc(arow + 2 * ks * ACT_PLANE, ACT_PLANE, 128);
                                uint64_t b = make_desc(bbase + 2 * ks * bplane, bplane, 128);
                                mma_bf16(d, a, b, idesc, (tap | ks) > 0);
                            }
                            if (tap == 8) umma_commit(b_acc_full + 8 * t);
                        }
                        umma_commit(b_empty + 8 * stage);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else {
        // ================= epilogue (warps 2..9) =================
        const int ew = warp - 2;               // 0..7
        const int q = warp & 3;                // TMEM lane quadrant
        const int hh = ew >> 2;                // column half
        const int et = threadIdx.x - 64;       // 0..255
        const int row = 32 * q + lane;         // row within a tile
        const int wt = row >> 6, pix = row & 63, py = pix >> 3, px = pix & 7;
        const bool interior = py >= 1 && py <= 6 && px >= 1 && px <= 6;
        const uint32_t lane_addr = uint32_t(32 * q) << 16;
        uint32_t af_ph[T] = {0, 0, 0};
        uint32_t i2c_empty_ph = 0;
        bool first_build = true;
        // pre-arrive: every accumulator starts free
        if (lane == 0)
            for (int t = 0; t < T; ++t) mbar_arrive(b_act_ready + 8 * t);
        const float *head_a = consts;
        const float *up_a = consts + 64 + 192 * P.nl;
        const float *tail_b = up_a + 64;
        for (int g = blockIdx.x; g < P.ngroups; g += gridDim.x) {
            const long long k0 = (long long)g * WPG;
            // ---- q tables of the 6 windows (fp64 normalise -> fp32) ----
            for (int i = et; i < WPG * 36; i += 256) {
                const int wk = i / 36, pp = i % 36;
                Win W = window_of(P, k0 + wk);
                const double sh = P.c_shift ? *P.c_shift : 0.0;
                double v = P.c[(long long)(W.iw + pp / 6) * P.nc + W.jw + pp % 6] - sh;
                misc[i] = float(normalize_q(v, P.log_lo, P.span));
            }
            epi_bar();
            // ---- head: im2col per tile (tf32) + head weights, MMA, PReLU epilogue ----
            for (int t = 0; t < T; ++t) {
                if (!first_build) {
                    mbar_wait(b_i2c_empty, i2c_empty_ph);
                    i2c_empty_ph ^= 1;
                }
                if (first_build || t == 0) {
                    // head weights (tf32, UMMA layout) into the union
                    const uint4 *src = reinterpret_cast<const uint4 *>(P.blob + BL.head_b);
                    uint4 *dst = reinterpret_cast<uint4 *>(uni + HB_OFF);
                    for (int i = et; i < HB_BYTES / 16; i += 256) dst[i] = src[i];
                }
                first_build = false;
                {
                    // row `r` of tile t: 2 threads per row split the 22 planes
                    const int r = et & 127, part = et >> 7;
                    const int rw = r >> 6, rp = r & 63;
                    const int cy = min(max((rp >> 3) - 1, 0), 5), cx = min(max((rp & 7) - 1, 0), 5);
                    const float *qt = misc + (t * WPT + rw) * 36;
                    for (int kc = part * 11; kc < part * 11 + 11; ++kc) {
                        float v[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int k = 4 * kc + e;
                            if (k < 81) {
                                const int dy = k / 9, dx = k % 9;
                                const int y = min(max(cy + dy - 4, 0), 5), x = min(max(cx + dx - 4, 0), 5);
                                v[e] = to_tf32(qt[y * 6 + x]);
                            } else {
                                v[e] = 0.f;
                            }
                        }
                        *reinterpret_cast<float4 *>(uni + kc * (ROWS * 16) + r * 16) = make_float4(v[0], v[1], v[2], v[3]);
                    }
                }
                fence_async_smem();
                epi_bar();
                if (et == 0) mbar_arrive(b_i2c_full);
            }
            // ---- per-layer epilogues ----
            for (int L = -1; L < P.nl; ++L) {
                for (int t = 0; t < T; ++t) {
                    mbar_wait(b_acc_full + 8 * t, af_ph[t]);
                    af_ph[t] ^= 1;
                    tc_fence_after();
                    uint32_t v[32];
                    TMEM_LD32(tmem + lane_addr + 128 * t + 32 * hh, v);
                    tmem_wait_ld();
                    float y[32];
                    const int cb = 32 * hh;
                    if (L < 0) {
                        // head: PReLU, residual stream := y, skip := y
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            float x = __uint_as_float(v[j]);
                            y[j] = x > 0.f ? x : __ldg(head_a + cb + j) * x;
                        }
                        uint32_t st[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) st[j] = __float_as_uint(y[j]);
                        TMEM_ST32(tmem + lane_addr + 128 * t + 64 + cb, st);
                        tmem_wait_st();
                        uint32_t pk[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(y[2 * j], y[2 * j + 1]);
                        if (interior) {
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                *reinterpret_cast<uint4 *>(skip + t * SKIP_TILE + (4 * hh + k) * (ROWS * 16) + row * 16) =
                                    make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
                        }
                        store_act_row(act, t, row, 4 * hh, pk);
                    } else {
                        const float *sc = consts + 64 + 192 * L;
                        const bool conv1 = (L < P.nl - 1) && !(L & 1);
                        const bool post = L == P.nl - 1;
                        if (conv1) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                float x = fmaf(__uint_as_float(v[j]), __ldg(sc + cb + j), __ldg(sc + 64 + cb + j));
                                y[j] = x > 0.f ? x : __ldg(sc + 128 + cb + j) * x;
                            }
                        } else if (!post) {
                            uint32_t rv[32];
                            TMEM_LD32(tmem + lane_addr + 128 * t + 64 + cb, rv);
                            tmem_wait_ld();
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                y[j] = __uint_as_float(rv[j]) +
                                       fmaf(__uint_as_float(v[j]), __ldg(sc + cb + j), __ldg(sc + 64 + cb + j));
                            uint32_t st[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) st[j] = __float_as_uint(y[j]);
                            TMEM_ST32(tmem + lane_addr + 128 * t + 64 + cb, st);
                            tmem_wait_st();
                        } else {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                uint4 s4 = *reinterpret_cast<const uint4 *>(skip + t * SKIP_TILE + (4 * hh + k) * (ROWS * 16) + row * 16);
                                uint32_t s[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const int j = 8 * k + 2 * e;
                                    y[j] = fmaf(__uint_as_float(v[j]), __ldg(sc + cb + j), __ldg(sc + 64 + cb + j)) + bf16_lo(s[e]);
                                    y[j + 1] = fmaf(__uint_as_float(v[j + 1]), __ldg(sc + cb + j + 1), __ldg(sc + 64 + cb + j + 1)) + bf16_hi(s[e]);
                                }
                            }
                        }
                        uint32_t pk[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(y[2 * j], y[2 * j + 1]);
                        store_act_row(act, t, row, 4 * hh, pk);
                    }
                    if (P.dbg && P.dbg_layer == L + 1 && interior) {
                        const long long k = k0 + t * WPT + wt;
                        if (k < P.nwin) {
                            const int pp = (py - 1) * 6 + (px - 1);
#pragma unroll
                            for (int j = 0; j < 32; ++j) P.dbg[(k * 36 + pp) * 64 + cb + j] = y[j];
                        }
                    }
                    fence_async_smem();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(b_act_ready + 8 * t);
                }
            }
            // ---- up conv halves + pixel shuffle + PReLU -> U; pruned fp32 tail ----
            float *U = reinterpret_cast<float *>(uni);
            const float *TW = reinterpret_cast<const float *>(uni + TW_OFF);
            float *part = reinterpret_cast<float *>(skip);   // [T][72][12] partial tail sums
            for (int h = 0; h < 2; ++h) {
                epi_bar();   // previous users of the union are done
                {
                    const uint4 *src = reinterpret_cast<const uint4 *>(P.blob + BL.tail + size_t(h) * TW_BYTES);
                    uint4 *dst = reinterpret_cast<uint4 *>(uni + TW_OFF);
                    for (int i = et; i < TW_BYTES / 16; i += 256) dst[i] = src[i];
                }
                for (int t = 0; t < T; ++t) {
                    mbar_wait(b_acc_full + 8 * t, af_ph[t]);
                    af_ph[t] ^= 1;
                    tc_fence_after();
                    uint32_t v0[32], v1[32];
                    TMEM_LD32(tmem + lane_addr + 128 * t + 64 * hh, v0);
                    TMEM_LD32(tmem + lane_addr + 128 * t + 64 * hh + 32, v1);
                    tmem_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(b_act_ready + 8 * t);   // accumulator free
                    if (t > 0) epi_bar();   // tail of the previous tile done reading U
                    if (interior) {
                        const int y0 = 2 * (py - 1), x0 = 2 * (px - 1);
                        float *Uw = U + wt * 144 * U_PIX;
#pragma unroll
                        for (int j = 0; j < 64; ++j) {
                            const int ocl = 64 * hh + j, cl = ocl >> 2, i = (ocl >> 1) & 1, jj = ocl & 1;
                            float x = __uint_as_float(j < 32 ? v0[j] : v1[j - 32]);
                            x = x > 0.f ? x : __ldg(up_a + 32 * h + cl) * x;
                            Uw[((y0 + i) * 12 + x0 + jj) * U_PIX + cl] = x;
                            if (P.dbg && P.dbg_layer == P.nl + 1) {
                                const long long k = k0 + t * WPT + wt;
                                if (k < P.nwin) P.dbg[(k * 144 + (y0 + i) * 12 + x0 + jj) * 64 + 32 * h + cl] = x;
                            }
                        }
                    }
                    epi_bar();   // U complete
                    // tail over the kept segments of the tile's two windows
                    Win W0 = window_of(P, k0 + t * WPT), W1 = window_of(P, k0 + t * WPT + 1);
                    const int sx0 = (W0.hi_j - W0.lo_j) / 2, sx1 = (W1.hi_j - W1.lo_j) / 2;
                    const int n0 = W0.valid ? 2 * (W0.hi_i - W0.lo_i) * sx0 : 0;
                    const int n1 = W1.valid ? 2 * (W1.hi_i - W1.lo_i) * sx1 : 0;
                    for (int s = ew; s < n0 + n1; s += 8) {
                        const int w = s < n0 ? 0 : 1;
                        const Win &Wn = w ? W1 : W0;
                        const int ls = w ? s - n0 : s, sx = w ? sx1 : sx0;
                        const int fy = 2 * Wn.lo_i + ls / sx, fx0 = 2 * Wn.lo_j + 4 * (ls % sx);
                        const float *Uw = U + w * 144 * U_PIX + lane;
                        float acc[12];
#pragma unroll
                        for (int a = 0; a < 12; ++a) acc[a] = 0.f;
#pragma unroll 1
                        for (int dy = 0; dy < 9; ++dy) {
                            const int Y = min(max(fy + dy - 4, 0), 11);
                            float u[12];
#pragma unroll
                            for (int m = 0; m < 12; ++m) u[m] = Uw[(Y * 12 + min(max(fx0 - 4 + m, 0), 11)) * U_PIX];
                            const float *tw = TW + dy * 9 * 96 + lane;
#pragma unroll
                            for (int dx = 0; dx < 9; ++dx) {
                                const float w0 = tw[dx * 96], w1 = tw[dx * 96 + 32], w2 = tw[dx * 96 + 64];
#pragma unroll
                                for (int p = 0; p < 4; ++p) {
                                    acc[3 * p] = fmaf(u[p + dx], w0, acc[3 * p]);
                                    acc[3 * p + 1] = fmaf(u[p + dx], w1, acc[3 * p + 1]);
                                    acc[3 * p + 2] = fmaf(u[p + dx], w2, acc[3 * p + 2]);
                                }
                            }
                        }
#pragma unroll
                        for (int a = 0; a < 12; ++a) {
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) acc[a] += __shfl_xor_sync(0xffffffffu, acc[a], o);
                        }
                        float *pp = part + (t * 72 + s) * 12;
                        if (h == 0) {
                            if (lane == 0) {
#pragma unroll
                                for (int a = 0; a < 12; ++a) pp[a] = acc[a];
                            }
                        } else {
                            const long long k = k0 + t * WPT + w;
                            const int fy_g = 2 * Wn.iw + fy;
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                if (lane != p) continue;
                                double m = 0.0;
#pragma unroll
                                for (int o = 0; o < 3; ++o) {
                                    const float pre = pp[3 * p + o] + acc[3 * p + o] + __ldg(tail_b + o);
                                    m += double(P.tanh_s * tanhf(pre / P.tanh_s));
                                }
                                m = m / 3.0;
                                double outv = 0.0;
                                if (m != 0.0) {
                                    double mag = pow(10.0, P.log_lo + fabs(m) * P.span);
                                    outv = m > 0.0 ? mag : -mag;
                                }
                                (void)k;
                                P.fine[(long long)fy_g * P.nf + 2 * Wn.jw + fx0 + p] = outv;
                            }
                        }
                    }
                }
            }
            epi_bar();
        }
    }
    // teardown
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace tc

// ---------------------------------------------------------------------------
// host side

static inline uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    uint32_t r = u + 0x7FFFu + ((u >> 16) & 1u);   // round to nearest even
    return uint16_t(r >> 16);
}
static inline float tf32_rna(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

int tc_pack_weights(mgsr_gen *g, const float *const *t) {
    using namespace tc;
    const int B = g->blocks;
    BlobLayout BL = blob_layout(B);
    std::vector<uint8_t> blob(BL.total, 0);
    // head B: 22 planes x 64 oc x 4 tf32 (3 identical input channels folded)
    {
        float *hb = reinterpret_cast<float *>(blob.data() + BL.head_b);
        const float *w = t[0];
        for (int kc = 0; kc < HPLANES; ++kc)
            for (int oc = 0; oc < 64; ++oc)
                for (int e = 0; e < 4; ++e) {
                    int k = 4 * kc + e;
                    float v = 0.f;
                    if (k < 81) {
                        int dy = k / 9, dx = k % 9;
                        double s = 0.0;
                        for (int c = 0; c < 3; ++c) s += double(w[((oc * 3 + c) * 9 + dy) * 9 + dx]);
                        v = tf32_rna(float(s));
                    }
                    hb[(kc * 64 + oc) * 4 + e] = v;
                }
    }
    auto conv_index = [&](int L) -> int {   // tensor index of body layer L's conv weight
        if (L == 2 * B) return 2 + 11 * B;
        return 2 + 11 * (L / 2) + ((L & 1) ? 6 : 0);
    };
    for (int L = 0; L < BL.nl; ++L) {
        const float *w = t[conv_index(L)];
        for (int tap = 0; tap < 9; ++tap) {
            uint16_t *dst = reinterpret_cast<uint16_t *>(blob.data() + BL.body + (size_t(L) * 9 + tap) * BODY_TAP_BYTES);
            int dy = tap / 3, dx = tap % 3;
            for (int kc = 0; kc < 8; ++kc)
                for (int oc = 0; oc < 64; ++oc)
                    for (int e = 0; e < 8; ++e) {
                        int ic = 8 * kc + e;
                        dst[(kc * 64 + oc) * 8 + e] = f2bf(w[((oc * 64 + ic) * 3 + dy) * 3 + dx]);
                    }
        }
    }
    const int ip = 2 + 11 * B;   // post conv index
    {
        const float *w = t[ip + 5];   // up.conv.weight 256 x 64 x 3 x 3
        for (int h = 0; h < 2; ++h)
            for (int tap = 0; tap < 9; ++tap) {
                uint16_t *dst = reinterpret_cast<uint16_t *>(blob.data() + BL.up + (size_t(h) * 9 + tap) * UP_TAP_BYTES);
                int dy = tap / 3, dx = tap % 3;
                for (int kc = 0; kc < 8; ++kc)
                    for (int ocl = 0; ocl < 128; ++ocl)
                        for (int e = 0; e < 8; ++e) {
                            int ic = 8 * kc + e, oc = 128 * h + ocl;
                            dst[(kc * 128 + ocl) * 8 + e] = f2bf(w[((oc * 64 + ic) * 3 + dy) * 3 + dx]);
                        }
            }
    }
    {
        const float *w = t[ip + 7];   // tail.conv.weight 3 x 64 x 9 x 9
        for (int h = 0; h < 2; ++h) {
            float *dst = reinterpret_cast<float *>(blob.data() + BL.tail + size_t(h) * TW_BYTES);
            for (int dy = 0; dy < 9; ++dy)
                for (int dx = 0; dx < 9; ++dx)
                    for (int o = 0; o < 3; ++o)
                        for (int cl = 0; cl < 32; ++cl)
                            dst[((dy * 9 + dx) * 3 + o) * 32 + cl] = w[((o * 64 + 32 * h + cl) * 9 + dy) * 9 + dx];
        }
    }
    {
        float *cs = reinterpret_cast<float *>(blob.data() + BL.consts);
        for (int i = 0; i < 64; ++i) cs[i] = t[1][i];
        auto bn = [&](int L, int gi) {
            float *sc = cs + 64 + 192 * L;
            for (int i = 0; i < 64; ++i) {
                double k = double(t[gi][i]) / std::sqrt(double(t[gi + 3][i]) + 1e-5);
                sc[i] = float(k);
                sc[64 + i] = float(double(t[gi + 1][i]) - double(t[gi + 2][i]) * k);
            }
        };
        for (int b = 0; b < B; ++b) {
            int base = 2 + 11 * b;
            bn(2 * b, base + 1);
            for (int i = 0; i < 64; ++i) cs[64 + 192 * (2 * b) + 128 + i] = t[base + 5][i];
            bn(2 * b + 1, base + 7);
        }
        bn(2 * B, ip + 1);
        float *upa = cs + 64 + 192 * BL.nl;
        for (int i = 0; i < 64; ++i) upa[i] = t[ip + 6][i];
        for (int o = 0; o < 3; ++o) upa[64 + o] = t[ip + 8][o];
    }
    MGSR_CUDA_TRY(cudaMalloc(&g->tc_blob, BL.total));
    MGSR_CUDA_TRY(cudaMemcpy(g->tc_blob, blob.data(), BL.total, cudaMemcpyHostToDevice));
    g->tc_bytes = BL.total;
    return MGSR_OK;
}

size_t tc_workspace_bytes(int64_t nc) {
    (void)nc;
    return 0;
}

static int g_num_sms = 0;

int launch_sr_pass_tc_dbg(const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo,
                          double span, double *fine, float *dbg, int dbg_layer, cudaStream_t st) {
    using namespace tc;
    if (!g->tc_blob) { set_error("tensor-core weights not packed"); return MGSR_E_UNSUPPORTED; }
    Params P{};
    P.c = c;
    P.c_shift = c_shift;
    P.nc = nc;
    P.npos = nc / 2 - 2;
    P.nwin = (long long)P.npos * P.npos;
    P.ngroups = int((P.nwin + WPG - 1) / WPG);
    P.log_lo = log_lo;
    P.span = span;
    P.fine = fine;
    P.nf = 2 * nc;
    P.blob = static_cast<const uint8_t *>(g->tc_blob);
    P.nl = 2 * g->blocks + 1;
    P.tanh_s = float(g->tanh_scale);
    P.dbg = dbg;
    P.dbg_layer = dbg_layer;
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        MGSR_CUDA_TRY(cudaFuncSetAttribute(k_gen_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    }
    int grid = P.ngroups < g_num_sms ? P.ngroups : g_num_sms;
    k_gen_tc<<<grid, NTHREADS, SMEM_BYTES, st>>>(P);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_sr_pass_tc(const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo, double span,
                      double *fine, void *ws, size_t ws_bytes, cudaStream_t st) {
    (void)ws;
    (void)ws_bytes;
    return launch_sr_pass_tc_dbg(g, c, c_shift, nc, log_lo, span, fine, nullptr, -1, st);
}

}  // namespace mgsr

// debug entry (not in the public header): dump one layer's fp32 output
extern "C" int mgsr_debug_tc_pass(const mgsr_gen *g, const double *c, int64_t nc, double p_min, double p_max,
                                  double *fine, float *dbg, int32_t dbg_layer, void *stream) {
    return mgsr::launch_sr_pass_tc_dbg(g, c, nullptr, int(nc), std::log10(p_min),
                                       std::log10(p_max) - std::log10(p_min), fine, dbg, dbg_layer,
                                       static_cast<cudaStream_t>(stream));
}
