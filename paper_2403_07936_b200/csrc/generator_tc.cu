// Tensor-core (tcgen05/TMEM) generator megakernel for ratio-2 SR passes.
//
// Reference semantics: srmodel.py:285-344 (generator), 414-463 (windowed
// pass), grid.py:103-114 (log normalisation).  Persistent CTA pairs (clusters
// of 2, one CTA per SM) walk groups of 8 windows per CTA; every layer of a
// window group stays on chip:
//
//   * activations: fp16 (or bf16) in shared memory, each 6x6 window stored as
//     an 8x8 image (pad rows py = 0, 7 written; the pad columns are dead data);
//     the group's 8 images are interleaved by image row.  Tile t (M = 128 rows)
//     holds padded rows py = 2t+1, 2t+2 of all 8 windows; three tiles per
//     group; two buffers (layer L reads buffer L % 2).
//   * a 3x3 conv is three MMA chains per tile, one per kernel row dy: A is the
//     plane shifted by dy * 64 rows (the UMMA A-descriptor start address moves,
//     K-major, no swizzle -- no im2col) and B stacks the row's three dx taps
//     (N = 192); the epilogue sums y_0[r - 1] + y_1[r] + y_2[r + 1] with lane
//     shuffles (px -+ 1 are the adjacent lanes; replicate padding = a lane's own
//     partial at px = 1, 6).
//   * cta_group::2: the leader issues M = 256 MMAs (128 rows from each CTA);
//     B is split along N, 32 output channels (x 3 dx) per CTA.
//   * TMEM (512 columns): two 192-column fp32 accumulator buffers (units
//     alternate) and the packed global skip (96 columns); the tail
//     accumulators (Z) reuse the skip columns.  The residual stream is the
//     fp16 activation plane itself.
//   * weights: pre-packed in the UMMA core-matrix layout (BN scale folded),
//     streamed through a 5-unit ring of 12 KB kernel rows (cp.async.bulk +
//     mbarrier complete_tx), read from L2 once per group.
//   * head 9x9 conv: fp16 MMA (K = 81 taps padded to 96, the 3 identical input
//     channels folded) on an im2col built per tile (two buffers), built for
//     the next group before the current group's stitched-pixel epilogue.
//   * body: 2B+1 3x3 convs (fp32 accumulate); PReLU / residual add / global
//     skip fused into the TMEM -> register -> smem epilogue.
//   * up conv 64->256 as four quarters of 64 outputs; PReLU fused; each quarter is
//     drained pixel-shuffled into U (shared memory), the tail's A operand.
//   * tail 9x9 conv (64 -> 3), pruned to the stitched (kept) fine rows of
//     interior windows: the kept rows are M, the vertical tap dy is an A-row
//     shift of U, the horizontal tap dx and the 3 outputs go along N (27 of
//     32), reduced over dx by warp shuffles; windows touching the grid edge
//     (0.4% at n_c = 2048) spill their up-conv output to global memory and an
//     exact fp32 kernel (k_tail_edge) evaluates their tail with the
//     reference's replicate clamping.
//   * bias + s*tanh(x/s) + channel mean + sign-preserving 10^ map in the final
//     epilogue, written straight into the fine fp64 grid.
//
// Warp roles: warp 0 = weight producer, warp 1 = MMA issuer + TMEM allocator
// (the peer CTA's warp 1 forwards its "slot landed" signals to the leader),
// warps 2..17 = epilogue (512 threads; warp w reads TMEM lane quadrant w%4,
// channel quarter (w-2)/4).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
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
constexpr int ROWS = 128;            // rows per tile
constexpr int GUARD = 8;             // plane rows before / after the image
// Pass variants (template parameter V of k_gen_tc):
//   V = 0  ratio-2 pass: 6x6 windows of q (3 identical channels), tail pruned to the kept pixels;
//   V = 1  first application of a ratio-4 pass: 6x6 windows of q, the full 12x12x3 output (replicate-
//          padded 9x9 tail at every pixel) -> X1 in global memory (fp16, the next head's operand format);
//   V = 2  second application: 12x12 windows of X1 (3 distinct channels), tail pruned to the kept 8x8 fine
//          pixels of the 24x24 output (srmodel.py:443-467, _PASS_PLAN).
// Activations: per 8-channel plane, padded image row py (0 .. WS + 1) of the group's windows occupies RPY
// plane rows: RPY / 32 lane blocks of 32 rows, each holding WPB windows' WS interior pixels (px = 1..WS, row
// WS w' + px - 1) plus spare rows (dead data).  The pad columns px = 0, WS + 1 are not stored: replicate
// padding is a lane's own partial (see load_dx3).  Tile tau holds rows py = TPY tau + 1 .. TPY tau + TPY
// (M = 128), so the pad rows py = 0, WS + 1 are stored but never computed.  Tap row dy is the descriptor
// shift dy * RPY rows.  Two buffers (ping-pong: layer L reads buffer L % 2), because a tile's taps read its
// neighbours' rows.
//   V = 0, 1: 10 windows per group (two lane blocks of 5 x 6 px + 2 spare; 94% useful M rows);
//   V = 2:    2 windows per group (one lane block of 2 x 12 px + 8 spare; 75%).
template <int V>
struct Geo {
    static constexpr int WS = V == 2 ? 12 : 6;            // input window side
    static constexpr int NPY = WS + 2;                    // padded image rows
    static constexpr int RPY = V == 2 ? 32 : 64;          // plane rows per padded image row
    static constexpr int TPY = ROWS / RPY;                // padded rows per tile
    static constexpr int WPB = 32 / WS;                   // windows per 32-lane block (5, 2)
    static constexpr int WPG = (RPY / 32) * WPB;          // windows per group (per CTA): 10, 2
    static constexpr int ACT_PLANE = (2 * GUARD + NPY * RPY) * 16;   // bytes per 8-channel plane
    static constexpr int HK = V == 2 ? 256 : 96;          // head K: 81 (x 3 distinct channels) taps, padded
    static constexpr int I2C_PLANES = V == 2 ? 8 : 12;    // planes per im2col build (K 64 / 96)
    static constexpr int NBUILD = HK / (8 * I2C_PLANES);  // im2col builds per tile (4 / 1)
    static constexpr int HUNITS = V == 2 ? 2 : 1;         // ring units of this CTA's head weights
    static constexpr int NZC = V == 1 ? 3 : 1;            // up-phase chunks (V = 1: 4 output rows each)
    static constexpr int ZT = V == 2 ? 2 : 4;             // Z tiles per chunk
    static constexpr int UROWS_Y = V == 2 ? 32 : 128;     // U pixel rows per fine row
    static constexpr int UNY = V == 2 ? 16 : 12;          // U fine rows held
    static constexpr int U_PLANE = UNY * UROWS_Y * 16;
    static constexpr int ZSH = V == 2 ? 4 : 1;            // fine rows per Z tile (Z tile j: shift ZSH j)
    static constexpr int QN = V == 2 ? 432 : 36;          // input values per window (misc q tables)
    __host__ __device__ static constexpr bool spare(int r) { return (r & 31) >= WPB * WS; }
    __host__ __device__ static constexpr int window(int r) { return spare(r) ? 0 : ((r % RPY) >> 5) * WPB + (r & 31) / WS; }
    __host__ __device__ static constexpr int px(int r) { return spare(r) ? 1 : (r & 31) % WS + 1; }
};
constexpr int ACT_BYTES = 8 * Geo<0>::ACT_PLANE;     // 67584 per buffer (the largest variant)
static_assert(8 * Geo<2>::ACT_PLANE <= ACT_BYTES, "activation buffer");
// CTA pair (cta_group::2): the leader CTA issues M = 256 MMAs whose A rows come 128 from each CTA's
// activations.  The three taps of a kernel row dy (dx = 0, 1, 2) are ONE MMA with N = 3 x 64 = 192: A is the
// plane shifted by dy rows only and the accumulator holds y_dx[r] = sum_dy W(dy, dx) a[r + RPY (dy - 1)];
// the epilogue forms out[r] = y_0[r - 1] + y_1[r] + y_2[r + 1] with lane shuffles (a row's px -+ 1
// neighbours are the adjacent lanes), so A is read from shared memory 3 times per layer instead of 9.
// B is split along N: each CTA's ring unit holds its 32 output channels for the 3 dx taps (N = 96).
constexpr int NUNIT = 5;                              // ring units (> 3: the next layer's first rows prefetch)
constexpr int TAP_BYTES = 8192;                       // one 3x3 tap in the blob (both 32-oc halves)
constexpr int UNIT_BYTES = 3 * 4096;                  // this CTA's half of a kernel row: [dx 3][ng 4][kc 8][8 oc][8]
constexpr int ROW_BYTES = 2 * UNIT_BYTES;             // a kernel row in the blob (both halves)
constexpr int RING_BYTES = NUNIT * UNIT_BYTES;        // 61440
static_assert(3 * ROW_BYTES == 9 * TAP_BYTES, "a layer is 9 taps");
constexpr int MISC_BYTES = 8192;                      // q tables (10 x 36 / 2 x 432 floats) + head im2col index table
constexpr int BAR_BYTES = 1024;
// head phase, in activation buffer 1 (free until layer 0's epilogue): im2col, two buffers.  V = 0, 1: fp16
// MMA over the 81 folded taps (the 3 identical input channels summed into the weights) padded to K = 96,
// indices from a table; V = 2: K = 3 x 81 padded to 256, built in four K = 64 parts per tile.
constexpr int HPLANES = 12;                              // V = 0, 1 head K planes of 8 fp16
constexpr int I2C_BYTES = 12 * ROWS * 16;                // 24576 per im2col buffer (two buffers)
constexpr int HB_BYTES = HPLANES * 64 * 16;              // 12288: two halves of 32 oc
constexpr int HB_HALF = HB_BYTES / 2;                    // 6144, streamed through the ring (one unit)
constexpr int HB4_BYTES = 32 * 64 * 16;                  // V = 2: 32768, halves of 16384 = two ring units
constexpr int HB4_HALF = HB4_BYTES / 2;
constexpr int IDX_OFF = 2048;                            // in misc: uint8 [64 padded pixels][96 k] -> q index
static_assert(2 * I2C_BYTES <= ACT_BYTES, "im2col");
static_assert(Geo<0>::WPG * 36 * 4 <= IDX_OFF && IDX_OFF + 64 * 96 <= MISC_BYTES, "misc");
static_assert(Geo<2>::WPG * 432 * 4 <= MISC_BYTES, "misc (V = 2)");
// up phase, in activation buffer 0 (free once the post layer's MMAs completed): the up-conv quarter
// pixel-shuffled onto the fine windows, as the tail's A operand: 2 planes (8 channels each) x UNY fine rows x
// UROWS_Y pixel rows of 16 B.
//   V = 0: rows [Y 12][12 w + X] (120 of 128 used); Z tile j = kept fine row y = 4 + j of the 10 windows
//          (A rows (window, X)), so the vertical tap dy is a 128-row descriptor shift;
//   V = 1: chunk zc holds fine rows 4 zc - 4 .. 4 zc + 7 (replicate-clamped at the window edge); Z tile j =
//          fine row 4 zc + j;
//   V = 2: rows [Y 4..19][16 w + X - 4] (X 4..19: what the kept X 8..15 read); Z tile j = fine rows
//          8 + 4 j .. 11 + 4 j.
// The horizontal tap dx and the output o go along N (n = 3 dx + o, 27 of 32).  V = 0, 1 sum over dx through
// shared memory (a window's row crosses lane quadrants), V = 2 by lane shuffles.  Tail weights per quarter:
// this CTA's 16 N rows, [dy 9][k 2][16 n][8].
constexpr int UQ = 16;
constexpr int UP_QUARTERS_C = 4;
// Up-conv column order: epilogue thread cq's 16 columns j of a quarter are 8 shuffled channels (m = j / 2 of
// the quarter's channel group cq / 2) x the two sub-pixels jj = j % 2 of sub-row ii = cq % 2, so a thread
// writes two adjacent 16-byte U pixel rows (32 B contiguous, lanes contiguous).  Column 16 cq + j holds the
// up conv's output channel 64 u + up_col_channel(16 cq + j) = 4 c + 2 ii + jj (pixel shuffle, srmodel.py:321).
__host__ __device__ constexpr int up_col_channel(int col) {
    return 32 * ((col >> 4) >> 1) + 4 * ((col & 15) >> 1) + 2 * ((col >> 4) & 1) + (col & 1);
}
constexpr int U_BYTES_MAX = 2 * Geo<0>::U_PLANE;       // 49152
constexpr int TW_HALF = 9 * 512;                       // 4608: this CTA's half of a quarter's tail weights
constexpr int TW_QBYTES = 2 * TW_HALF;                 // a quarter in the blob (both halves)
constexpr int TW_OFF0 = U_BYTES_MAX;
static_assert(2 * Geo<2>::U_PLANE <= TW_OFF0 && 2 * Geo<1>::U_PLANE <= TW_OFF0, "U");
static_assert(TW_OFF0 + UP_QUARTERS_C * TW_HALF <= ACT_BYTES, "up phase");
constexpr int ZS_STRIDE = 27;                         // Z scratch: [tile][row 128][27] fp32 in buffer 0
static_assert(4 * ROWS * ZS_STRIDE * 4 <= ACT_BYTES, "Z scratch (V = 0)");
static_assert(2 * ROWS * ZS_STRIDE * 4 <= U_BYTES_MAX, "Z scratch (V = 1, in U)");
constexpr int OFF_ACT = 0;                             // two buffers
constexpr int OFF_RING = OFF_ACT + 2 * ACT_BYTES;
constexpr int OFF_MISC = OFF_RING + RING_BYTES;
constexpr int OFF_BAR = OFF_MISC + MISC_BYTES;
constexpr int OFF_CONST = OFF_BAR + BAR_BYTES;
// TMEM columns: two 192-column accumulator buffers (accumulator units alternate between them: head tiles,
// body / post tiles, up-quarter tiles), then the packed global skip
constexpr int COL_ACC = 0, ACC_COLS = 192, COL_SKIP = 384;
constexpr int COL_Z = COL_SKIP;   // tail accumulators (32 per Z tile, <= 4 tiles) reuse the skip columns + the spare 32

constexpr int NEPI = 16;                       // epilogue warps
constexpr int NTHREADS = 64 + 32 * NEPI;       // 576
constexpr int UP_QUARTERS = 4;
constexpr int BLOB_COPIES = 1;                 // weight blob replicas in HBM/L2: CTA b streams copy b % 8,
                                               // spreading the lockstep weight stream over more L2 slices

__host__ __device__ inline int const_floats(int nl) { return 64 + 192 * nl + 64 + 4; }
__host__ __device__ inline int smem_bytes(int nl) { return OFF_CONST + 4 * const_floats(nl); }

// blob layout (bytes); body layer count NL = 2B + 1
struct BlobLayout {
    size_t head_b, body, up, tail, tail_f32, consts, head4, fmt_stride, total;
    int nl;
};

__host__ __device__ inline BlobLayout blob_layout(int blocks) {
    BlobLayout L;
    L.nl = 2 * blocks + 1;
    L.head_b = 0;
    L.body = L.head_b + HB_BYTES;
    L.up = L.body + size_t(L.nl) * 3 * ROW_BYTES;
    L.tail = L.up + size_t(UP_QUARTERS) * 3 * ROW_BYTES;
    L.tail_f32 = L.tail + size_t(UP_QUARTERS) * TW_QBYTES;   // then [3][64][81] fp32 (edge kernels)
    L.consts = L.tail_f32 + sizeof(float) * 3 * 64 * 81;
    // V = 2 head (3 distinct input channels, fp16): [half][kc 32][32 oc][8]
    L.head4 = ((L.consts + sizeof(float) * const_floats(L.nl)) + 1023) & ~size_t(1023);
    // fp16 operand set (body, up, tail) follows at +fmt_stride from the bf16 set
    L.fmt_stride = (L.head4 + HB4_BYTES + 1023) & ~size_t(1023);
    L.total = L.fmt_stride + L.tail_f32;
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
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n\t"
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
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// completion of the pair's MMAs -> the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"((unsigned short)3)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the leader CTA's barrier at this offset (the leader's MMA warp waits on it)
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(bar));
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");   // .release.cta (as CUTLASS)
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

#define TMEM_LD16(taddr, v)                                                                                   \
    asm volatile(                                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),     \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]) \
        : "r"(taddr))
#define TMEM_ST16(taddr, v)                                                                                   \
    asm volatile(                                                                                             \
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), \
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])          \
        : "memory")
#define TMEM_LD32(taddr, v)                                                                                   \
    asm volatile(                                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"       \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                            \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),     \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),          \
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),          \
          "=r"(v[30]), "=r"(v[31])                                                                           \
        : "r"(taddr))
#define TMEM_LD8(taddr, v)                                                                                    \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                     \
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),       \
                   "=r"(v[7])                                                                                 \
                 : "r"(taddr))
#define TMEM_ST8(taddr, v)                                                                                    \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),        \
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])     \
                 : "memory")

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void lds16(const float *src, float (&dst)[16]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float4 v = reinterpret_cast<const float4 *>(src)[k];
        dst[4 * k] = v.x;
        dst[4 * k + 1] = v.y;
        dst[4 * k + 2] = v.z;
        dst[4 * k + 3] = v.w;
    }
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
template <bool F16>
__device__ __forceinline__ uint32_t pack_op(float a, float b) {
    if (F16) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t *>(&h);
    }
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
template <bool F16>
__device__ __forceinline__ float op_lo(uint32_t u) {
    if (F16) return __half2float(__ushort_as_half(uint16_t(u & 0xFFFFu)));
    return __uint_as_float(u << 16);
}
template <bool F16>
__device__ __forceinline__ float op_hi(uint32_t u) {
    if (F16) return __half2float(__ushort_as_half(uint16_t(u >> 16)));
    return __uint_as_float(u & 0xFFFF0000u);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ float bf16_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// instruction descriptors: D fp32, K-major A and B, M = 256 (CTA pair)
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_f16(int n) {   // a/b format 0 = F16
    return (1u << 4) | (uint32_t(n >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}

struct Params {
    const double *c;
    const double *c_shift;
    int nc, npos;
    long long nwin;
    int ngroups;
    double log_lo, span;
    double *fine;
    int nf;
    const float *qgrid;   // normalised coarse grid, tf32-rounded fp32 (k_normalize)
    const uint8_t *blob;
    int nl;
    float tanh_s;
    uint16_t *edge_u;   // [n_edge][36][256] bf16 up-conv output of edge windows
    size_t wfmt;        // byte offset of the operand-format weight set (0: bf16, BL.fmt_stride: fp16)
    float *dbg;
    int dbg_layer;
    unsigned long long *prof;   // optional event trace (bring-up instrumentation, tests/tc_trace.py)
    uint16_t *x1;               // ratio-4 passes: [nwin][3][12][12] fp16 first-application output (V = 1 -> V = 2)
    // batched ratio-2 passes (V = 0, mgsr_plan_solve_batch): the windows of the *rhs_count grids listed in
    // rhs_list, nwin1 windows each; grid r's q at qgrid + r q_stride, its output at fine + r fine_stride, its
    // edge spill at edge_u + r edge_count(npos) windows.  rhs_list == nullptr: one grid.
    const int *rhs_list;
    const int *rhs_count;
    long long nwin1, q_stride, fine_stride;
};

// Event trace of one steady-state group of CTA 0: role r (0 producer, 1 MMA, 2 epilogue warp 2,
// 3 epilogue warp 10) appends (id, clock64) pairs at prof[r * 4096 + 2 i]; id = type * 1000 + a * 10 + b.
constexpr int TRACE_GROUP = 3;
template <bool ON>
struct Tracer {
    unsigned long long *buf;
    int n;
    __device__ __forceinline__ void operator()(int type, int a, int b) {
        if (ON && buf && n < 2040) {
            buf[2 * n] = (unsigned long long)(type * 1000 + a * 10 + b);
            buf[2 * n + 1] = (unsigned long long)clock64();
            ++n;
        }
    }
};

// window geometry of a global window index (srmodel.py:414-440)
struct Win {
    int iw, jw, wi, wj, rhs;
    bool valid, edge;
};
template <bool BATCH>
__device__ __forceinline__ Win window_of(const Params &P, long long k, long long nwin) {
    Win w;
    w.valid = k < nwin;
    w.rhs = 0;
    int kk;
    if (BATCH) {
        long long kg = w.valid ? k : nwin - 1;
        const long long slot = kg / P.nwin1;
        w.rhs = P.rhs_list[slot];
        kk = int(kg - slot * P.nwin1);
    } else {
        kk = int(w.valid ? k : P.nwin - 1);
    }
    w.wi = kk / P.npos;
    w.wj = kk - w.wi * P.npos;
    w.iw = 2 * w.wi;
    w.jw = 2 * w.wj;
    w.edge = w.wi == 0 || w.wj == 0 || w.wi == P.npos - 1 || w.wj == P.npos - 1;
    return w;
}
// index of an edge window among the 4 npos - 4 edge windows (row 0, row last, then the side columns)
__host__ __device__ __forceinline__ int edge_index(int wi, int wj, int npos) {
    if (npos == 1) return 0;
    if (wi == 0) return wj;
    if (wi == npos - 1) return npos + wj;
    return 2 * npos + 2 * (wi - 1) + (wj == 0 ? 0 : 1);
}
__host__ __device__ inline int edge_count(int npos) { return npos == 1 ? 1 : 4 * npos - 4; }

__device__ __forceinline__ double normalize_q(double v, double log_lo, double span) {
    if (v == 0.0) return 0.0;
    double t = (log10(fabs(v)) - log_lo) / span;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    return v > 0.0 ? t : -t;
}
__device__ __forceinline__ double denormalize_q(double q, double log_lo, double span) {
    if (q == 0.0) return 0.0;   // sign 0 annihilates (grid.py:112-114)
    const double mag = pow(10.0, log_lo + fabs(q) * span);
    return q > 0.0 ? mag : -mag;
}

// INSTR: bring-up instrumentation (P.prof event trace, P.dbg layer dumps) compiled in
// BATCH (V = 0 only): the windows of several grids (Params::rhs_list), mgsr_plan_solve_batch
template <bool F16, bool INSTR, int V, bool BATCH = false>
__global__ void __launch_bounds__(NTHREADS, 1) k_gen_tc(Params P) {
    using G = Geo<V>;
    constexpr int RPY = G::RPY, TPY = G::TPY, GWPG = G::WPG, ACT_PLANE = G::ACT_PLANE;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t *act = smem + OFF_ACT;   // two buffers of ACT_BYTES
    uint8_t *ring = smem + OFF_RING;
    float *misc = reinterpret_cast<float *>(smem + OFF_MISC);
    float *cs = reinterpret_cast<float *>(smem + OFF_CONST);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + OFF_BAR);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + OFF_BAR + BAR_BYTES - 8);
    uint8_t *i2c = act + ACT_BYTES;   // head phase: im2col in buffer 1
    uint8_t *ubuf = act;              // up phase: U + tail weights in buffer 0
    // Barriers marked (leader) are waited on by the leader's MMA warp only and collect the arrivals of
    // both CTAs; (both) are signalled in both CTAs by the leader's multicast commits; the rest are local.
    const uint32_t b_full = smem_u32(bars + 0);                     // [NUNIT] this CTA's ring unit landed
    const uint32_t b_empty = smem_u32(bars + NUNIT);                // [NUNIT] (both) unit consumed
    const uint32_t b_peerfull = smem_u32(bars + 2 * NUNIT);         // [NUNIT] (leader) peer's unit landed
    constexpr int BB = 3 * NUNIT;
    const uint32_t b_acc_full = smem_u32(bars + BB + 0);    // [2] (both) MMA -> epilogue: accumulator buffer ready
    const uint32_t b_drained = smem_u32(bars + BB + 2);     // [2] (leader) epilogues -> MMA: accumulator buffer read
    const uint32_t b_act_ready = smem_u32(bars + BB + 4);   // [T] (leader) epilogues -> MMA: tile's rows written
    const uint32_t b_i2c_full = smem_u32(bars + BB + 7);    // [2] (leader) im2col buffer built (both CTAs)
    const uint32_t b_i2c_empty = smem_u32(bars + BB + 9);   // [2] (both) im2col buffer consumed
    const uint32_t b_ubuf_full = smem_u32(bars + BB + 11);  // (leader) drains -> MMA: the quarter's U written
    const uint32_t b_ubuf_free = smem_u32(bars + BB + 12);  // (both) tail MMAs -> drains: U consumed
    const uint32_t b_zfull = smem_u32(bars + BB + 13);      // [4] (both) last tail MMAs -> epilogue: Z ready
    const uint32_t b_tw_full = smem_u32(bars + BB + 17);    // [4] this CTA's quarter tail weights landed
    const uint32_t b_tw_peerfull = smem_u32(bars + BB + 21);   // [4] (leader) the peer's landed
    const uint32_t b_tw_empty = smem_u32(bars + BB + 25);   // [4] (both) tail MMAs of the quarter done
    const uint32_t b_post_done = smem_u32(bars + BB + 29);  // (both) post layer's MMAs done: buffer 0 free
    static_assert((BB + 30) * 8 <= BAR_BYTES - 8, "barriers");
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = int(blockIdx.x >> 1), npairs = int(gridDim.x >> 1);
    // batched passes: the device-side count of grids in this launch
    const long long nwin = BATCH ? (long long)(*P.rhs_count) * P.nwin1 : P.nwin;
    const int ngp = ((BATCH ? int((nwin + GWPG - 1) / GWPG) : P.ngroups) + 1) >> 1;   // the pair processes groups 2 gp (leader) and 2 gp + 1 (peer)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NL = P.nl, NLAYERS = P.nl;
    const BlobLayout BL = blob_layout((P.nl - 1) / 2);
    const uint8_t *wblob = P.blob + size_t(blockIdx.x % BLOB_COPIES) * ((BL.total + 1023) & ~size_t(1023));

    {
        const float4 *src = reinterpret_cast<const float4 *>(P.blob + BL.consts);
        float4 *dst = reinterpret_cast<float4 *>(cs);
        for (int i = threadIdx.x; i < const_floats(NL) / 4; i += NTHREADS) dst[i] = src[i];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NUNIT; ++s) {
            mbar_init(b_full + 8 * s, 1);
            mbar_init(b_empty + 8 * s, 1);
            mbar_init(b_peerfull + 8 * s, 1);
        }
        for (int b2 = 0; b2 < 2; ++b2) {
            mbar_init(b_i2c_full + 8 * b2, 2);
            mbar_init(b_i2c_empty + 8 * b2, 1);
        }
        for (int b2 = 0; b2 < 2; ++b2) {
            mbar_init(b_acc_full + 8 * b2, 1);
            mbar_init(b_drained + 8 * b2, 2 * NEPI);
        }
        for (int t = 0; t < T; ++t) mbar_init(b_act_ready + 8 * t, 2 * NEPI);
        mbar_init(b_ubuf_full, 2 * NEPI);
        mbar_init(b_ubuf_free, 1);
        mbar_init(b_post_done, 1);
        for (int j = 0; j < 4; ++j) mbar_init(b_zfull + 8 * j, 1);
        for (int u = 0; u < UP_QUARTERS_C; ++u) {
            mbar_init(b_tw_full + 8 * u, 1);
            mbar_init(b_tw_peerfull + 8 * u, 1);
            mbar_init(b_tw_empty + 8 * u, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {   // both CTAs of the pair, same warp
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();   // barriers of both CTAs initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ================= weight producer =================
        uint32_t ph = 0;   // bit s = fill parity of unit s
        int slot = 0;      // kernel rows stream through the ring in order: unit = global row index mod NUNIT
        uint32_t tw_ph[UP_QUARTERS_C] = {0, 0, 0, 0};
        uint32_t grp_ph = 0;
        auto fill = [&](const uint8_t *src, uint32_t bytes = UNIT_BYTES) {
            mbar_wait(b_empty + 8 * slot, ((ph >> slot) & 1u) ^ 1u);
            if (elect_one()) {
                mbar_expect_tx(b_full + 8 * slot, bytes);
                bulk_g2s(smem_u32(ring + slot * UNIT_BYTES), src, bytes, b_full + 8 * slot);
            }
            __syncwarp();
            ph ^= 1u << slot;
            slot = slot == NUNIT - 1 ? 0 : slot + 1;
        };
        for (int gp = pair; gp < ngp; gp += npairs) {
            if constexpr (V == 2) {   // this CTA's half of the 3-channel head weights, two K halves
                fill(wblob + BL.head4 + rank * HB4_HALF, HB4_HALF / 2);
                fill(wblob + BL.head4 + rank * HB4_HALF + HB4_HALF / 2, HB4_HALF / 2);
            } else {
                fill(wblob + BL.head_b + rank * HB_HALF, HB_HALF);   // this CTA's half of the head weights
            }
            for (int L = 0; L < NLAYERS; ++L)
                for (int dy = 0; dy < 3; ++dy)
                    fill(wblob + P.wfmt + BL.body + (size_t(L) * 3 + dy) * ROW_BYTES + rank * UNIT_BYTES);
            for (int zc = 0; zc < G::NZC; ++zc)
                for (int u = 0; u < UP_QUARTERS; ++u) {
                    for (int dy = 0; dy < 3; ++dy)
                        fill(wblob + P.wfmt + BL.up + (size_t(u) * 3 + dy) * ROW_BYTES + rank * UNIT_BYTES);
                    if (zc > 0) continue;   // the tail weights stay for every chunk of the group
                    // this CTA's half of the quarter's tail weights -> buffer 0, once the post layer's MMAs
                    // released it and the last group's tail MMAs of quarter u completed
                    if (u == 0) mbar_wait(b_post_done, grp_ph);
                    mbar_wait(b_tw_empty + 8 * u, tw_ph[u] ^ 1u);
                    tw_ph[u] ^= 1u;
                    if (elect_one()) {
                        mbar_expect_tx(b_tw_full + 8 * u, TW_HALF);
                        bulk_g2s(smem_u32(ubuf + TW_OFF0 + u * TW_HALF),
                                 wblob + P.wfmt + BL.tail + size_t(u) * TW_QBYTES + rank * TW_HALF, TW_HALF,
                                 b_tw_full + 8 * u);
                    }
                    __syncwarp();
                }
            grp_ph ^= 1u;
        }
    } else if (warp == 1 && !leader) {
        // ================= peer: forward "slot landed" to the leader =================
        uint32_t ph = 0, twp = 0;
        int slot = 0;
        auto fwd = [&](int nfills) {
            for (int i = 0; i < nfills; ++i) {
                mbar_wait(b_full + 8 * slot, (ph >> slot) & 1u);
                if (elect_one()) mbar_arrive_leader(b_peerfull + 8 * slot);
                __syncwarp();
                ph ^= 1u << slot;
                slot = slot == NUNIT - 1 ? 0 : slot + 1;
            }
        };
        for (int gp = pair; gp < ngp; gp += npairs) {   // same order as the producer's fills
            fwd(G::HUNITS + NLAYERS * 3);
            for (int zc = 0; zc < G::NZC; ++zc)
                for (int u = 0; u < UP_QUARTERS; ++u) {
                    fwd(3);
                    if (zc > 0) continue;
                    mbar_wait(b_tw_full + 8 * u, twp);
                    if (elect_one()) mbar_arrive_leader(b_tw_peerfull + 8 * u);
                    __syncwarp();
                }
            twp ^= 1u;
        }
    } else if (warp == 1) {
        // ================= MMA issuer (leader; warp-uniform control, one elected lane issues) =================
        uint32_t ph = 0, i2c_ph = 0;   // i2c_ph bit b: parity of the next completion of b_i2c_full[b]
        int slot0 = 0;   // ring unit of kernel row 0 of the current layer
        uint32_t ar_ph = 0;   // bit t: parity of the next completion of b_act_ready[t]
        uint32_t dr_ph = 0;   // bit b: parity of the next completion of b_drained[b]
        int vb = 0;           // accumulator buffer of the next accumulator unit (units alternate buffers)
        const uint32_t act_base = smem_u32(act), ring_base = smem_u32(ring);
        const uint32_t i2c_base = smem_u32(i2c), u_base = smem_u32(ubuf);
        const uint32_t id192 = F16 ? idesc_f16(192) : idesc_bf16(192);
        Tracer<INSTR> tr{nullptr, 0};
        // the accumulator buffer of the next unit was read by the epilogue of the unit two before
        auto acquire_acc = [&] {
            mbar_wait(b_drained + 8 * vb, (dr_ph >> vb) & 1u);
            dr_ph ^= 1u << vb;
        };
        // one 3x3 64 -> 64 layer over the three tiles (body, post, up quarter), reading buffer `buf`: per tile
        // three N = 192 MMA chains (kernel rows dy) of K = 64.  wait_act: the rows each kernel row reads are
        // written -- tile t's rows dy = 0, 1 read padded rows up to its own, only dy = 2 reaches the first row
        // of tile t + 1, so the previous layer's tile t + 1 epilogue is waited for just before it
        auto conv_layer = [&](int lid, int buf, bool wait_act, auto &&after_t0) {
            const uint64_t a_desc0 = make_desc(act_base + buf * ACT_BYTES, ACT_PLANE, 128);
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const uint32_t arp = ar_ph;
                acquire_acc();
                if (lane == 0) tr(2, lid, t);
                tc_fence_after();
                const uint64_t a_t = a_desc0 + uint64_t(GUARD + (TPY * t + 1) * RPY);
                const uint32_t d = tmem + COL_ACC + ACC_COLS * vb;
                if (elect_one()) {
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy) {
                        int s = slot0 + dy;
                        s = s >= NUNIT ? s - NUNIT : s;
                        if (wait_act && ((t == 0 && dy == 0) || (t < T - 1 && dy == 2))) {
                            const int ta = dy == 0 ? 0 : t + 1;
                            mbar_wait(b_act_ready + 8 * ta, (arp >> ta) & 1u);
                            tc_fence_after();
                        }
                        if (t == 0) {
                            mbar_wait(b_full + 8 * s, (ph >> s) & 1u);
                            mbar_wait(b_peerfull + 8 * s, (ph >> s) & 1u);
                            if (dy == 0) tr(4, lid, 0);
                            tc_fence_after();
                        }
                        const uint64_t a = a_t + uint64_t(int64_t((dy - 1) * RPY));
                        const uint64_t b = make_desc(ring_base + s * UNIT_BYTES, 128, 1024);   // 12 n-groups of 8
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            mma_bf16(d, a + uint64_t(ks * (2 * ACT_PLANE / 16)), b + uint64_t(ks * (256 / 16)), id192,
                                     (dy | ks) > 0);
                        if (t == T - 1) umma_commit(b_empty + 8 * s);
                    }
                    umma_commit(b_acc_full + 8 * vb);
                    if (lid == NLAYERS && t == T - 1) umma_commit(b_post_done);   // buffer 0 no longer read
                }
                __syncwarp();
                if (wait_act) ar_ph ^= t == 0 ? 3u : (t == 1 ? 4u : 0u);
                vb ^= 1;
                if (lane == 0) tr(3, lid, t);
                if (t == 0) after_t0();
            }
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
                int s = slot0 + dy;
                s = s >= NUNIT ? s - NUNIT : s;
                ph ^= 1u << s;
            }
            slot0 += 3;
            slot0 = slot0 >= NUNIT ? slot0 - NUNIT : slot0;
        };
        // pruned 9x9 tail, quarter u: Z[j] (M = 256 pixels of the tile's fine rows, N = 32 = 3 dx + o) +=
        // sum over dy of U shifted by ZSH j + dy fine rows x TW[u][dy]
        const uint32_t idz = F16 ? idesc_f16(32) : idesc_bf16(32);
        uint32_t grp_ph = 0;   // parity of this pair's group iteration (one TW completion per group)
        auto tail_mma = [&](int u, bool last_chunk) {
            mbar_wait(b_tw_full + 8 * u, grp_ph);
            mbar_wait(b_tw_peerfull + 8 * u, grp_ph);
            mbar_wait(b_ubuf_full, uint32_t(u & 1));
            if (lane == 0) tr(16, u, 0);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll 1
                for (int j = 0; j < G::ZT; ++j) {
                    const uint32_t d = tmem + COL_Z + 32 * j;
#pragma unroll
                    for (int dy = 0; dy < 9; ++dy) {
                        const uint64_t a = make_desc(u_base + (G::ZSH * j + dy) * (G::UROWS_Y * 16), G::U_PLANE, 128);
                        const uint64_t b = make_desc(u_base + TW_OFF0 + u * TW_HALF + dy * 512, 256, 128);
                        mma_bf16(d, a, b, idz, (u | dy) > 0);
                    }
                    if (u == UP_QUARTERS - 1) umma_commit(b_zfull + 8 * j);
                }
                umma_commit(b_ubuf_free);
                if (last_chunk) umma_commit(b_tw_empty + 8 * u);
            }
            __syncwarp();
        };
        int hb = 0;   // im2col builds consumed (buffer hb & 1)
        for (int gp = pair; gp < ngp; gp += npairs) {
            tr.buf = (P.prof && blockIdx.x == 0 && gp == TRACE_GROUP * npairs) ? P.prof + 4096 : nullptr;
            // head: D[t] = im2col (128 x HK, fp16) x Wh^T (HK x 64), in G::NBUILD K parts per tile, each part one
            // im2col build (buffers alternate)
            for (int t = 0; t < T; ++t) {
                acquire_acc();
                if (lane == 0) tr(2, 0, t);
                const uint32_t d = tmem + COL_ACC + ACC_COLS * vb;
#pragma unroll 1
                for (int kq = 0; kq < G::NBUILD; ++kq) {
                    const int ib = hb & 1;
                    mbar_wait(b_i2c_full + 8 * ib, (i2c_ph >> ib) & 1u);
                    if (lane == 0) tr(5, kq, t);
                    i2c_ph ^= 1u << ib;
                    tc_fence_after();
                    int s = slot0 + (V == 2 ? (kq >> 1) : 0);
                    s = s >= NUNIT ? s - NUNIT : s;
                    if (elect_one()) {
                        if (t == 0 && (V != 2 || (kq & 1) == 0)) {
                            mbar_wait(b_full + 8 * s, (ph >> s) & 1u);
                            mbar_wait(b_peerfull + 8 * s, (ph >> s) & 1u);
                            tc_fence_after();
                        }
#pragma unroll
                        for (int ks = 0; ks < G::I2C_PLANES / 2; ++ks) {
                            uint64_t a = make_desc(i2c_base + ib * I2C_BYTES + 2 * ks * (ROWS * 16), ROWS * 16, 128);
                            const int bk = V == 2 ? (kq & 1) * 4 + ks : ks;
                            uint64_t b = make_desc(ring_base + s * UNIT_BYTES + bk * 1024, 32 * 16, 128);
                            mma_bf16(d, a, b, idesc_f16(64), (kq | ks) > 0);
                        }
                        if (t == T - 1 && (V != 2 || (kq & 1) == 1)) umma_commit(b_empty + 8 * s);
                        if (kq == G::NBUILD - 1) umma_commit(b_acc_full + 8 * vb);
                        umma_commit(b_i2c_empty + 8 * ib);
                    }
                    __syncwarp();
                    ++hb;
                }
                vb ^= 1;
                if (lane == 0) tr(3, 0, t);
            }
#pragma unroll
            for (int h = 0; h < G::HUNITS; ++h) {
                ph ^= 1u << slot0;
                slot0 = slot0 == NUNIT - 1 ? 0 : slot0 + 1;
            }
            auto none = [] {};
#pragma unroll 1
            for (int L = 0; L < NLAYERS; ++L) conv_layer(L + 1, L & 1, true, none);
            // up quarters (reading buffer NL & 1 = 1); the tail of quarter u issues after tile 0 of up
            // quarter u + 1 (u is drained into U by then), so it completes before that quarter's tiles 1, 2
            // and the drain of u + 1 (which rewrites U) overlaps their MMAs
#pragma unroll 1
            for (int zc = 0; zc < G::NZC; ++zc) {
                const bool lc = zc == G::NZC - 1;
                conv_layer(40, 1, zc == 0, none);
                conv_layer(41, 1, false, [&] { tail_mma(0, lc); });
                conv_layer(42, 1, false, [&] { tail_mma(1, lc); });
                conv_layer(43, 1, false, [&] { tail_mma(2, lc); });
                tail_mma(3, lc);
            }
            grp_ph ^= 1u;
        }
    } else {
        // ================= epilogue (warps 2..17) =================
        const int ew = warp - 2;               // 0..15
        const int q = warp & 3;                // TMEM lane quadrant
        const int cq = ew >> 2;                // channel quarter
        const int cb = 16 * cq;                // first channel of this thread
        const int et = threadIdx.x - 64;       // 0..511
        const int row = 32 * q + lane;         // row within a tile
        const int pyl = row / RPY, wrow = G::window(row), px = G::px(row);   // tile row = (py - TPY t - 1, window, px)
        const bool interior = !G::spare(row);
        const uint32_t lane_addr = uint32_t(32 * q) << 16;
        uint32_t af_ph = 0;   // bit b: parity of the next completion of b_acc_full[b]
        int vb = 0;           // accumulator buffer of the next unit (the MMA warp's order)
        int nbuilt = 0;             // im2col builds so far (buffer nbuilt & 1)
        if (lane == 0)
            for (int b2 = 0; b2 < 2; ++b2) mbar_arrive_leader(b_drained + 8 * b2);   // both buffers start free
        // wait for the next accumulator unit; returns this lane's TMEM address of its buffer
        auto acc_wait = [&]() -> uint32_t {
            mbar_wait(b_acc_full + 8 * vb, (af_ph >> vb) & 1u);
            af_ph ^= 1u << vb;
            tc_fence_after();
            return tmem + lane_addr + COL_ACC + ACC_COLS * vb;
        };
        auto acc_release = [&] {   // this warp has read the unit's accumulator
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(b_drained + 8 * vb);
            vb ^= 1;
        };
        // a 3x3 unit: columns n = 96 h + 48 (oc' / 16) + 16 dx + oc' % 16 (h = output-channel half, so a
        // thread's 48 columns are contiguous: one x32 and one x16 load); out[r] = y_0[r - 1] + y_1[r]
        // + y_2[r + 1], the row's px -+ 1 neighbours being lanes -+ 1.  Replicate padding: the pad column
        // px = 0 equals px = 1, so the y_0 px = 1 needs is its own (and px = WS takes its own y_2); the pad
        // columns are therefore never stored.  Spare lanes take their own partials (dead data).  One indexed
        // shuffle per partial.
        const int src_l = (px == 1 || !interior) ? lane : lane - 1, src_r = (px == G::WS || !interior) ? lane : lane + 1;
        auto load_dx3 = [&](float (&y)[16]) {
            const uint32_t c = acc_wait() + (cq >> 1) * 96 + (cq & 1) * 48;
            uint32_t v01[32], v2[16];
            TMEM_LD32(c, v01);
            TMEM_LD16(c + 32, v2);
            tmem_wait_ld();
            acc_release();
#pragma unroll
            for (int j = 0; j < 16; ++j)
                y[j] = (__uint_as_float(v01[16 + j]) + __shfl_sync(0xffffffffu, __uint_as_float(v01[j]), src_l)) +
                       __shfl_sync(0xffffffffu, __uint_as_float(v2[j]), src_r);
        };
        const float *head_a = cs;
        uint8_t *idx_tab = reinterpret_cast<uint8_t *>(smem + OFF_MISC + IDX_OFF);
        if constexpr (V != 2) {
            for (int i = et; i < 64 * 96; i += 32 * NEPI) {   // im2col index table (replicate-clamped 9x9 taps)
                const int rp = i / 96, k = i - rp * 96;
                const int cy = min(max((rp >> 3) - 1, 0), 5), cx = min(max((rp & 7) - 1, 0), 5);
                uint8_t v = 255;
                if (k < 81) {
                    const int y = min(max(cy + k / 9 - 4, 0), 5), x = min(max(cx + k % 9 - 4, 0), 5);
                    v = uint8_t(y * 6 + x);
                }
                idx_tab[i] = v;
            }
        }
        const float *up_a = cs + 64 + 192 * NL;
        const float *tail_b = up_a + 64;
        Tracer<INSTR> tr{nullptr, 0};
        uint32_t z_ph = 0;     // parity of the next completion of b_zfull (one per chunk)
        // input tables of a group's windows -> misc: V = 0, 1 the 6x6 q values (fp64 normalise -> fp32);
        // V = 2 the 3 x 12 x 12 X1 values
        auto load_q = [&](int gq) {
            const long long kq = (long long)(2 * gq + int(rank)) * GWPG;
            for (int i = et; i < GWPG * G::QN; i += 32 * NEPI) {
                const int wk = i / G::QN, pp = i - wk * G::QN;
                const Win W = window_of<BATCH>(P, kq + wk, nwin);
                if constexpr (V == 2) {
                    const long long kk = W.valid ? kq + wk : nwin - 1;
                    misc[i] = __half2float(__ushort_as_half(P.x1[kk * 432 + pp]));
                } else {
                    if (BATCH) misc[i] = __ldg(P.qgrid + W.rhs * P.q_stride + (long long)(W.iw + pp / 6) * P.nc + W.jw + pp % 6);
                    else misc[i] = __ldg(P.qgrid + (long long)(W.iw + pp / 6) * P.nc + W.jw + pp % 6);
                }
            }
            epi_bar();
        };
        // head im2col build b (tile b / NBUILD, K part b % NBUILD) from misc (fp16, two buffers: build b + 1
        // is written while build b multiplies)
        auto build_i2c = [&](int b) {
            const int ib = nbuilt & 1;   // the (nbuilt / 2)-th use of buffer ib: wait for the MMAs of the previous one
            if (nbuilt >= 2) mbar_wait(b_i2c_empty + 8 * ib, uint32_t((nbuilt >> 1) - 1) & 1u);
            ++nbuilt;
            const int t = b / G::NBUILD, kq = b - t * G::NBUILD;
            const int r = et & 127, part4 = et >> 7;
            const int py = TPY * t + 1 + (r / RPY);
            if constexpr (V == 2) {
                // K = 64 kq + 16 part4 + e: channel c = k / 81, tap (dy, dx), replicate-clamped in the 12x12 window
                const float *qt = misc + G::window(r) * 432;
                const int pxr = G::px(r);
                uint32_t w[8];
#pragma unroll
                for (int e2 = 0; e2 < 8; ++e2) {
                    float v2[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int k = 64 * kq + 16 * part4 + 2 * e2 + h;
                        float v = 0.f;
                        if (k < 243) {
                            const int c = k / 81, tap = k - 81 * c, dy = tap / 9, dx = tap - 9 * dy;
                            const int y = min(max(py - 1 + dy - 4, 0), 11), x = min(max(pxr - 1 + dx - 4, 0), 11);
                            v = qt[c * 144 + y * 12 + x];
                        }
                        v2[h] = v;
                    }
                    w[e2] = pack_op<true>(v2[0], v2[1]);
                }
                uint8_t *base = i2c + ib * I2C_BYTES + (2 * part4) * (ROWS * 16) + r * 16;
                *reinterpret_cast<uint4 *>(base) = make_uint4(w[0], w[1], w[2], w[3]);
                *reinterpret_cast<uint4 *>(base + ROWS * 16) = make_uint4(w[4], w[5], w[6], w[7]);
            } else {
                (void)kq;
                const int rp = py * 8 + G::px(r);   // padded pixel (py, px)
                const float *qt = misc + G::window(r) * 36;
                const uint2 *ix = reinterpret_cast<const uint2 *>(idx_tab + rp * 96);
#pragma unroll
                for (int kk = 0; kk < HPLANES / 4; ++kk) {
                    const int kc = part4 * (HPLANES / 4) + kk;
                    const uint2 i8 = ix[kc];
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const uint32_t src = e < 2 ? i8.x : i8.y;
                        const uint32_t id0 = (src >> (16 * (e & 1))) & 0xFFu, id1 = (src >> (16 * (e & 1) + 8)) & 0xFFu;
                        w[e] = pack_op<true>(id0 < 36 ? qt[id0] : 0.f, id1 < 36 ? qt[id1] : 0.f);
                    }
                    *reinterpret_cast<uint4 *>(i2c + ib * I2C_BYTES + kc * (ROWS * 16) + r * 16) =
                        make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
            fence_async_smem();
            epi_bar();
            if (et == 0) mbar_arrive_leader(b_i2c_full + 8 * ib);
            tr(12, kq, t);
        };
        // Builds made before the previous group's stitched-pixel epilogue (activation buffer 1 is free once
        // the last up quarter's MMAs completed), so the head MMAs of the next group issue right behind the
        // last tail MMAs and overlap that epilogue.  V = 0, 1: all three (tile 2 reuses buffer 0 once tile 0's
        // head MMAs completed); V = 2: the first two of twelve, the rest interleaved with the head epilogues
        // (a build waits for the MMAs two builds back, which for tile 2 need tile 0's accumulator drained).
        constexpr int PRE = V == 2 ? 2 : T;
        epi_bar();   // the index table is complete
        if (pair < ngp) {
            load_q(pair);
            for (int b = 0; b < PRE; ++b) build_i2c(b);
        }
        for (int gp = pair; gp < ngp; gp += npairs) {
            const int g = 2 * gp + int(rank);
            const long long k0 = (long long)g * GWPG;
            tr.buf = (P.prof && blockIdx.x == 0 && gp == TRACE_GROUP * npairs && lane == 0 &&
                      (warp == 2 || warp == 10)) ? P.prof + (warp == 2 ? 2 : 3) * 4096 : nullptr;
            tr(11, 0, 0);
            const Win Wd = window_of<BATCH>(P, k0 + wrow, nwin);   // this thread's window in the up drains
            // ---- head + body + post epilogues: layer L (head = -1) writes buffer (L + 1) & 1 ----
            for (int L = -1; L < NL; ++L) {
                uint8_t *obuf = act + ((L + 1) & 1) * ACT_BYTES;
                for (int t = 0; t < T; ++t) {
                    if constexpr (V == 2) {
                        if (L < 0 && t == 0)
                            for (int b = PRE; b < 8; ++b) build_i2c(b);
                        if (L < 0 && t == 1)
                            for (int b = 8; b < 12; ++b) build_i2c(b);
                    }
                    tr(6, L + 1, t);
                    // this thread's row of the output buffer (for a residual block's second conv it holds the
                    // block input x_k: the fp16 residual stream, updated in place)
                    uint8_t *dst = obuf + (2 * cq) * ACT_PLANE + (GUARD + (TPY * t + 1) * RPY + row) * 16;
                    float y[16];
                    if (L < 0) {
                        uint32_t v[16];
                        TMEM_LD16(acc_wait() + cb, v);
                        tmem_wait_ld();
                        acc_release();
                        float al[16];
                        lds16(head_a + cb, al);
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            float x = __uint_as_float(v[j]);
                            y[j] = x > 0.f ? x : al[j] * x;
                        }
                        uint32_t sk[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) sk[j] = pack_op<F16>(y[2 * j], y[2 * j + 1]);
                        TMEM_ST8(tmem + lane_addr + COL_SKIP + 32 * t + 8 * cq, sk);
                        tmem_wait_st();
                    } else {
                        const float *sc = cs + 64 + 192 * L;
                        const bool conv1 = (L < NL - 1) && !(L & 1);
                        const bool post = L == NL - 1;
                        float kb[16];   // BN scale is folded into the packed weights; shift remains
                        lds16(sc + 64 + cb, kb);
                        float a[16];
                        load_dx3(a);
                        tr(17, L + 1, t);
                        if (conv1) {
                            float al[16];
                            lds16(sc + 128 + cb, al);
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                float x = a[j] + kb[j];
                                y[j] = x > 0.f ? x : al[j] * x;
                            }
                        } else if (!post) {
                            const uint4 r0 = *reinterpret_cast<const uint4 *>(dst);
                            const uint4 r1 = *reinterpret_cast<const uint4 *>(dst + ACT_PLANE);
                            const uint32_t rv[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                y[2 * e] = op_lo<F16>(rv[e]) + (a[2 * e] + kb[2 * e]);
                                y[2 * e + 1] = op_hi<F16>(rv[e]) + (a[2 * e + 1] + kb[2 * e + 1]);
                            }
                        } else {
                            uint32_t sk[8];
                            TMEM_LD8(tmem + lane_addr + COL_SKIP + 32 * t + 8 * cq, sk);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                y[2 * e] = (a[2 * e] + kb[2 * e]) + op_lo<F16>(sk[e]);
                                y[2 * e + 1] = (a[2 * e + 1] + kb[2 * e + 1]) + op_hi<F16>(sk[e]);
                            }
                        }
                    }
                    uint32_t pk[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) pk[j] = pack_op<F16>(y[2 * j], y[2 * j + 1]);
                    {   // every lane writes its own row (spare rows are dead data, see load_dx3); the first and
                        // last image rows (tiles 0 and T - 1) also write the pad rows py = 0 and WS + 1 (the
                        // kernel rows dy = 0, 2 read them)
                        const uint32_t *sv = pk;
                        const uint4 v0 = make_uint4(sv[0], sv[1], sv[2], sv[3]), v1 = make_uint4(sv[4], sv[5], sv[6], sv[7]);
                        *reinterpret_cast<uint4 *>(dst) = v0;
                        *reinterpret_cast<uint4 *>(dst + ACT_PLANE) = v1;
                        if ((t == 0 && pyl == 0) || (t == T - 1 && pyl == TPY - 1)) {
                            uint8_t *dp = dst + (t == 0 ? -RPY : RPY) * 16;
                            *reinterpret_cast<uint4 *>(dp) = v0;
                            *reinterpret_cast<uint4 *>(dp + ACT_PLANE) = v1;
                        }
                    }
                    if constexpr (INSTR && V == 0) {
                        if (P.dbg && P.dbg_layer == L + 1 && interior) {
                            const long long k = k0 + wrow;
                            if (k < nwin) {
                                const int pp = (2 * t + pyl) * 6 + (px - 1);
#pragma unroll
                                for (int j = 0; j < 16; ++j) P.dbg[(k * 36 + pp) * 64 + cb + j] = y[j];
                            }
                        }
                    }
                    fence_async_smem();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_leader(b_act_ready + 8 * t);
                    tr(7, L + 1, t);
                }
            }
            for (int zc = 0; zc < G::NZC; ++zc) {
                // ---- up quarters: every epilogue warp drains 16 columns (4 shuffled channels x 4 sub-pixels) of
                // its lane quadrant: PReLU, then the quarter goes pixel-shuffled into U, the A operand of the
                // tail MMAs (V = 0, 2: edge windows also spill it for the edge-tail kernel).  U is rewritten
                // for quarter u once the tail MMAs of quarter u - 1 released it. ----
                for (int u = 0; u < UP_QUARTERS; ++u) {
                    float ua[8];   // PReLU alpha of this thread's 8 shuffled channels
#pragma unroll
                    for (int m = 0; m < 8; ++m) ua[m] = up_a[UQ * u + 8 * (cq >> 1) + m];
#pragma unroll
                    for (int t = 0; t < T; ++t) {
                        tr(8, u, t);
                        float a[16];
                        load_dx3(a);
                        if (u > 0 && t == 0) mbar_wait(b_ubuf_free, uint32_t(u - 1) & 1u);
                        tr(9, u, t);
                        if (interior) {
                            // column j -> shuffled channel 16 u + 8 (cq >> 1) + j / 2, sub-pixel (cq & 1, j & 1)
                            const int py = TPY * t + 1 + pyl, ii = cq & 1;
                            float y[16];
#pragma unroll
                            for (int j = 0; j < 16; ++j) {
                                const float x = a[j];
                                y[j] = x > 0.f ? x : ua[j >> 1] * x;
                            }
                            uint8_t *Ub = ubuf + (cq >> 1) * G::U_PLANE;
                            const int Y = 2 * (py - 1) + ii, X0 = 2 * (px - 1);
                            uint4 val[2];
#pragma unroll
                            for (int jj = 0; jj < 2; ++jj)
                                val[jj] = make_uint4(pack_op<F16>(y[jj], y[2 + jj]), pack_op<F16>(y[4 + jj], y[6 + jj]),
                                                     pack_op<F16>(y[8 + jj], y[10 + jj]), pack_op<F16>(y[12 + jj], y[14 + jj]));
                            auto put = [&](int urow) {   // pixels (Y, X0), (Y, X0 + 1) of U rows urow, urow + 1
                                uint4 *d = reinterpret_cast<uint4 *>(Ub + urow * 16);
                                d[0] = val[0];
                                d[1] = val[1];
                            };
                            if constexpr (V == 0) {
                                put(Y * G::UROWS_Y + 12 * wrow + X0);
                            } else if constexpr (V == 1) {
                                // chunk rows 4 zc - 4 .. 4 zc + 7, replicate-clamped at the window edge
                                const int Yu = Y - 4 * zc + 4;
                                if (Yu >= 0 && Yu < 12) put(Yu * G::UROWS_Y + 12 * wrow + X0);
                                if (zc == 0 && Y == 0)
#pragma unroll
                                    for (int e = 0; e < 4; ++e) put(e * G::UROWS_Y + 12 * wrow + X0);
                                if (zc == 2 && Y == 11)
#pragma unroll
                                    for (int e = 8; e < 12; ++e) put(e * G::UROWS_Y + 12 * wrow + X0);
                            } else {
                                if (Y >= 4 && Y < 20 && X0 >= 4 && X0 < 20) put((Y - 4) * G::UROWS_Y + 16 * wrow + X0 - 4);
                            }
                            if constexpr (V != 1) {
                                const Win &W = Wd;
                                const int pp = (py - 1) * G::WS + (px - 1);
                                if (W.valid && W.edge) {   // spill in the up conv's channel order (edge-tail kernels)
                                    const size_t ei = BATCH ? size_t(W.rhs) * edge_count(P.npos) + edge_index(W.wi, W.wj, P.npos)
                                                            : size_t(edge_index(W.wi, W.wj, P.npos));
                                    uint32_t *dst = reinterpret_cast<uint32_t *>(
                                        P.edge_u + (ei * (G::WS * G::WS) + pp) * 256 + 64 * u + 32 * (cq >> 1) + 2 * ii);
#pragma unroll
                                    for (int m = 0; m < 8; ++m) dst[2 * m] = pack_op<F16>(y[2 * m], y[2 * m + 1]);
                                }
                            }
                            if constexpr (INSTR && V == 0) {
                                const long long k = k0 + wrow;
                                if (P.dbg && P.dbg_layer == NL + 1 && Wd.valid) {
#pragma unroll
                                    for (int j = 0; j < 16; ++j) {
                                        const int c = UQ * u + 8 * (cq >> 1) + (j >> 1), X = X0 + (j & 1);
                                        P.dbg[(k * 144 + Y * 12 + X) * 64 + c] = y[j];
                                    }
                                }
                            }
                        }
                        tr(10, u, t);
                    }
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_leader(b_ubuf_full);
                }
                // ---- next group's input tables and head im2col (buffer 1: the up MMAs are complete) ----
                if (zc == G::NZC - 1 && gp + npairs < ngp) {
                    load_q(gp + npairs);
                    tr(11, 1, 0);
                    for (int b = 0; b < PRE; ++b) build_i2c(b);
                }
                if constexpr (V == 0) {
                    // ---- stitched pixels: warps of channel quarter cq = j finish Z tile j (kept fine row y = 4 + j).
                    // Lane (quadrant q, lane) holds Z row 32 q + lane = 12 w + X; its 27 partials go to shared
                    // memory (buffer 0: U and the tail weights are consumed once the last Z tile's MMAs completed),
                    // then the kept pixel (w, X' = 4..7) sums Z[12 w + X' + dx - 4][3 dx + o] over dx, adds the bias,
                    // applies s tanh(./s), the channel mean and the denormalisation, straight into the fine grid.
                    // Edge windows are k_tail_edge's. ----
                    const int j = cq;
                    mbar_wait(b_zfull + 8 * (G::ZT - 1), z_ph);   // every Z tile done: buffer 0 is free
                    tr(13, 0, j);
                    tc_fence_after();
                    uint32_t z0[16], z1[16];
                    TMEM_LD16(tmem + lane_addr + COL_Z + 32 * j, z0);
                    TMEM_LD16(tmem + lane_addr + COL_Z + 32 * j + 16, z1);
                    tmem_wait_ld();
                    float *zs = reinterpret_cast<float *>(ubuf) + j * (ROWS * ZS_STRIDE);
#pragma unroll
                    for (int n = 0; n < 27; ++n) zs[row * ZS_STRIDE + n] = __uint_as_float(n < 16 ? z0[n] : z1[n - 16]);
                    asm volatile("bar.sync %0, 128;" ::"r"(2 + j) : "memory");   // the 4 warps of Z tile j
                    if (row < GWPG * 4) {
                        const int w = row >> 2, X = 4 + (row & 3);
                        float pre[3] = {tail_b[0], tail_b[1], tail_b[2]};
#pragma unroll
                        for (int dx = 0; dx < 9; ++dx) {
                            const float *zr = zs + (12 * w + X + dx - 4) * ZS_STRIDE + 3 * dx;
#pragma unroll
                            for (int o = 0; o < 3; ++o) pre[o] += zr[o];
                        }
                        const Win W = window_of<BATCH>(P, k0 + w, nwin);
                        if (W.valid && !W.edge) {
                            double m = 0.0;
#pragma unroll
                            for (int o = 0; o < 3; ++o) m += double(P.tanh_s * tanhf(pre[o] / P.tanh_s));
                            m = m / 3.0;
                            // sign(q) 10^(log_lo + |q| span) in fp32 (exp2f; <= 3e-6 relative, far inside the fp16
                            // operands' error), off the critical path's fp64 pow
                            const float e = (float(P.log_lo) + float(fabs(m)) * float(P.span)) * 3.32192809488736f;
                            const double mag = double(exp2f(e));
                            P.fine[(BATCH ? W.rhs * P.fine_stride : 0) + (long long)(2 * W.iw + 4 + j) * P.nf + 2 * W.jw + X] = m > 0.0 ? mag : (m < 0.0 ? -mag : 0.0);
                        }
                    }
                    tr(14, 0, j);
                } else if constexpr (V == 1) {
                    // ---- full output rows 4 zc + j of every window -> X1 (fp16): the dx sum (replicate-clamped at
                    // the window edge) through shared memory in U, two Z tiles at a time ----
                    const int j = cq;
                    mbar_wait(b_zfull + 8 * (G::ZT - 1), z_ph);
                    tc_fence_after();
                    uint32_t z0[16], z1[16];
                    TMEM_LD16(tmem + lane_addr + COL_Z + 32 * j, z0);
                    TMEM_LD16(tmem + lane_addr + COL_Z + 32 * j + 16, z1);
                    tmem_wait_ld();
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        if ((j >> 1) == h) {
                            float *zs = reinterpret_cast<float *>(ubuf) + (j & 1) * (ROWS * ZS_STRIDE);
#pragma unroll
                            for (int n = 0; n < 27; ++n)
                                zs[row * ZS_STRIDE + n] = __uint_as_float(n < 16 ? z0[n] : z1[n - 16]);
                            asm volatile("bar.sync %0, 128;" ::"r"(2 + j) : "memory");
                            if (row < GWPG * 12) {
                                const int w = row / 12, X = row - 12 * w, Y = 4 * zc + j;
                                float pre[3] = {tail_b[0], tail_b[1], tail_b[2]};
#pragma unroll
                                for (int dx = 0; dx < 9; ++dx) {
                                    const int xs = min(max(X + dx - 4, 0), 11);
                                    const float *zr = zs + (12 * w + xs) * ZS_STRIDE + 3 * dx;
#pragma unroll
                                    for (int o = 0; o < 3; ++o) pre[o] += zr[o];
                                }
                                const long long k = k0 + w;
                                if (k < nwin) {
#pragma unroll
                                    for (int o = 0; o < 3; ++o)
                                        P.x1[(k * 3 + o) * 144 + Y * 12 + X] =
                                            __half_as_ushort(__float2half_rn(P.tanh_s * tanhf(pre[o] / P.tanh_s)));
                                }
                            }
                        }
                        epi_bar();   // the scratch half is read before the next half (or the next chunk's U) reuses it
                    }
                } else {
                    // ---- stitched pixels (V = 2): warps of channel quarters 0, 1 finish Z tile j = cq (fine rows
                    // 8 + 4 j + q).  Lane holds Z row (window lane / 16, X = 4 + lane % 16); the kept X = 8..15 sums
                    // Z[X + dx - 4][3 dx + o] over dx by lane shuffles. ----
                    if (cq < G::ZT) {
                        const int j = cq;
                        mbar_wait(b_zfull + 8 * j, z_ph);
                        tc_fence_after();
                        uint32_t z0[16], z1[16];
                        TMEM_LD16(tmem + lane_addr + COL_Z + 32 * j, z0);
                        TMEM_LD16(tmem + lane_addr + COL_Z + 32 * j + 16, z1);
                        tmem_wait_ld();
                        const int Xp = lane & 15;
                        float pre[3] = {tail_b[0], tail_b[1], tail_b[2]};
#pragma unroll
                        for (int dx = 0; dx < 9; ++dx) {
                            const int src = (lane & 16) | ((Xp + dx - 4) & 15);
#pragma unroll
                            for (int o = 0; o < 3; ++o) {
                                const int n = 3 * dx + o;
                                pre[o] += __shfl_sync(0xffffffffu, __uint_as_float(n < 16 ? z0[n] : z1[n - 16]), src);
                            }
                        }
                        if (Xp >= 4 && Xp < 12) {
                            const Win W = window_of<BATCH>(P, k0 + (lane >> 4), nwin);
                            if (W.valid && !W.edge) {
                                double m = 0.0;
#pragma unroll
                                for (int o = 0; o < 3; ++o) m += double(P.tanh_s * tanhf(pre[o] / P.tanh_s));
                                m = m / 3.0;
                                const float e = (float(P.log_lo) + float(fabs(m)) * float(P.span)) * 3.32192809488736f;
                                const double mag = double(exp2f(e));
                                P.fine[(long long)(4 * W.iw + 8 + 4 * j + q) * P.nf + 4 * W.jw + 4 + Xp] =
                                    m > 0.0 ? mag : (m < 0.0 ? -mag : 0.0);
                            }
                        }
                    }
                }
                z_ph ^= 1u;
            }
            tc_fence_before();
            tr(15, 0, 0);
            epi_bar();
            tc_fence_after();
            tr(15, 1, 0);
        }
    }
    // teardown
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// q = clip((log10|c - shift| - log_lo)/span, 0, 1) * sign (rounded to fp16 in the head im2col)
__global__ void k_normalize(const double *__restrict__ c, const double *shift, int nc, double log_lo, double span,
                            float *__restrict__ q) {
    const double sh = shift ? *shift : 0.0;
    const long long total = (long long)nc * nc;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
        q[i] = float(normalize_q(c[i] - sh, log_lo, span));
}

// batched normalise: grids cs[0..B) (device pointer array) -> q[r][nc][nc]
__global__ void k_normalize_batch(const double *const *cs, int B, int nc, double log_lo, double span,
                                  float *__restrict__ q) {
    const long long per = (long long)nc * nc, total = per * B;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / per;
        q[i] = float(normalize_q(cs[r][i - r * per], log_lo, span));
    }
}

// Tail of the edge windows (kept band touching the grid edge), exact fp32 with
// the reference's replicate clamping (srmodel.py:285-289) on the 12x12 field.
// Register-blocked and persistent: the fp32 tail weights are staged once per CTA as [c][dy][o][dx (12)], each
// edge window's up-conv output as a replicate-padded [c][20][20] fp32 image (so every 9 x 9 tap
// reads in bounds and 4 consecutive pixels' taps are one 12-float row); thread = (2 channels,
// a strip of 4 kept pixels) accumulates 4 px x 3 outputs, 108 FMAs per 21 16-byte loads; the
// 32 channel groups are reduced through shared memory.
constexpr int TE_THREADS = 256, TE_PAD = 20, TE_WROW = 12;
constexpr int TE_W_FLOATS = 64 * 9 * 3 * TE_WROW;        // 20736
constexpr int TE_U_FLOATS = 64 * TE_PAD * TE_PAD;        // 25600
constexpr int TE_R_FLOATS = 32 * 8 * 12;                 // partial sums [group][strip slot][4 px x 3 o]
constexpr size_t TE_SMEM = sizeof(float) * (TE_W_FLOATS + TE_U_FLOATS + TE_R_FLOATS);

template <bool F16>
__global__ void __launch_bounds__(TE_THREADS) k_tail_edge(Params P, int nedge) {
    extern __shared__ __align__(16) float te[];
    float *Wt = te, *U = te + TE_W_FLOATS, *red = U + TE_U_FLOATS;
    const int tid = threadIdx.x;
    const BlobLayout BL = blob_layout((P.nl - 1) / 2);
    const float *w = reinterpret_cast<const float *>(P.blob + BL.tail_f32);   // [3][64][81]
    const float *bias = reinterpret_cast<const float *>(P.blob + BL.consts) + 64 + 192 * P.nl + 64;
    for (int i = tid; i < TE_W_FLOATS; i += TE_THREADS) {
        const int dx = i % TE_WROW, o = (i / TE_WROW) % 3, dy = (i / (3 * TE_WROW)) % 9, c = i / (27 * TE_WROW);
        Wt[i] = dx < 9 ? __ldg(w + (o * 64 + c) * 81 + dy * 9 + dx) : 0.f;
    }
    const int g = tid >> 3, slot = tid & 7;   // channels 2g, 2g + 1; strip slot
    const int n = P.npos, last = n - 1;
    const int ne1 = edge_count(n);
    if (P.rhs_count) nedge = *P.rhs_count * ne1;   // batched: the listed grids' edge windows
    for (int eg = blockIdx.x; eg < nedge; eg += gridDim.x) {
        const int gs = eg / ne1, e = eg - gs * ne1, rhs = P.rhs_list ? P.rhs_list[gs] : 0;
        double *fine = P.fine + rhs * P.fine_stride;
        int wi, wj;
        if (n == 1) { wi = 0; wj = 0; }
        else if (e < n) { wi = 0; wj = e; }
        else if (e < 2 * n) { wi = n - 1; wj = e - n; }
        else { wi = 1 + (e - 2 * n) / 2; wj = ((e - 2 * n) & 1) ? n - 1 : 0; }
        __syncthreads();   // previous window's U / partials consumed (and the weights staged)
        const uint16_t *src = P.edge_u + (size_t(rhs) * ne1 + e) * 36 * 256;
        for (int i = tid; i < 36 * 256; i += TE_THREADS) {
            const int pp = i >> 8, oc = i & 255, c = oc >> 2, ii = (oc >> 1) & 1, jj = oc & 1;
            const int Y = 2 * (pp / 6) + ii, X = 2 * (pp % 6) + jj;
            U[(c * TE_PAD + Y + 4) * TE_PAD + X + 4] = op_lo<F16>(uint32_t(src[i]));
        }
        __syncthreads();
        // replicate padding: rows first (interior columns), then whole columns
        for (int i = tid; i < 64 * 8 * 12; i += TE_THREADS) {
            const int c = i / 96, r = (i / 12) % 8, x = i % 12;
            const int Y = r < 4 ? r : 16 + (r - 4), ys = r < 4 ? 4 : 15;
            U[(c * TE_PAD + Y) * TE_PAD + x + 4] = U[(c * TE_PAD + ys) * TE_PAD + x + 4];
        }
        __syncthreads();
        for (int i = tid; i < 64 * TE_PAD * 8; i += TE_THREADS) {
            const int c = i / (TE_PAD * 8), Y = (i / 8) % TE_PAD, k = i % 8;
            const int X = k < 4 ? k : 16 + (k - 4), xs = k < 4 ? 4 : 15;
            U[(c * TE_PAD + Y) * TE_PAD + X] = U[(c * TE_PAD + Y) * TE_PAD + xs];
        }
        __syncthreads();
        const int lo_i = wi == 0 ? 0 : 2, hi_i = wi == last ? 6 : 4, lo_j = wj == 0 ? 0 : 2, hi_j = wj == last ? 6 : 4;
        const int wk = 2 * (hi_j - lo_j), nstrip = 2 * (hi_i - lo_i) * (wk / 4);   // <= 36 strips of 4 px
        for (int s0 = 0; s0 < nstrip; s0 += 8) {
            const int sidx = s0 + slot;
            float acc[4][3];
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int o = 0; o < 3; ++o) acc[k][o] = 0.f;
            if (sidx < nstrip) {
                const int fy = 2 * lo_i + sidx / (wk / 4), fx0 = 2 * lo_j + 4 * (sidx % (wk / 4));
#pragma unroll 1
                for (int cc = 0; cc < 2; ++cc) {
                    const int c = 2 * g + cc;
#pragma unroll 1
                    for (int dy = 0; dy < 9; ++dy) {
                        float u[12], wv[3][12];
                        const float4 *ur = reinterpret_cast<const float4 *>(U + (c * TE_PAD + fy + dy) * TE_PAD + fx0);
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            const float4 t4 = ur[q];
                            u[4 * q] = t4.x; u[4 * q + 1] = t4.y; u[4 * q + 2] = t4.z; u[4 * q + 3] = t4.w;
                        }
                        const float4 *wr = reinterpret_cast<const float4 *>(Wt + ((c * 9 + dy) * 3) * TE_WROW);
#pragma unroll
                        for (int o = 0; o < 3; ++o)
#pragma unroll
                            for (int q = 0; q < 3; ++q) {
                                const float4 t4 = wr[o * 3 + q];
                                wv[o][4 * q] = t4.x; wv[o][4 * q + 1] = t4.y; wv[o][4 * q + 2] = t4.z; wv[o][4 * q + 3] = t4.w;
                            }
#pragma unroll
                        for (int dx = 0; dx < 9; ++dx)
#pragma unroll
                            for (int k = 0; k < 4; ++k)
#pragma unroll
                                for (int o = 0; o < 3; ++o) acc[k][o] = fmaf(u[k + dx], wv[o][dx], acc[k][o]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int o = 0; o < 3; ++o) red[(g * 8 + slot) * 12 + k * 3 + o] = acc[k][o];
            __syncthreads();
            if (tid < 8 * 12) {
                const int sl = tid / 12, ko = tid % 12, sidx2 = s0 + sl;
                float sum = 0.f;
                for (int gg = 0; gg < 32; ++gg) sum += red[(gg * 8 + sl) * 12 + ko];
                red[32 * 8 * 12 - 8 * 12 + tid] = sum;   // reuse the last group's row for the totals
                (void)sidx2;
            }
            __syncthreads();
            if (tid < 8 * 4) {
                const int sl = tid >> 2, k = tid & 3, sidx2 = s0 + sl;
                if (sidx2 < nstrip) {
                    const int fy = 2 * lo_i + sidx2 / (wk / 4), fx = 2 * lo_j + 4 * (sidx2 % (wk / 4)) + k;
                    double m = 0.0;
#pragma unroll
                    for (int o = 0; o < 3; ++o) {
                        const float pre = red[32 * 8 * 12 - 8 * 12 + sl * 12 + k * 3 + o] + __ldg(bias + o);
                        m += double(P.tanh_s * tanhf(pre / P.tanh_s));
                    }
                    m = m / 3.0;
                    fine[(long long)(2 * (2 * wi) + fy) * P.nf + 2 * (2 * wj) + fx] = denormalize_q(m, P.log_lo, P.span);
                }
            }
            __syncthreads();
        }
    }
}

// Tail of the edge windows of a ratio-4 pass's second application (V = 2), exact fp32 with the reference's
// replicate clamping on the 24x24 field: one CTA per edge window, one thread per kept fine pixel (the band
// touching the grid edge: at most 16 x 16), the up-conv output staged 16 channels at a time as replicate-
// padded [16][32][32] fp32 images, the chunk's tail weights as [16][3][81].
constexpr int TE4_THREADS = 256, TE4_PAD = 32, TE4_CH = 16;
constexpr size_t TE4_SMEM = sizeof(float) * (TE4_CH * TE4_PAD * TE4_PAD + TE4_CH * 3 * 81);

template <bool F16>
__global__ void __launch_bounds__(TE4_THREADS) k_tail_edge4(Params P, int nedge) {
    extern __shared__ __align__(16) float te4[];
    float *U = te4, *Wc = te4 + TE4_CH * TE4_PAD * TE4_PAD;
    const int tid = threadIdx.x;
    const BlobLayout BL = blob_layout((P.nl - 1) / 2);
    const float *w = reinterpret_cast<const float *>(P.blob + BL.tail_f32);   // [3][64][81]
    const float *bias = reinterpret_cast<const float *>(P.blob + BL.consts) + 64 + 192 * P.nl + 64;
    const int n = P.npos, last = n - 1;
    for (int e = blockIdx.x; e < nedge; e += gridDim.x) {
        int wi, wj;
        if (n == 1) { wi = 0; wj = 0; }
        else if (e < n) { wi = 0; wj = e; }
        else if (e < 2 * n) { wi = n - 1; wj = e - n; }
        else { wi = 1 + (e - 2 * n) / 2; wj = ((e - 2 * n) & 1) ? n - 1 : 0; }
        const int lo_i = wi == 0 ? 0 : 8, hi_i = wi == last ? 24 : 16, lo_j = wj == 0 ? 0 : 8, hi_j = wj == last ? 24 : 16;
        const int wk = hi_j - lo_j, npx = (hi_i - lo_i) * wk;   // <= 16 x 16, or 24 x 24 for a single window
        const uint16_t *src = P.edge_u + size_t(e) * 144 * 256;
#pragma unroll 1
        for (int p0 = 0; p0 < npx; p0 += TE4_THREADS) {
            const int pix = p0 + tid;
            const int fy = pix < npx ? lo_i + pix / wk : lo_i, fx = pix < npx ? lo_j + pix % wk : lo_j;
            float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += TE4_CH) {
                __syncthreads();   // the previous chunk / window is consumed
                for (int i = tid; i < TE4_CH * TE4_PAD * TE4_PAD; i += TE4_THREADS) {
                    const int c = i / (TE4_PAD * TE4_PAD), yp = (i / TE4_PAD) % TE4_PAD, xp = i % TE4_PAD;
                    const int Y = min(max(yp - 4, 0), 23), X = min(max(xp - 4, 0), 23);
                    const int oc = 4 * (c0 + c) + 2 * (Y & 1) + (X & 1);
                    U[i] = op_lo<F16>(uint32_t(src[((Y >> 1) * 12 + (X >> 1)) * 256 + oc]));
                }
                for (int i = tid; i < TE4_CH * 3 * 81; i += TE4_THREADS) {
                    const int c = i / 243, o = (i / 81) % 3, tap = i % 81;
                    Wc[i] = __ldg(w + (o * 64 + c0 + c) * 81 + tap);
                }
                __syncthreads();
                if (pix < npx) {
#pragma unroll 1
                    for (int c = 0; c < TE4_CH; ++c)
#pragma unroll 1
                        for (int dy = 0; dy < 9; ++dy) {
                            const float *ur = U + (c * TE4_PAD + fy + dy) * TE4_PAD + fx;
                            const float *wr = Wc + c * 243 + dy * 9;
#pragma unroll
                            for (int dx = 0; dx < 9; ++dx) {
                                const float u = ur[dx];
#pragma unroll
                                for (int o = 0; o < 3; ++o) acc[o] = fmaf(u, wr[o * 81 + dx], acc[o]);
                            }
                        }
                }
            }
            if (pix < npx) {
                double m = 0.0;
#pragma unroll
                for (int o = 0; o < 3; ++o) {
                    const float pre = acc[o] + __ldg(bias + o);
                    m += double(P.tanh_s * tanhf(pre / P.tanh_s));
                }
                m = m / 3.0;
                P.fine[(long long)(4 * (2 * wi) + fy) * P.nf + 4 * (2 * wj) + fx] = denormalize_q(m, P.log_lo, P.span);
            }
        }
    }
}

}  // namespace tc

// ---------------------------------------------------------------------------
// host side

static inline uint16_t f2h(float f) {
    __half h = __float2half_rn(f);
    uint16_t u;
    std::memcpy(&u, &h, 2);
    return u;
}
static inline uint16_t f2bf(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    uint32_t r = u + 0x7FFFu + ((u >> 16) & 1u);   // round to nearest even
    return uint16_t(r >> 16);
}

// Pack the MGSR1 tensors (host f32, expected_tensor_shapes order) into the
// kernel's weight blob: UMMA core-matrix layout (K-major, 8-element planes).
int tc_pack_weights(mgsr_gen *g, const float *const *t) {
    using namespace tc;
    const int B = g->blocks;
    BlobLayout BL = blob_layout(B);
    std::vector<uint8_t> blob(BL.total, 0);
    // head B: 12 planes x 64 oc x 8 fp16 (3 identical input channels folded), split in two 32-oc halves
    {
        uint16_t *hb = reinterpret_cast<uint16_t *>(blob.data() + BL.head_b);
        const float *w = t[0];
        for (int kc = 0; kc < HPLANES; ++kc)
            for (int oc = 0; oc < 64; ++oc)
                for (int e = 0; e < 8; ++e) {
                    int k = 8 * kc + e;
                    float v = 0.f;
                    if (k < 81) {
                        int dy = k / 9, dx = k % 9;
                        double s = 0.0;
                        for (int c = 0; c < 3; ++c) s += double(w[((oc * 3 + c) * 9 + dy) * 9 + dx]);
                        v = float(s);
                    }
                    hb[(((oc >> 5) * HPLANES + kc) * 32 + (oc & 31)) * 8 + e] = f2h(v);   // [half][kc][32 oc][8] fp16
                }
    }
    // ratio-4 second-application head (3 distinct input channels): [half][kc 32][32 oc][8] fp16, k = 81 c + tap
    {
        uint16_t *hb = reinterpret_cast<uint16_t *>(blob.data() + BL.head4);
        const float *w = t[0];
        for (int kc = 0; kc < 32; ++kc)
            for (int oc = 0; oc < 64; ++oc)
                for (int e = 0; e < 8; ++e) {
                    const int k = 8 * kc + e;
                    float v = 0.f;
                    if (k < 243) {
                        const int c = k / 81, tap = k % 81;
                        v = w[(oc * 3 + c) * 81 + tap];
                    }
                    hb[(((oc >> 5) * 32 + kc) * 32 + (oc & 31)) * 8 + e] = f2h(v);
                }
    }
    auto conv_index = [&](int L) -> int {   // tensor index of body layer L's conv weight
        if (L == 2 * B) return 2 + 11 * B;
        return 2 + 11 * (L / 2) + ((L & 1) ? 6 : 0);
    };
    // BN(conv(x)) = conv(x; W * k) + (beta - mean * k), k = gamma / sqrt(var + 1e-5): the scale is
    // folded into the packed weights (per output channel), the shift stays in the epilogue.
    auto bn_scale = [&](int gi, int oc) { return double(t[gi][oc]) / std::sqrt(double(t[gi + 3][oc]) + 1e-5); };
    // kernel row dy of a 3x3 64 -> 64 conv (output channels oc0..oc0 + 63): [half][ng 12][kc 8][8 rows][8 ic], so
    // a CTA's unit is one K-major B operand of N = 96 rows with 8-row groups 1 KB apart; row n' = 48 (oc' / 16)
    // + 16 dx + oc' % 16 (oc' = oc % 32), so an epilogue thread's 16 channels x 3 dx are adjacent columns
    // perm: the up conv's column order (up_col_channel); identity for the body layers
    auto pack_row = [&](uint16_t *dst, const float *w, int oc0, int dy, int bn_gi, bool perm) {
        uint16_t *dst16 = reinterpret_cast<uint16_t *>(reinterpret_cast<uint8_t *>(dst) + BL.fmt_stride);
        for (int dx = 0; dx < 3; ++dx)
            for (int kc = 0; kc < 8; ++kc)
                for (int oc = 0; oc < 64; ++oc) {
                    const int wc = oc0 + (perm ? up_col_channel(oc) : oc);
                    const double k = bn_gi >= 0 ? bn_scale(bn_gi, wc) : 1.0;
                    for (int e = 0; e < 8; ++e) {
                        int ic = 8 * kc + e;
                        const float v = float(double(w[((wc * 64 + ic) * 3 + dy) * 3 + dx]) * k);
                        const int nr = 48 * ((oc & 31) >> 4) + 16 * dx + (oc & 15);
                        const int o = ((((oc >> 5) * 12 + (nr >> 3)) * 8 + kc) * 8 + (nr & 7)) * 8 + e;
                        dst[o] = f2bf(v);
                        dst16[o] = f2h(v);
                    }
                }
    };
    const int ip = 2 + 11 * B;   // post conv index
    auto bn_index = [&](int L) -> int {   // tensor index of body layer L's BN gamma
        if (L == 2 * B) return ip + 1;
        return 2 + 11 * (L / 2) + ((L & 1) ? 7 : 1);
    };
    for (int L = 0; L < BL.nl; ++L)
        for (int dy = 0; dy < 3; ++dy)
            pack_row(reinterpret_cast<uint16_t *>(blob.data() + BL.body + (size_t(L) * 3 + dy) * ROW_BYTES),
                     t[conv_index(L)], 0, dy, bn_index(L), false);
    for (int u = 0; u < UP_QUARTERS; ++u)
        for (int dy = 0; dy < 3; ++dy)
            pack_row(reinterpret_cast<uint16_t *>(blob.data() + BL.up + (size_t(u) * 3 + dy) * ROW_BYTES),
                     t[ip + 5], 64 * u, dy, -1, true);
    {
        // tail B operand: per quarter u and CTA half h, [dy 9][k 2][16 n][8] with n = 16 h + n' = 3 dx + o
        // (27 of 32 used) and k = shuffled channel 16 u + 8 k + e
        const float *w = t[ip + 7];   // tail.conv.weight 3 x 64 x 9 x 9
        uint16_t *dst = reinterpret_cast<uint16_t *>(blob.data() + BL.tail);
        uint16_t *dst16 = reinterpret_cast<uint16_t *>(blob.data() + BL.fmt_stride + BL.tail);
        for (int u = 0; u < UP_QUARTERS; ++u)
            for (int h = 0; h < 2; ++h)
                for (int dy = 0; dy < 9; ++dy)
                    for (int kc = 0; kc < 2; ++kc)
                        for (int nl = 0; nl < 16; ++nl)
                            for (int e = 0; e < 8; ++e) {
                                const int n = 16 * h + nl, dx = n / 3, o = n % 3, c = UQ * u + 8 * kc + e;
                                const float v = n < 27 ? w[((o * 64 + c) * 9 + dy) * 9 + dx] : 0.f;
                                const size_t i = (((size_t(u * 2 + h) * 9 + dy) * 2 + kc) * 16 + nl) * 8 + e;
                                dst[i] = f2bf(v);
                                dst16[i] = f2h(v);
                            }
        float *wf = reinterpret_cast<float *>(blob.data() + BL.tail_f32);
        std::memcpy(wf, w, sizeof(float) * 3 * 64 * 81);
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
    const size_t stride = (BL.total + 1023) & ~size_t(1023);
    MGSR_CUDA_TRY(cudaMalloc(&g->tc_blob, stride * BLOB_COPIES));
    for (int c = 0; c < BLOB_COPIES; ++c)
        MGSR_CUDA_TRY(cudaMemcpy(static_cast<uint8_t *>(g->tc_blob) + c * stride, blob.data(), BL.total,
                                 cudaMemcpyHostToDevice));
    g->tc_bytes = stride * BLOB_COPIES;
    return MGSR_OK;
}

// workspace: [edge-window up outputs (fp16)][normalised coarse grid q (fp32)]
static size_t tc_edge_bytes(int64_t nc) {
    const int npos = int(nc / 2 - 2);
    const size_t b = npos >= 1 ? size_t(tc::edge_count(npos)) * 36 * 256 * sizeof(uint16_t) : 0;
    return (b + 255) & ~size_t(255);
}
size_t tc_workspace_bytes(int64_t nc) { return tc_edge_bytes(nc) + sizeof(float) * size_t(nc) * nc + 256; }

// ratio-4 pass workspace: [edge-window up outputs of the second application (144 px)][X1 (fp16)][q (fp32)]
static size_t tc4_edge_bytes(int64_t nc) {
    const int npos = int(nc / 2 - 2);
    const size_t b = npos >= 1 ? size_t(tc::edge_count(npos)) * 144 * 256 * sizeof(uint16_t) : 0;
    return (b + 255) & ~size_t(255);
}
static size_t tc4_x1_bytes(int64_t nc) {
    const int64_t npos = nc / 2 - 2;
    return (size_t(npos > 0 ? npos * npos : 0) * 432 * sizeof(uint16_t) + 255) & ~size_t(255);
}
size_t tc4_workspace_bytes(int64_t nc) {
    return tc4_edge_bytes(nc) + tc4_x1_bytes(nc) + sizeof(float) * size_t(nc) * nc + 256;
}

// one persistent k_gen_tc<F16, INSTR, V> launch: CTA pairs (clusters of 2), one CTA per SM, as many pairs as
// can be co-resident
template <int V, bool BATCH = false>
static int launch_gen(tc::Params &P, bool f16, bool instr, cudaStream_t st) {
    using namespace tc;
    const int smem = smem_bytes(P.nl);
    if (smem > 232448) { set_error("generator too deep for the tensor-core kernel's shared memory"); return MGSR_E_UNSUPPORTED; }
    int dev = 0, nsm = 0;
    MGSR_CUDA_TRY(cudaGetDevice(&dev));
    MGSR_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    auto kern = f16 ? (instr ? k_gen_tc<true, true, V, BATCH> : k_gen_tc<true, false, V, BATCH>)
                    : (instr ? k_gen_tc<false, true, V, BATCH> : k_gen_tc<false, false, V, BATCH>);
    MGSR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    P.ngroups = int((P.nwin + Geo<V>::WPG - 1) / Geo<V>::WPG);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int ngp = (P.ngroups + 1) / 2;
    static int max_pairs[2] = {0, 0};
    int &mp = max_pairs[f16 ? 1 : 0];
    if (mp == 0) {
        cfg.gridDim = dim3(2 * (nsm / 2));
        int ncl = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
        mp = (e == cudaSuccess && ncl > 0) ? ncl : nsm / 2;
    }
    const int pairs = ngp < mp ? ngp : mp;
    cfg.gridDim = dim3(2 * pairs);
    MGSR_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, P));
    return MGSR_OK;
}

static void fill_params(tc::Params &P, const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo,
                        double span, double *fine, int ratio, int f16) {
    using namespace tc;
    P.c = c;
    P.c_shift = c_shift;
    P.nc = nc;
    P.npos = nc / 2 - 2;
    P.nwin = (long long)P.npos * P.npos;
    P.log_lo = log_lo;
    P.span = span;
    P.fine = fine;
    P.nf = ratio * nc;
    P.blob = static_cast<const uint8_t *>(g->tc_blob);
    P.nl = 2 * g->blocks + 1;
    P.tanh_s = float(g->tanh_scale);
    P.wfmt = f16 ? blob_layout(g->blocks).fmt_stride : 0;
}

int launch_sr_pass_tc_dbg(const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo,
                          double span, double *fine, void *ws, size_t ws_bytes, float *dbg, int dbg_layer,
                          cudaStream_t st, unsigned long long *prof = nullptr, int f16 = 0) {
    using namespace tc;
    if (!g->tc_blob) { set_error("tensor-core weights not packed"); return MGSR_E_UNSUPPORTED; }
    if (ws_bytes < tc_workspace_bytes(nc)) { set_error("tensor-core workspace too small"); return MGSR_E_WORKSPACE; }
    Params P{};
    fill_params(P, g, c, c_shift, nc, log_lo, span, fine, 2, f16);
    P.edge_u = static_cast<uint16_t *>(ws);
    float *qgrid = reinterpret_cast<float *>(static_cast<char *>(ws) + tc_edge_bytes(nc));
    P.qgrid = qgrid;
    P.dbg = dbg;
    P.dbg_layer = dbg_layer;
    P.prof = prof;
    int nsm = 0, dev = 0;
    MGSR_CUDA_TRY(cudaGetDevice(&dev));
    MGSR_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    k_normalize<<<grid_for((long long)nc * nc, 256), 256, 0, st>>>(c, c_shift, nc, log_lo, span, qgrid);
    MGSR_LAUNCH_CHECK();
    if (int r = launch_gen<0>(P, f16 != 0, dbg != nullptr || prof != nullptr, st)) return r;
    {
        const int ne = edge_count(P.npos);
        // per current device (function attributes are per device), like k_gen_tc's above
        MGSR_CUDA_TRY(cudaFuncSetAttribute(f16 ? k_tail_edge<true> : k_tail_edge<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(TE_SMEM)));
        const int nb = ne < nsm ? ne : nsm;
        if (f16) k_tail_edge<true><<<nb, TE_THREADS, TE_SMEM, st>>>(P, ne);
        else k_tail_edge<false><<<nb, TE_THREADS, TE_SMEM, st>>>(P, ne);
    }
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

int launch_sr_pass_tc(const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo, double span,
                      double *fine, void *ws, size_t ws_bytes, cudaStream_t st, int f16) {
    return launch_sr_pass_tc_dbg(g, c, c_shift, nc, log_lo, span, fine, ws, ws_bytes, nullptr, -1, st, nullptr, f16);
}

// Batched ratio-2 passes (config 5, mgsr_plan_solve_batch): the windows of the *count grids listed in `list`
// (device-side, written by the solve loop's controller) in ONE persistent k_gen_tc launch and one edge-tail
// launch; grid r's coarse correction is cs[r] (device pointer array), its output fine_base + r nf^2.  Each
// window's arithmetic is the single-grid launch's, so the outputs are bitwise those of launch_sr_pass_tc.
size_t tc_batch_workspace_bytes(int64_t nc, int B) {
    return size_t(B) * tc_edge_bytes(nc) + sizeof(float) * size_t(B) * nc * nc + 256;
}
int launch_sr_pass_tc_batch(const mgsr_gen *g, const double *const *cs, int B, const int *list, const int *count,
                            int nc, double log_lo, double span, double *fine_base, void *ws, size_t ws_bytes,
                            cudaStream_t st, int f16) {
    using namespace tc;
    if (!g->tc_blob) { set_error("tensor-core weights not packed"); return MGSR_E_UNSUPPORTED; }
    if (ws_bytes < tc_batch_workspace_bytes(nc, B)) { set_error("tensor-core workspace too small"); return MGSR_E_WORKSPACE; }
    Params P{};
    fill_params(P, g, nullptr, nullptr, nc, log_lo, span, fine_base, 2, f16);
    P.nwin1 = P.nwin;
    P.nwin = P.nwin1 * B;   // the launch's capacity; the kernels read *count
    P.rhs_list = list;
    P.rhs_count = count;
    P.q_stride = (long long)nc * nc;
    P.fine_stride = 4LL * nc * nc;
    char *w = static_cast<char *>(ws);
    P.edge_u = reinterpret_cast<uint16_t *>(w);
    float *qgrid = reinterpret_cast<float *>(w + size_t(B) * tc_edge_bytes(nc));
    P.qgrid = qgrid;
    int nsm = 0, dev = 0;
    MGSR_CUDA_TRY(cudaGetDevice(&dev));
    MGSR_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    k_normalize_batch<<<grid_for((long long)B * nc * nc, 256), 256, 0, st>>>(cs, B, nc, log_lo, span, qgrid);
    MGSR_LAUNCH_CHECK();
    if (int r = launch_gen<0, true>(P, f16 != 0, false, st)) return r;
    const int ne = edge_count(P.npos) * B;
    MGSR_CUDA_TRY(cudaFuncSetAttribute(f16 ? k_tail_edge<true> : k_tail_edge<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, int(TE_SMEM)));
    const int nb = ne < nsm ? ne : nsm;
    if (f16) k_tail_edge<true><<<nb, TE_THREADS, TE_SMEM, st>>>(P, ne);
    else k_tail_edge<false><<<nb, TE_THREADS, TE_SMEM, st>>>(P, ne);
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

// A ratio-4 windowed pass (two generator applications, srmodel.py:443-463 with applications = 2) on the tensor
// cores: normalise -> k_gen_tc<V = 1> (6x6 windows -> full 12x12x3 X1) -> k_gen_tc<V = 2> (X1 -> kept 8x8
// fine pixels of interior windows) -> k_tail_edge4 (edge windows' kept bands, exact fp32 tail).
int launch_sr_pass4_tc(const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo, double span,
                       double *fine, void *ws, size_t ws_bytes, cudaStream_t st, int f16) {
    using namespace tc;
    if (!g->tc_blob) { set_error("tensor-core weights not packed"); return MGSR_E_UNSUPPORTED; }
    if (ws_bytes < tc4_workspace_bytes(nc)) { set_error("tensor-core workspace too small"); return MGSR_E_WORKSPACE; }
    Params P{};
    fill_params(P, g, c, c_shift, nc, log_lo, span, fine, 4, f16);
    char *w = static_cast<char *>(ws);
    P.edge_u = reinterpret_cast<uint16_t *>(w);
    P.x1 = reinterpret_cast<uint16_t *>(w + tc4_edge_bytes(nc));
    float *qgrid = reinterpret_cast<float *>(w + tc4_edge_bytes(nc) + tc4_x1_bytes(nc));
    P.qgrid = qgrid;
    int nsm = 0, dev = 0;
    MGSR_CUDA_TRY(cudaGetDevice(&dev));
    MGSR_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    k_normalize<<<grid_for((long long)nc * nc, 256), 256, 0, st>>>(c, c_shift, nc, log_lo, span, qgrid);
    MGSR_LAUNCH_CHECK();
    if (int r = launch_gen<1>(P, f16 != 0, false, st)) return r;
    if (int r = launch_gen<2>(P, f16 != 0, false, st)) return r;
    {
        const int ne = edge_count(P.npos);
        MGSR_CUDA_TRY(cudaFuncSetAttribute(f16 ? k_tail_edge4<true> : k_tail_edge4<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(TE4_SMEM)));
        const int nb = ne < 4 * nsm ? ne : 4 * nsm;
        if (f16) k_tail_edge4<true><<<nb, TE4_THREADS, TE4_SMEM, st>>>(P, ne);
        else k_tail_edge4<false><<<nb, TE4_THREADS, TE4_SMEM, st>>>(P, ne);
    }
    MGSR_LAUNCH_CHECK();
    return MGSR_OK;
}

}  // namespace mgsr

// debug entries (not in the public header)
extern "C" int mgsr_debug_tc_pass(const mgsr_gen *g, const double *c, int64_t nc, double p_min, double p_max,
                                  double *fine, float *dbg, int32_t dbg_layer, int32_t f16, void *stream) {
    const size_t wsb = mgsr::tc_workspace_bytes(nc);
    void *ws = nullptr;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int e = mgsr::scratch_alloc(&ws, wsb, st)) return e;
    int r = mgsr::launch_sr_pass_tc_dbg(g, c, nullptr, int(nc), std::log10(p_min),
                                        std::log10(p_max) - std::log10(p_min), fine, ws, wsb, dbg, dbg_layer, st,
                                        nullptr, f16);
    cudaFreeAsync(ws, st);
    return r;
}

extern "C" int mgsr_debug_tc_prof(const mgsr_gen *g, const double *c, int64_t nc, double *fine,
                                  unsigned long long *prof, int32_t f16, void *stream) {
    const size_t wsb = mgsr::tc_workspace_bytes(nc);
    void *ws = nullptr;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (int e = mgsr::scratch_alloc(&ws, wsb, st)) return e;
    int r = mgsr::launch_sr_pass_tc_dbg(g, c, nullptr, int(nc), -10.0, 7.0, fine, ws, wsb, nullptr, -1, st, prof, f16);
    cudaFreeAsync(ws, st);
    return r;
}
