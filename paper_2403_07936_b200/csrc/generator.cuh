// Generator handle and SR-prolongation launchers (internal).
#pragma once
#include <vector>

#include "common.cuh"

struct mgsr_gen {
    int blocks = 0;
    double tanh_scale = 1.0;
    // fp32 device tensors (reference layout, OIHW)
    float *head_w = nullptr;   // 64 x 3 x 9 x 9
    float *head_a = nullptr;   // 64
    std::vector<float *> c1, c2;           // per block 64x64x3x3
    std::vector<float *> bn1s, bn1b, bn2s, bn2b, pa;   // folded BN scale / shift, PReLU alpha
    float *post_w = nullptr, *post_s = nullptr, *post_b = nullptr;
    float *up_w = nullptr, *up_a = nullptr;  // 256x64x3x3, 64
    float *tail_w = nullptr, *tail_b = nullptr;  // 3x64x9x9, 3
    // the same conv weights as [C][taps][O] (tail: O padded to 4) for the row-tiled fp32 kernels
    float *head_t = nullptr, *post_t = nullptr, *up_t = nullptr, *tail_t = nullptr;
    std::vector<float *> c1_t, c2_t;
    // tensor-core path: packed weights / constants (one device blob), see generator_tc.cu
    void *tc_blob = nullptr;
    size_t tc_bytes = 0;
    std::vector<void *> allocations;
};

namespace mgsr {

// One predicate decides both the workspace size and the kernel of a precision mode.
inline bool valid_precision(int p) {
    return p == MGSR_PREC_FP32 || p == MGSR_PREC_BF16 || p == MGSR_PREC_FP16 || p == MGSR_PREC_MIXED;
}
// the tensor-core path for ratio-2 / single-pass work (MIXED = fp16 there)
inline bool tensor_core_precision(int p) { return p == MGSR_PREC_BF16 || p == MGSR_PREC_FP16 || p == MGSR_PREC_MIXED; }
// the precision of pass `ip` of `npass` under a precision mode: MIXED runs the first pass of a two-pass
// ratio in fp32 and everything else as fp16
inline int pass_precision(int p, int ip, int npass) {
    if (p != MGSR_PREC_MIXED) return p;
    return (npass == 2 && ip == 0) ? MGSR_PREC_FP32 : MGSR_PREC_FP16;
}

// Windowed SR prolongation (one full sr_prolong, all passes).
// c_shift: optional device scalar subtracted from c before normalising.
// out: fine grid (nc*s)^2 raw data (before the final mean subtraction);
// out_mean: device scalar = mean(out).
size_t sr_workspace_bytes(int64_t nc, int s, int precision);
int launch_sr_prolong(const mgsr_gen *g, const double *c, const double *c_shift, int nc, int s, double p_min,
                      double p_max, int precision, double *out, double *out_mean, void *ws, size_t ws_bytes,
                      void *red_slot, cudaStream_t st, cudaEvent_t *gen_markers = nullptr);

// tensor-core generator (generator_tc.cu): a ratio-2 pass (one application) and a ratio-4 pass (two).
int tc_pack_weights(mgsr_gen *g, const float *const *host_tensors);
size_t tc_workspace_bytes(int64_t nc);
size_t tc4_workspace_bytes(int64_t nc);
int launch_sr_pass_tc(const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo,
                      double span, double *fine, void *ws, size_t ws_bytes, cudaStream_t st, int f16);
size_t tc_batch_workspace_bytes(int64_t nc, int B);
int launch_sr_pass_tc_batch(const mgsr_gen *g, const double *const *cs, int B, const int *list, const int *count,
                            int nc, double log_lo, double span, double *fine_base, void *ws, size_t ws_bytes,
                            cudaStream_t st, int f16);
int launch_mean_f64(const double *a, int64_t count, void *red_slot, double *result, cudaStream_t st);
int launch_sr_pass4_tc(const mgsr_gen *g, const double *c, const double *c_shift, int nc, double log_lo,
                       double span, double *fine, void *ws, size_t ws_bytes, cudaStream_t st, int f16);

}  // namespace mgsr
