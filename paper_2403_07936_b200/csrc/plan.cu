// Device-resident V-cycle (solver.py:158-197) plus the solve-loop logging pass
// (solver.py:311-313), captured once per (operator, buffers) variant into a
// CUDA graph and replayed: one graph launch per cycle.
//
// Level buffers (fine -> coarse, sides from level_sides, solver.py:100-119):
//   level 0: caller's p (iterate) and f; S = smoothed iterate, then out.
//   level l>=1: rc[l] = raw injected residual of level l-1 (its RHS is
//     0.5 * (rc[l] - mean(rc[l])), consumed on the fly, solver.py:178-179),
//     d[l] = Gauss-Seidel correction from zero (raw, mean d_mean[l]),
//     then d[l] <- (d[l] - d_mean[l]) + up[l]   (solver.py:190).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "generator.cuh"
#include "stencil.cuh"

using namespace mgsr;

namespace {

enum Scalar {
    SC_S_MEAN = 0,    // mean of the smoothed top iterate
    SC_OUT_MEAN = 1,  // mean of out (top)
    SC_ACC = 2,       // 3 accumulators for the logging pass (2..4)
    SC_STATS = 5,     // diff_norm, residual rms (5..6) -- internal copy
    SC_LEVEL0 = 8     // per level l: rc_mean 8+4l, d_mean 9+4l, sr_mean 10+4l
};

}  // namespace

struct mgsr_plan {
    mgsr_plan_config cfg{};
    const mgsr_gen *gen = nullptr;
    std::vector<int> sides;
    void *mem = nullptr;
    size_t mem_bytes = 0;
    double *scal = nullptr;
    void *red = nullptr;      // 4 reduction slots
    double *S = nullptr, *tmp = nullptr, *srbuf = nullptr;
    std::vector<double *> rc, d;
    void *srws = nullptr;
    size_t srws_bytes = 0;
    cudaStream_t cap = nullptr;
    struct Graph {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        std::vector<std::pair<int, cudaGraphNode_t>> marker_nodes;
        int kernel_nodes = 0;
    };
    std::map<std::tuple<double *, const double *, int>, Graph> graphs;
    // device-resident solve loops: graph per (p, f, schedule) with conditional nodes
    struct SolveGraph {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
    };
    std::map<std::tuple<double *, const double *, int, int, double, double, int, int, int>, SolveGraph> solves;
    int *solve_state = nullptr;      // [4] it, latched, op, iterations (device)
    double *solve_rec = nullptr;     // [rec_cap][4] diff_norm, residual_rms, op, latched (device)
    int rec_cap = 0;
    // instrumentation: placeholder events captured as event-record nodes
    cudaEvent_t cap_ev[6] = {};
    bool capturing_markers = false;
    std::vector<cudaEvent_t> pool;
    int pool_used = 0, pool_cap = 0;
    // debug (parity tests): per level l, copy the SR prolongation's input correction (nc^2) and its raw
    // output (nf^2, before the mean subtraction) to caller buffers inside the captured cycle
    std::map<int, std::pair<double *, double *>> sr_dump;
};

namespace {

// Under Nsight Compute (its injection sets NV_NSIGHT_INJECTION_TRANSPORT_TYPE / NV_TPS_LAUNCH_TOKEN /
// NV_COMPUTE_PROFILER_PERFWORKS_DIR; other injecting tools CUDA_INJECTION64_PATH) the first kernel
// launched into a stream capture fails ("LaunchFailed"), so the plan issues the same kernel sequence
// eagerly, as MGSR_NO_GRAPH=1 does.
bool graphs_disabled() {
    for (const char *v : {"MGSR_NO_GRAPH", "CUDA_INJECTION64_PATH", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                          "NV_TPS_LAUNCH_TOKEN", "NV_COMPUTE_PROFILER_PERFWORKS_DIR"})
        if (std::getenv(v)) return true;
    return false;
}

double *sc(mgsr_plan *pl, int i) { return pl->scal + i; }
double *rc_mean(mgsr_plan *pl, int l) { return pl->scal + SC_LEVEL0 + 4 * l; }
double *d_mean(mgsr_plan *pl, int l) { return pl->scal + SC_LEVEL0 + 4 * l + 1; }
double *sr_mean(mgsr_plan *pl, int l) { return pl->scal + SC_LEVEL0 + 4 * l + 2; }
void *slot(mgsr_plan *pl, int k) { return static_cast<char *>(pl->red) + k * kRedSlotBytes; }

int ladder(int64_t n, int n_step, int r_min, std::vector<int> &sides) {
    if (n <= r_min) { set_error("fine side must exceed r_min"); return MGSR_E_LADDER; }
    sides.assign(1, int(n));
    while (sides.back() > r_min) {
        int nxt = sides.back() >> n_step;
        if (nxt < r_min) nxt = r_min;
        int ratio = sides.back() / nxt;
        if (nxt * ratio != sides.back() || !(ratio == 2 || ratio == 4 || ratio == 8 || ratio == 16)) {
            set_error("no valid ladder from " + std::to_string(n) + " to r_min " + std::to_string(r_min) +
                      " with step 2^" + std::to_string(n_step));
            return MGSR_E_LADDER;
        }
        sides.push_back(nxt);
    }
    return MGSR_OK;
}

// The finest prolongation of a spline (or non-SR-at-level-1) cycle fused with the logging pass
// (k_prolong_finalize_rows): the mean of out is the mean of d[1], which the level-2 prolongation emits.
bool fused_top(const mgsr_plan *pl, int use_sr) {
    return pl->sides.size() >= 3 && pl->sides[0] == 2 * pl->sides[1] && prolong_finalize_applies(pl->sides[0]) &&
           !(use_sr && (pl->cfg.sr_level_mask & 1u));
}
double *d1_out_mean(mgsr_plan *pl) { return pl->scal + SC_LEVEL0 + 4 * 1 + 3; }

// Prolong the correction of level l (buffer d[l], or the coarsest GS result)
// into level l-1 and add to `base` (level l-1 GS result with mean *bshift):
// out = (base - *bshift) + P(corr).  mean_out (optional) = mean(out).
int prolong_into(mgsr_plan *pl, int l, int use_sr, const double *base, const double *bshift, double *out,
                 double *mean_out, cudaStream_t st) {
    const int nc = pl->sides[l], s = pl->sides[l - 1] / pl->sides[l];
    const double *corr = pl->d[l];
    const bool sr = use_sr && ((pl->cfg.sr_level_mask >> (l - 1)) & 1u);
    if (!sr) return launch_prolong_add(corr, nc, s, base, bshift, out, mean_out, slot(pl, 3), st);
    int r = launch_sr_prolong(pl->gen, corr, nullptr, nc, s, pl->cfg.p_min, pl->cfg.p_max, pl->cfg.precision,
                              pl->srbuf, sr_mean(pl, l), pl->srws, pl->srws_bytes, slot(pl, 2), st,
                              (l == 1 && pl->capturing_markers) ? pl->cap_ev : nullptr);
    if (r) return r;
    const int64_t nf = int64_t(nc) * s;
    auto dump = pl->sr_dump.find(l);
    if (dump != pl->sr_dump.end()) {
        if (dump->second.first)
            MGSR_CUDA_TRY(cudaMemcpyAsync(dump->second.first, corr, sizeof(double) * nc * nc, cudaMemcpyDeviceToDevice, st));
        if (dump->second.second)
            MGSR_CUDA_TRY(cudaMemcpyAsync(dump->second.second, pl->srbuf, sizeof(double) * nf * nf,
                                          cudaMemcpyDeviceToDevice, st));
    }
    return launch_add2(base, bshift, pl->srbuf, sr_mean(pl, l), out, nf * nf, mean_out, slot(pl, 3), st);
}

// correction(rhs_l, l) of solver.py:181-190; leaves the gauge-fixed result in d[l].  stop > 0 (batched
// solves): the prolongations from levels <= stop are left to the caller (prolong_level, level-major).
int correction(mgsr_plan *pl, int l, int use_sr, cudaStream_t st, int stop = 0) {
    const int L = int(pl->sides.size());
    const int n = pl->sides[l];
    const double h = 2.0 * M_PI / n;
    FSrc fs{pl->rc[l], rc_mean(pl, l), 0.5};
    int r;
    if (n <= kSmallN && !std::getenv("MGSR_NO_FUSED_SMALL")) {
        // the whole bottom of the ladder in one CTA, when it is ratio 2 and spline-prolonged
        bool fusable = L - l <= 8;
        for (int j = l; fusable && j < L - 1; ++j) {
            if (pl->sides[j] != 2 * pl->sides[j + 1]) fusable = false;
            if (use_sr && ((pl->cfg.sr_level_mask >> j) & 1u)) fusable = false;
        }
        if (fusable)
            return launch_correction_small(pl->rc[l], rc_mean(pl, l), pl->d[l], pl->sides.data() + l, L - l,
                                           pl->cfg.n_smooth, pl->cfg.coarse_sweeps, st);
    }
    if (l == L - 1) {
        r = launch_gs(nullptr, pl->d[l], pl->tmp, fs, n, h * h, pl->cfg.coarse_sweeps, 1, nullptr, nullptr,
                      d_mean(pl, l), pl->red, st);
        if (r) return r;
        if (n > kSmallN) return launch_affine(pl->d[l], pl->d[l], int64_t(n) * n, d_mean(pl, l), 1.0, st);
        return MGSR_OK;
    }
    const int s = n / pl->sides[l + 1];
    const bool fuse_rc = (s == 2);
    r = launch_gs(nullptr, pl->d[l], pl->tmp, fs, n, h * h, pl->cfg.n_smooth, 1, fuse_rc ? pl->rc[l + 1] : nullptr,
                  fuse_rc ? rc_mean(pl, l + 1) : nullptr, d_mean(pl, l), pl->red, st);
    if (r) return r;
    if (!fuse_rc && (r = launch_res_restrict(pl->d[l], fs, n, s, pl->rc[l + 1], rc_mean(pl, l + 1), slot(pl, 1), st)))
        return r;
    if ((r = correction(pl, l + 1, use_sr, st, stop))) return r;
    if (l + 1 <= stop) return MGSR_OK;
    // d[l] = (d[l] - d_mean) + up  (in place: elementwise)
    const double *bshift = n <= kSmallN ? nullptr : d_mean(pl, l);
    return prolong_into(pl, l + 1, use_sr, pl->d[l], bshift, pl->d[l],
                        (l == 1 && fused_top(pl, use_sr)) ? d1_out_mean(pl) : nullptr, st);
}

int record_top(mgsr_plan *pl, double *p, const double *f, int use_sr, cudaStream_t st);

int record_vcycle(mgsr_plan *pl, double *p, const double *f, int use_sr, cudaStream_t st) {
    const int n = pl->sides[0];
    const double h = 2.0 * M_PI / n;
    const int s0 = n / pl->sides[1];
    FSrc fs{f, nullptr, 1.0};
    const bool mk = pl->capturing_markers;
    if (mk) MGSR_CUDA_TRY(cudaEventRecordWithFlags(pl->cap_ev[4], st, cudaEventRecordExternal));
    const int L = int(pl->sides.size());
    bool tiny = n <= kSmallN && L >= 2 && L <= 8 && !std::getenv("MGSR_NO_FUSED_SMALL");
    for (int j = 0; tiny && j < L - 1; ++j) {
        if (pl->sides[j] != 2 * pl->sides[j + 1]) tiny = false;
        if (use_sr && ((pl->cfg.sr_level_mask >> j) & 1u)) tiny = false;
    }
    if (tiny) {   // the whole spline cycle + logging pass of a small grid in one CTA
        int r = launch_vcycle_small(p, f, pl->sides.data(), L, pl->cfg.n_smooth, pl->cfg.coarse_sweeps,
                                    sc(pl, SC_STATS), st);
        if (r) return r;
        if (mk) MGSR_CUDA_TRY(cudaEventRecordWithFlags(pl->cap_ev[5], st, cudaEventRecordExternal));
        return MGSR_OK;
    }
    if (mk) MGSR_CUDA_TRY(cudaEventRecordWithFlags(pl->cap_ev[2], st, cudaEventRecordExternal));
    int r = launch_gs(p, pl->S, pl->tmp, fs, n, h * h, pl->cfg.n_smooth, 0, s0 == 2 ? pl->rc[1] : nullptr,
                      s0 == 2 ? rc_mean(pl, 1) : nullptr, sc(pl, SC_S_MEAN), pl->red, st);
    if (r) return r;
    if (mk) MGSR_CUDA_TRY(cudaEventRecordWithFlags(pl->cap_ev[3], st, cudaEventRecordExternal));
    if (s0 != 2 && (r = launch_res_restrict(pl->S, fs, n, s0, pl->rc[1], rc_mean(pl, 1), slot(pl, 1), st))) return r;
    if ((r = correction(pl, 1, use_sr, st))) return r;
    if ((r = record_top(pl, p, f, use_sr, st))) return r;
    if (mk) MGSR_CUDA_TRY(cudaEventRecordWithFlags(pl->cap_ev[5], st, cudaEventRecordExternal));
    return MGSR_OK;
}

// The batched solve's pieces of record_vcycle (same kernels, same order per grid): everything before the
// prolongation from level `stop` (record_down), one prolongation (prolong_level / sr_add_level), the
// logging pass (record_finalize).
int prolong_level(mgsr_plan *pl, int l, int use_sr, cudaStream_t st) {
    if (l == 1) {
        const double *bshift = pl->sides[0] <= kSmallN ? nullptr : sc(pl, SC_S_MEAN);
        return prolong_into(pl, 1, use_sr, pl->S, bshift, pl->S, sc(pl, SC_OUT_MEAN), st);
    }
    const double *bshift = pl->sides[l - 1] <= kSmallN ? nullptr : d_mean(pl, l - 1);
    return prolong_into(pl, l, use_sr, pl->d[l - 1], bshift, pl->d[l - 1],
                        (l == 2 && fused_top(pl, use_sr)) ? d1_out_mean(pl) : nullptr, st);
}

int record_down(mgsr_plan *pl, double *p, const double *f, int use_sr, cudaStream_t st, int stop) {
    const int n = pl->sides[0];
    const double h = 2.0 * M_PI / n;
    const int s0 = n / pl->sides[1];
    FSrc fs{f, nullptr, 1.0};
    int r = launch_gs(p, pl->S, pl->tmp, fs, n, h * h, pl->cfg.n_smooth, 0, s0 == 2 ? pl->rc[1] : nullptr,
                      s0 == 2 ? rc_mean(pl, 1) : nullptr, sc(pl, SC_S_MEAN), pl->red, st);
    if (r) return r;
    if (s0 != 2 && (r = launch_res_restrict(pl->S, fs, n, s0, pl->rc[1], rc_mean(pl, 1), slot(pl, 1), st))) return r;
    return correction(pl, 1, use_sr, st, stop);
}

// the SR branch of prolong_into after the (batched) generator wrote this grid's raw output to srbuf
int sr_add_level(mgsr_plan *pl, int l, const double *srbuf, cudaStream_t st) {
    const int64_t nf = pl->sides[l - 1];
    int r = launch_mean_f64(srbuf, nf * nf, slot(pl, 2), sr_mean(pl, l), st);
    if (r) return r;
    double *base = l == 1 ? pl->S : pl->d[l - 1];
    const double *bshift = l == 1 ? (pl->sides[0] <= kSmallN ? nullptr : sc(pl, SC_S_MEAN))
                                  : (pl->sides[l - 1] <= kSmallN ? nullptr : d_mean(pl, l - 1));
    double *mean_out = l == 1 ? sc(pl, SC_OUT_MEAN) : ((l == 2 && fused_top(pl, 1)) ? d1_out_mean(pl) : nullptr);
    return launch_add2(base, bshift, srbuf, sr_mean(pl, l), base, nf * nf, mean_out, slot(pl, 3), st);
}

int record_finalize(mgsr_plan *pl, double *p, const double *f, cudaStream_t st) {
    FSrc fs{f, nullptr, 1.0};
    return launch_finalize(pl->S, sc(pl, SC_OUT_MEAN), p, fs, pl->sides[0], sc(pl, SC_ACC), sc(pl, SC_STATS),
                           slot(pl, 0), st);
}

// the finest prolongation and the logging pass of a cycle (record_vcycle's tail)
int record_top(mgsr_plan *pl, double *p, const double *f, int use_sr, cudaStream_t st) {
    if (fused_top(pl, use_sr)) {
        FSrc fs{f, nullptr, 1.0};
        return launch_prolong_finalize(pl->S, sc(pl, SC_S_MEAN), pl->d[1], pl->sides[1], d1_out_mean(pl), p, fs,
                                       sc(pl, SC_ACC), sc(pl, SC_STATS), slot(pl, 0), st);
    }
    int r = prolong_level(pl, 1, use_sr, st);
    return r ? r : record_finalize(pl, p, f, st);
}

}  // namespace

extern "C" int mgsr_plan_create(const mgsr_plan_config *cfg, const mgsr_gen *gen, mgsr_plan **out) {
    if (!cfg || !out) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    if (cfg->n_smooth < 1 || cfg->coarse_sweeps < 1) { set_error("sweep counts must be positive"); return MGSR_E_BAD_ARG; }
    if (cfg->r_min < 2 || cfg->r_min % 2) { set_error("r_min must be an even integer >= 2"); return MGSR_E_BAD_ARG; }
    if (!valid_precision(cfg->precision)) { set_error("precision must be one of fp32, bf16, fp16, mixed"); return MGSR_E_BAD_ARG; }
    mgsr_plan *pl = new mgsr_plan();
    pl->cfg = *cfg;
    pl->gen = gen;
    int r = ladder(cfg->n, cfg->n_step, cfg->r_min, pl->sides);
    if (r) { delete pl; return r; }
    const int L = int(pl->sides.size());
    if (L > 24) { delete pl; set_error("ladder too deep"); return MGSR_E_LADDER; }
    const int64_t n = cfg->n;
    // SR needs every prolongation's coarse side >= 6 and even
    bool any_sr = false;
    int64_t sr_ws = 0, sr_fine_max = 0;
    if (gen) {
        for (int l = 1; l < L; ++l) {
            if (!((cfg->sr_level_mask >> (l - 1)) & 1u)) continue;
            int nc = pl->sides[l], s = pl->sides[l - 1] / nc;
            if (nc < 6 || nc % 2) continue;
            any_sr = true;
            int64_t w = int64_t(sr_workspace_bytes(nc, s, cfg->precision));
            if (w > sr_ws) sr_ws = w;
            int64_t nf = int64_t(nc) * s;
            if (nf * nf > sr_fine_max) sr_fine_max = nf * nf;
        }
    }
    size_t bytes = 4096 + 4 * kRedSlotBytes;          // scalars + slots
    bytes += sizeof(double) * size_t(n) * n * 2;      // S, tmp
    for (int l = 1; l < L; ++l) bytes += 2 * sizeof(double) * size_t(pl->sides[l]) * pl->sides[l];
    if (any_sr) bytes += sizeof(double) * size_t(sr_fine_max) + size_t(sr_ws) + 256;
    cudaError_t e = cudaMalloc(&pl->mem, bytes);
    if (e != cudaSuccess) { delete pl; set_error(std::string("plan alloc: ") + cudaGetErrorString(e)); return MGSR_E_CUDA; }
    cudaMemset(pl->mem, 0, 4096 + 4 * kRedSlotBytes);
    pl->mem_bytes = bytes;
    char *m = static_cast<char *>(pl->mem);
    pl->scal = reinterpret_cast<double *>(m);
    m += 4096;
    pl->red = m;
    m += 4 * kRedSlotBytes;
    pl->S = reinterpret_cast<double *>(m); m += sizeof(double) * size_t(n) * n;
    pl->tmp = reinterpret_cast<double *>(m); m += sizeof(double) * size_t(n) * n;
    pl->rc.assign(L, nullptr);
    pl->d.assign(L, nullptr);
    for (int l = 1; l < L; ++l) {
        size_t c = size_t(pl->sides[l]) * pl->sides[l];
        pl->rc[l] = reinterpret_cast<double *>(m); m += sizeof(double) * c;
        pl->d[l] = reinterpret_cast<double *>(m); m += sizeof(double) * c;
    }
    if (any_sr) {
        pl->srbuf = reinterpret_cast<double *>(m); m += sizeof(double) * size_t(sr_fine_max);
        m = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(m) + 255) & ~uintptr_t(255));
        pl->srws = m;
        pl->srws_bytes = size_t(sr_ws);
    }
    e = cudaStreamCreateWithFlags(&pl->cap, cudaStreamNonBlocking);
    if (e != cudaSuccess) { mgsr_plan_destroy(pl); set_error("stream create failed"); return MGSR_E_CUDA; }
    for (auto &ev : pl->cap_ev) cudaEventCreate(&ev);
    pl->capturing_markers = true;   // graphs always carry marker nodes (no-ops unless re-targeted)
    *out = pl;
    return MGSR_OK;
}

void batch_forget(const mgsr_plan *pl);

extern "C" int mgsr_plan_destroy(mgsr_plan *pl) {
    if (!pl) return MGSR_OK;
    batch_forget(pl);   // batched solve graphs that captured this plan's buffers
    for (auto &kv : pl->graphs) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaGraphDestroy(kv.second.graph);
    }
    for (auto &kv : pl->solves) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaGraphDestroy(kv.second.graph);
    }
    if (pl->solve_state) cudaFree(pl->solve_state);
    if (pl->solve_rec) cudaFree(pl->solve_rec);
    for (auto ev : pl->cap_ev) if (ev) cudaEventDestroy(ev);
    for (auto ev : pl->pool) cudaEventDestroy(ev);
    if (pl->cap) cudaStreamDestroy(pl->cap);
    if (pl->mem) cudaFree(pl->mem);
    delete pl;
    return MGSR_OK;
}

extern "C" int32_t mgsr_plan_levels(const mgsr_plan *pl, int64_t *sides_out) {
    if (!pl) return 0;
    for (size_t i = 0; i < pl->sides.size() && sides_out; ++i) sides_out[i] = pl->sides[i];
    return int32_t(pl->sides.size());
}

extern "C" int mgsr_plan_vcycle(mgsr_plan *pl, double *p, const double *f, int32_t use_sr, double *stats_dev,
                                void *stream) {
    if (!pl || !p || !f) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    if (use_sr && !pl->gen) { set_error("SR prolongation requires generator weights"); return MGSR_E_BAD_ARG; }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (graphs_disabled()) {
        // eager issue of the same kernel sequence (profilers that cannot replay graph nodes)
        const bool mk = pl->capturing_markers;
        pl->capturing_markers = false;   // external event records exist only inside captures
        int r = record_vcycle(pl, p, f, use_sr != 0, st);
        pl->capturing_markers = mk;
        if (r) return r;
        if (stats_dev)
            MGSR_CUDA_TRY(cudaMemcpyAsync(stats_dev, sc(pl, SC_STATS), 2 * sizeof(double), cudaMemcpyDeviceToDevice, st));
        return MGSR_OK;
    }
    auto key = std::make_tuple(p, f, int(use_sr != 0));
    auto it = pl->graphs.find(key);
    if (it == pl->graphs.end() && pl->graphs.size() >= 16) {
        // bounded cache: callers cycling through many buffers re-capture instead of growing without end
        for (auto &kv : pl->graphs) {
            cudaGraphExecDestroy(kv.second.exec);
            cudaGraphDestroy(kv.second.graph);
        }
        pl->graphs.clear();
    }
    if (it == pl->graphs.end()) {
        // capture on the plan's own stream, then instantiate once
        MGSR_CUDA_TRY(cudaStreamSynchronize(st));
        MGSR_CUDA_TRY(cudaStreamBeginCapture(pl->cap, cudaStreamCaptureModeRelaxed));
        int r = record_vcycle(pl, p, f, use_sr != 0, pl->cap);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(pl->cap, &graph);
        if (r) { if (graph) cudaGraphDestroy(graph); return r; }
        if (e != cudaSuccess) { set_error(std::string("graph capture: ") + cudaGetErrorString(e)); return MGSR_E_CUDA; }
        mgsr_plan::Graph G;
        G.graph = graph;
        size_t nn = 0;
        cudaGraphGetNodes(graph, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(graph, nodes.data(), &nn);
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            cudaGraphNodeGetType(nd, &t);
            if (t == cudaGraphNodeTypeKernel) G.kernel_nodes++;
            if (t == cudaGraphNodeTypeEventRecord) {
                cudaEvent_t ev;
                cudaGraphEventRecordNodeGetEvent(nd, &ev);
                for (int k = 0; k < 6; ++k)
                    if (ev == pl->cap_ev[k]) G.marker_nodes.push_back({k, nd});
            }
        }
        e = cudaGraphInstantiate(&G.exec, graph, 0);
        if (e != cudaSuccess) { cudaGraphDestroy(graph); set_error(std::string("graph instantiate: ") + cudaGetErrorString(e)); return MGSR_E_CUDA; }
        it = pl->graphs.emplace(key, G).first;
    }
    mgsr_plan::Graph &G = it->second;
    if (pl->pool_used < pl->pool_cap) {
        cudaEvent_t *evs = pl->pool.data() + 6 * pl->pool_used;
        for (auto &mn : G.marker_nodes) MGSR_CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(G.exec, mn.second, evs[mn.first]));
        pl->pool_used++;
    } else if (pl->pool_cap > 0 && pl->pool_used == pl->pool_cap) {
        // stop recording into the pool: point the nodes back at the placeholders
        for (auto &mn : G.marker_nodes) MGSR_CUDA_TRY(cudaGraphExecEventRecordNodeSetEvent(G.exec, mn.second, pl->cap_ev[mn.first]));
    }
    MGSR_CUDA_TRY(cudaGraphLaunch(G.exec, st));
    if (stats_dev)
        MGSR_CUDA_TRY(cudaMemcpyAsync(stats_dev, sc(pl, SC_STATS), 2 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return MGSR_OK;
}

// Debug entry (not in the public header; tests/test_gpu_solver.py): dump the SR prolongation from level
// `level` into level - 1 of every following cycle: c_dst receives its input correction (n_level^2 doubles),
// sr_dst its raw output (n_{level-1}^2, before the mean subtraction).  NULL pointers clear the dump.
// Drops the captured graphs so the copies enter the next capture.
extern "C" int mgsr_debug_plan_sr_dump(mgsr_plan *pl, int32_t level, double *c_dst, double *sr_dst) {
    if (!pl || level < 1 || level >= int(pl->sides.size())) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    if (c_dst || sr_dst) pl->sr_dump[level] = {c_dst, sr_dst};
    else pl->sr_dump.erase(level);
    for (auto &kv : pl->graphs) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaGraphDestroy(kv.second.graph);
    }
    pl->graphs.clear();
    for (auto &kv : pl->solves) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaGraphDestroy(kv.second.graph);
    }
    pl->solves.clear();
    return MGSR_OK;
}

extern "C" int mgsr_plan_timing_enable(mgsr_plan *pl, int32_t max_launches) {
    if (!pl || max_launches < 0) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    for (auto ev : pl->pool) cudaEventDestroy(ev);
    pl->pool.assign(size_t(max_launches) * 6, nullptr);
    for (auto &ev : pl->pool) MGSR_CUDA_TRY(cudaEventCreate(&ev));
    pl->pool_cap = max_launches;
    pl->pool_used = 0;
    return MGSR_OK;
}

extern "C" int mgsr_plan_timing_read(mgsr_plan *pl, double *ms_out, int32_t *launches_out) {
    if (!pl || !ms_out) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    double acc[3] = {0, 0, 0};
    int cnt[3] = {0, 0, 0};
    for (int i = 0; i < pl->pool_used; ++i) {
        cudaEvent_t *evs = pl->pool.data() + 6 * i;
        for (int k = 0; k < 3; ++k) {
            if (cudaEventSynchronize(evs[2 * k]) != cudaSuccess || cudaEventSynchronize(evs[2 * k + 1]) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, evs[2 * k], evs[2 * k + 1]) == cudaSuccess) {
                acc[k] += ms;
                cnt[k]++;
            } else {
                cudaGetLastError();   // event never recorded in this graph variant
            }
        }
    }
    for (int k = 0; k < 3; ++k) ms_out[k] = cnt[k] ? acc[k] / cnt[k] : 0.0;
    if (launches_out) *launches_out = pl->pool_used;
    return MGSR_OK;
}

extern "C" int32_t mgsr_plan_kernel_nodes(mgsr_plan *pl, int32_t use_sr) {
    if (!pl) return 0;
    for (auto &kv : pl->graphs)
        if (std::get<2>(kv.first) == int(use_sr != 0)) return kv.second.kernel_nodes;
    return 0;
}

// ---------------------------------------------------------------------------
// Device-resident solve loop (solver.py:280-330).  One graph launch runs the
// whole loop: a WHILE conditional node whose body is
//   k_solve_pre  -> operator of this iteration (schedule_operator,
//                   solver.py:122-144: N_GAN cadence, latch -> second operator)
//   IF(sr)       -> the captured SR V-cycle
//   IF(spline)   -> the captured spline V-cycle
//   k_solve_post -> record (diff_norm, residual rms, operator, latched), latch
//                   on diff <= S_thres, continue while diff >= tol and
//                   iterations < N_iter.
// No host round trip per cycle; the ConvergenceLog is read back once.

namespace {

__global__ void k_solve_init(int *state) {
    state[0] = 0;   // iterations done
    state[1] = 0;   // latched
    state[2] = 0;   // operator of the current iteration
    state[3] = 0;   // iterations (output)
}

__global__ void k_solve_pre(int *state, int mode, int cadence, int first_sr, int ngan_one,
                            cudaGraphConditionalHandle h_sr, cudaGraphConditionalHandle h_sp) {
    const int it = state[0] + 1;
    const int latched = state[1];
    int sr;
    if (mode == 0) sr = 0;
    else if (mode == 1) sr = 1;
    else if (latched) sr = !first_sr;
    else if (ngan_one) sr = it & 1;
    else sr = (it % cadence != 0) ? first_sr : !first_sr;
    state[2] = sr;
    cudaGraphSetConditional(h_sr, sr ? 1u : 0u);
    cudaGraphSetConditional(h_sp, sr ? 0u : 1u);
}

__global__ void k_solve_post(int *state, const double *stats, double *rec, int n_iter, double tol, double s_thres,
                             cudaGraphConditionalHandle h_while) {
    const int it = state[0] + 1;
    const double d = stats[0];
    double *r = rec + 4 * (it - 1);
    r[0] = d;
    r[1] = stats[1];
    r[2] = double(state[2]);
    r[3] = double(state[1]);
    if (!state[1] && d <= s_thres) state[1] = 1;
    state[0] = it;
    state[3] = it;
    cudaGraphSetConditional(h_while, (!(d < tol) && it < n_iter) ? 1u : 0u);
}

int add_kernel(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *deps, size_t ndeps, void *func,
               void **args) {
    cudaKernelNodeParams kp{};
    kp.func = func;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.sharedMemBytes = 0;
    kp.kernelParams = args;
    MGSR_CUDA_TRY(cudaGraphAddKernelNode(node, g, deps, ndeps, &kp));
    return MGSR_OK;
}

int add_if(cudaGraph_t g, cudaGraphNode_t *node, const cudaGraphNode_t *dep, cudaGraphConditionalHandle h,
           cudaGraphConditionalNodeType type, cudaGraph_t *body) {
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = type;
    np.conditional.size = 1;
    MGSR_CUDA_TRY(cudaGraphAddNode(node, g, dep, dep ? 1 : 0, &np));
    *body = np.conditional.phGraph_out[0];
    return MGSR_OK;
}

// capture one V-cycle's kernel sequence into an existing (conditional body) graph
int capture_cycle_into(mgsr_plan *pl, cudaGraph_t body, double *p, const double *f, int use_sr) {
    MGSR_CUDA_TRY(cudaStreamBeginCaptureToGraph(pl->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    const bool mk = pl->capturing_markers;
    pl->capturing_markers = false;
    int r = record_vcycle(pl, p, f, use_sr, pl->cap);
    pl->capturing_markers = mk;
    cudaGraph_t out = nullptr;
    cudaError_t e = cudaStreamEndCapture(pl->cap, &out);
    if (r) return r;
    if (e != cudaSuccess) { set_error(std::string("solve body capture: ") + cudaGetErrorString(e)); return MGSR_E_CUDA; }
    return MGSR_OK;
}

}  // namespace

extern "C" int mgsr_plan_solve(mgsr_plan *pl, double *p, const double *f, int32_t mode, int32_t n_iter, double tol,
                               double s_thres, int32_t cadence, int32_t first_sr, int32_t ngan_one,
                               double *records_dev, int32_t *iterations_dev, void *stream) {
    if (!pl || !p || !f || !records_dev || !iterations_dev || n_iter < 1 || mode < 0 || mode > 2 || cadence < 1) {
        set_error("bad argument");
        return MGSR_E_BAD_ARG;
    }
    if (mode != 0 && !pl->gen) { set_error("SR prolongation requires generator weights"); return MGSR_E_BAD_ARG; }
    if (graphs_disabled()) {
        set_error("the device-resident solve loop needs CUDA graphs (disabled by MGSR_NO_GRAPH or an attached "
                  "profiler); use the per-cycle loop");
        return MGSR_E_UNSUPPORTED;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!pl->solve_state) MGSR_CUDA_TRY(cudaMalloc(&pl->solve_state, 4 * sizeof(int)));
    if (pl->rec_cap < n_iter) {
        // records are baked into the graphs: drop them with the old buffer
        for (auto &kv : pl->solves) {
            cudaGraphExecDestroy(kv.second.exec);
            cudaGraphDestroy(kv.second.graph);
        }
        pl->solves.clear();
        if (pl->solve_rec) cudaFree(pl->solve_rec);
        MGSR_CUDA_TRY(cudaMalloc(&pl->solve_rec, 4 * sizeof(double) * size_t(n_iter)));
        pl->rec_cap = n_iter;
    }
    auto key = std::make_tuple(p, f, int(mode), int(n_iter), tol, s_thres, int(cadence), int(first_sr), int(ngan_one));
    auto it = pl->solves.find(key);
    if (it == pl->solves.end() && pl->solves.size() >= 8) {
        for (auto &kv : pl->solves) {
            cudaGraphExecDestroy(kv.second.exec);
            cudaGraphDestroy(kv.second.graph);
        }
        pl->solves.clear();
    }
    if (it == pl->solves.end()) {
        MGSR_CUDA_TRY(cudaStreamSynchronize(st));
        cudaGraph_t g = nullptr;
        MGSR_CUDA_TRY(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle hw, hs, hp;
        MGSR_CUDA_TRY(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
        MGSR_CUDA_TRY(cudaGraphConditionalHandleCreate(&hs, g, 0, cudaGraphCondAssignDefault));
        MGSR_CUDA_TRY(cudaGraphConditionalHandleCreate(&hp, g, 0, cudaGraphCondAssignDefault));
        int *state = pl->solve_state;
        double *rec = pl->solve_rec;
        double *stats = sc(pl, SC_STATS);
        cudaGraphNode_t n_init, n_while, n_pre, n_if_sr, n_if_sp, n_post;
        void *a_init[] = {&state};
        int r = add_kernel(g, &n_init, nullptr, 0, reinterpret_cast<void *>(k_solve_init), a_init);
        cudaGraph_t body = nullptr, body_sr = nullptr, body_sp = nullptr;
        if (!r) r = add_if(g, &n_while, &n_init, hw, cudaGraphCondTypeWhile, &body);
        int mode_ = mode, cad = cadence, fs_ = first_sr, g1 = ngan_one, nit = n_iter;
        double tol_ = tol, sth = s_thres;
        void *a_pre[] = {&state, &mode_, &cad, &fs_, &g1, &hs, &hp};
        if (!r) r = add_kernel(body, &n_pre, nullptr, 0, reinterpret_cast<void *>(k_solve_pre), a_pre);
        // both IF nodes always exist (every handle the controller sets must belong to a node); a pure
        // mode leaves the other operator's body empty
        if (!r) r = add_if(body, &n_if_sr, &n_pre, hs, cudaGraphCondTypeIf, &body_sr);
        if (!r) r = add_if(body, &n_if_sp, &n_if_sr, hp, cudaGraphCondTypeIf, &body_sp);
        void *a_post[] = {&state, &stats, &rec, &nit, &tol_, &sth, &hw};
        if (!r) r = add_kernel(body, &n_post, &n_if_sp, 1, reinterpret_cast<void *>(k_solve_post), a_post);
        if (!r && mode != 0) r = capture_cycle_into(pl, body_sr, p, f, 1);
        if (!r && mode != 1) r = capture_cycle_into(pl, body_sp, p, f, 0);
        mgsr_plan::SolveGraph SG;
        SG.graph = g;
        if (!r) {
            cudaError_t e = cudaGraphInstantiate(&SG.exec, g, 0);
            if (e != cudaSuccess) { set_error(std::string("solve graph instantiate: ") + cudaGetErrorString(e)); r = MGSR_E_CUDA; }
        }
        if (r) { cudaGraphDestroy(g); return r; }
        it = pl->solves.emplace(key, SG).first;
    }
    MGSR_CUDA_TRY(cudaGraphLaunch(it->second.exec, st));
    MGSR_CUDA_TRY(cudaMemcpyAsync(records_dev, pl->solve_rec, 4 * sizeof(double) * size_t(n_iter),
                                  cudaMemcpyDeviceToDevice, st));
    MGSR_CUDA_TRY(cudaMemcpyAsync(iterations_dev, pl->solve_state + 3, sizeof(int), cudaMemcpyDeviceToDevice, st));
    return MGSR_OK;
}

// ---------------------------------------------------------------------------
// Batched device-resident solves (BASELINE config 5: independent right-hand sides of one size solved
// concurrently with batch-N generator inference).  B plans of one configuration run their solve loops
// in lockstep inside ONE graph launch: a WHILE node whose body is
//   k_batch_pre   -> per grid: operator of its own iteration (its own N_GAN cadence and latch), the
//                    IF handles (active / spline this iteration / SR this iteration) and the device list
//                    of the grids that prolong by SR;
//   per grid, in parallel branches: IF(active) the cycle down to the SR levels (record_down);
//   per SR level, finest last: IF(spline) that grid's spline prolongation, and ONE batched generator
//                    launch over the listed grids' windows followed by IF(SR) that grid's mean + add;
//   per grid: IF(active) the logging pass;
//   k_batch_post  -> per grid: record, latch, deactivate on tol / N_iter; loop while any grid is active.
// Every grid sees exactly its single-solve kernel sequence, so results are bitwise those of
// mgsr_plan_solve on each grid.

namespace {

__global__ void k_batch_init(int *state, int *active, int B) {
    const int r = threadIdx.x;
    if (r < B) {
        state[4 * r] = state[4 * r + 1] = state[4 * r + 2] = state[4 * r + 3] = 0;
        active[r] = 1;
    }
}

// handles: [kind 3][grid B][nh] -- every IF node owns its handle; kind 0 = active, 1 = spline this
// iteration, 2 = SR this iteration
__global__ void k_batch_pre(int *state, const int *active, int B, int mode, int cadence, int first_sr, int ngan_one,
                            const cudaGraphConditionalHandle *hdl, int nh, int n0, int n1, int n2, int *list,
                            int *count) {
    __shared__ int flag[1024];
    const int r = threadIdx.x;
    int act = 0, sr = 0;
    if (r < B) {
        int *st = state + 4 * r;
        act = active[r];
        if (act) {   // k_solve_pre's schedule (solver.py:122-144)
            const int it = st[0] + 1, latched = st[1];
            if (mode == 0) sr = 0;
            else if (mode == 1) sr = 1;
            else if (latched) sr = !first_sr;
            else if (ngan_one) sr = it & 1;
            else sr = (it % cadence != 0) ? first_sr : !first_sr;
            st[2] = sr;
        }
        const unsigned v[3] = {act ? 1u : 0u, (act && !sr) ? 1u : 0u, (act && sr) ? 1u : 0u};
        const int used[3] = {n0, n1, n2};   // IF nodes of each kind per grid
        for (int k = 0; k < 3; ++k)
            for (int j = 0; j < used[k]; ++j) cudaGraphSetConditional(hdl[(size_t(k) * B + r) * nh + j], v[k]);
    }
    flag[r] = act && sr;
    __syncthreads();
    if (r == 0) {
        int c = 0;
        for (int k = 0; k < B; ++k)
            if (flag[k]) list[c++] = k;
        *count = c;
    }
}

__global__ void k_batch_post(int *state, int *active, int B, const double *const *stats, double *rec, int n_iter,
                             double tol, double s_thres, cudaGraphConditionalHandle h_while) {
    const int r = threadIdx.x;
    int more = 0;
    if (r < B && active[r]) {   // k_solve_post per grid
        int *st = state + 4 * r;
        const int it = st[0] + 1;
        const double d = stats[r][0];
        double *rr = rec + (size_t(r) * n_iter + (it - 1)) * 4;
        rr[0] = d;
        rr[1] = stats[r][1];
        rr[2] = double(st[2]);
        rr[3] = double(st[1]);
        if (!st[1] && d <= s_thres) st[1] = 1;
        st[0] = it;
        st[3] = it;
        more = (!(d < tol) && it < n_iter) ? 1 : 0;
        active[r] = more;
    }
    more = __syncthreads_or(more);
    if (r == 0) cudaGraphSetConditional(h_while, more ? 1u : 0u);
}

struct BatchGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    void *mem = nullptr;   // device: state, active, records, list, count, handles, pointer arrays, SR buffers
    int *state = nullptr, *active = nullptr, *list = nullptr, *count = nullptr;
    double *rec = nullptr;
    int n_iter = 0;
    cudaStream_t cap = nullptr;
};
using BatchKey = std::tuple<std::vector<const void *>, int, int, double, double, int, int, int>;
std::map<BatchKey, BatchGraph> g_batches;

void batch_free(BatchGraph &G) {
    if (G.exec) cudaGraphExecDestroy(G.exec);
    if (G.graph) cudaGraphDestroy(G.graph);
    if (G.mem) cudaFree(G.mem);
    if (G.cap) cudaStreamDestroy(G.cap);
    G = BatchGraph{};
}

int capture_into(cudaGraph_t body, cudaStream_t cap, const std::function<int(cudaStream_t)> &fn) {
    MGSR_CUDA_TRY(cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    int r = fn(cap);
    cudaGraph_t out = nullptr;
    cudaError_t e = cudaStreamEndCapture(cap, &out);
    if (r) return r;
    if (e != cudaSuccess) { set_error(std::string("batch capture: ") + cudaGetErrorString(e)); return MGSR_E_CUDA; }
    return MGSR_OK;
}

int build_batch(BatchGraph &G, mgsr_plan *const *pls, int B, double *const *p, const double *const *f, int mode,
                int n_iter, double tol, double s_thres, int cadence, int first_sr, int ngan_one) {
    mgsr_plan *p0 = pls[0];
    const int L = int(p0->sides.size());
    const bool tc = tensor_core_precision(p0->cfg.precision) && p0->gen && p0->gen->tc_blob;
    // the SR prolongations: from level l into l - 1 where the mask bit l - 1 is set (and the grid allows SR)
    std::vector<int> sr_lev(L, 0);
    int stop = 0;
    if (mode != 0 && p0->gen)
        for (int l = 1; l < L; ++l) {
            const int nc = p0->sides[l];
            if (((p0->cfg.sr_level_mask >> (l - 1)) & 1u) && nc >= 6 && nc % 2 == 0) {
                sr_lev[l] = 1;
                stop = std::max(stop, l);
            }
        }
    // device memory
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 255) & ~size_t(255); return o; };
    const size_t o_state = take(sizeof(int) * 4 * B), o_active = take(sizeof(int) * B), o_list = take(sizeof(int) * B),
                 o_count = take(sizeof(int)), o_rec = take(sizeof(double) * 4 * size_t(B) * n_iter),
                 o_h = take(sizeof(cudaGraphConditionalHandle) * 3 * B * (L + 2)), o_stats = take(sizeof(double *) * B),
                 o_cs = take(sizeof(double *) * B * L);
    size_t o_srbuf = 0, o_srws = 0, srws_bytes = 0;
    int64_t nf_max = 0;
    for (int l = 1; l < L; ++l)
        if (sr_lev[l] && tc && p0->sides[l - 1] == 2 * p0->sides[l]) {
            nf_max = std::max<int64_t>(nf_max, p0->sides[l - 1]);
            if (tc_batch_workspace_bytes(p0->sides[l], B) > srws_bytes) {
                srws_bytes = tc_batch_workspace_bytes(p0->sides[l], B);
            }
        }
    if (nf_max) {
        o_srbuf = take(sizeof(double) * size_t(B) * nf_max * nf_max);
        o_srws = take(srws_bytes);
    }
    MGSR_CUDA_TRY(cudaMalloc(&G.mem, off));
    char *m = static_cast<char *>(G.mem);
    G.state = reinterpret_cast<int *>(m + o_state);
    G.active = reinterpret_cast<int *>(m + o_active);
    G.list = reinterpret_cast<int *>(m + o_list);
    G.count = reinterpret_cast<int *>(m + o_count);
    G.rec = reinterpret_cast<double *>(m + o_rec);
    G.n_iter = n_iter;
    auto *hdev = reinterpret_cast<cudaGraphConditionalHandle *>(m + o_h);
    auto *stats_dev = reinterpret_cast<const double **>(m + o_stats);
    auto *cs_dev = reinterpret_cast<const double **>(m + o_cs);
    double *srbuf = nf_max ? reinterpret_cast<double *>(m + o_srbuf) : nullptr;
    void *srws = nf_max ? m + o_srws : nullptr;
    MGSR_CUDA_TRY(cudaStreamCreateWithFlags(&G.cap, cudaStreamNonBlocking));

    cudaGraph_t g = nullptr;
    MGSR_CUDA_TRY(cudaGraphCreate(&g, 0));
    G.graph = g;
    cudaGraphConditionalHandle hw;
    MGSR_CUDA_TRY(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    // every IF node owns a handle: [kind][grid][j], j < nh = L + 2 (kinds: 0 active, 1 spline, 2 SR)
    const int nh = L + 2;
    std::vector<cudaGraphConditionalHandle> hh(size_t(3) * B * nh, 0);
    std::vector<int> hused(3 * B, 0);
    auto new_handle = [&](int kind, int b, cudaGraphConditionalHandle *out) -> int {
        int &u = hused[kind * B + b];
        if (u >= nh) { set_error("batch: too many conditional nodes"); return MGSR_E_UNSUPPORTED; }
        MGSR_CUDA_TRY(cudaGraphConditionalHandleCreate(out, g, 0, cudaGraphCondAssignDefault));
        hh[(size_t(kind) * B + b) * nh + u++] = *out;
        return MGSR_OK;
    };
    std::vector<const double *> stats_h(B), cs_h(size_t(B) * L, nullptr);
    for (int b = 0; b < B; ++b) {
        stats_h[b] = sc(pls[b], SC_STATS);
        for (int l = 1; l < L; ++l) cs_h[size_t(l) * B + b] = pls[b]->d[l];
    }
    MGSR_CUDA_TRY(cudaMemcpy(stats_dev, stats_h.data(), sizeof(double *) * B, cudaMemcpyHostToDevice));
    MGSR_CUDA_TRY(cudaMemcpy(cs_dev, cs_h.data(), sizeof(double *) * B * L, cudaMemcpyHostToDevice));

    cudaGraphNode_t n_init, n_while, n_pre, n_post;
    int *state = G.state, *active = G.active, *list = G.list, *count = G.count;
    double *rec = G.rec;
    int B_ = B, mode_ = mode, cad = cadence, fs_ = first_sr, g1 = ngan_one, nit = n_iter;
    double tol_ = tol, sth = s_thres;
    void *a_init[] = {&state, &active, &B_};
    cudaKernelNodeParams kpi{};
    kpi.func = reinterpret_cast<void *>(k_batch_init);
    kpi.gridDim = dim3(1);
    kpi.blockDim = dim3(1024);
    kpi.kernelParams = a_init;
    int r = MGSR_OK;
    MGSR_CUDA_TRY(cudaGraphAddKernelNode(&n_init, g, nullptr, 0, &kpi));
    cudaGraph_t body = nullptr;
    if (!r) r = add_if(g, &n_while, &n_init, hw, cudaGraphCondTypeWhile, &body);
    const cudaGraphConditionalHandle *hdl = hdev;
    int nh_ = nh, nu[3] = {0, 0, 0};   // the per-kind counts are filled in once the body is built
    void *a_pre[] = {&state, &active, &B_, &mode_, &cad, &fs_, &g1, &hdl, &nh_, &nu[0], &nu[1], &nu[2], &list, &count};
    cudaKernelNodeParams kp{};
    kp.func = reinterpret_cast<void *>(k_batch_pre);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1024);
    kp.kernelParams = a_pre;
    if (!r) MGSR_CUDA_TRY(cudaGraphAddKernelNode(&n_pre, body, nullptr, 0, &kp));
    cudaKernelNodeParams kp_pre = kp;
    cudaGraphNode_t join = n_pre;
    // one IF node per grid after `join`, each capturing fn(b, stream); returns the join of them all (plus extra)
    auto per_grid = [&](int kind, const std::function<int(int, cudaStream_t)> &fn,
                        std::vector<cudaGraphNode_t> extra) -> int {
        std::vector<cudaGraphNode_t> ends = std::move(extra);
        for (int b = 0; b < B; ++b) {
            cudaGraphNode_t nd;
            cudaGraph_t bd = nullptr;
            cudaGraphConditionalHandle h;
            if (int e = new_handle(kind, b, &h)) return e;
            if (int e = add_if(body, &nd, &join, h, cudaGraphCondTypeIf, &bd)) return e;
            if (int e = capture_into(bd, G.cap, [&](cudaStream_t cs) { return fn(b, cs); })) return e;
            ends.push_back(nd);
        }
        cudaGraphNode_t j;
        MGSR_CUDA_TRY(cudaGraphAddEmptyNode(&j, body, ends.data(), ends.size()));
        join = j;
        return MGSR_OK;
    };
    // spline iterations: the whole cycle (its small-grid fusions included) up to the logging pass; SR iterations:
    // the cycle down to the finest SR level, then level-major below
    {
        std::vector<cudaGraphNode_t> sp;
        const cudaGraphNode_t j0 = join;
        for (int b = 0; b < B && !r; ++b) {
            cudaGraphNode_t nd;
            cudaGraph_t bd = nullptr;
            cudaGraphConditionalHandle h;
            r = new_handle(1, b, &h);
            if (!r) r = add_if(body, &nd, &j0, h, cudaGraphCondTypeIf, &bd);
            if (!r) r = capture_into(bd, G.cap, [&](cudaStream_t cs) { return record_vcycle(pls[b], p[b], f[b], 0, cs); });
            sp.push_back(nd);
        }
        if (!r) r = per_grid(2, [&](int b, cudaStream_t cs) {
            return stop > 0 ? record_down(pls[b], p[b], f[b], 1, cs, stop) : record_vcycle(pls[b], p[b], f[b], 1, cs);
        }, sp);
    }
    for (int l = stop; !r && l >= 1; --l) {
        const bool batched = sr_lev[l] && tc && p0->sides[l - 1] == 2 * p0->sides[l];
        if (l == 1 && !sr_lev[1]) {   // the cycle's spline top prolongation and its logging pass (maybe fused)
            r = per_grid(2, [&](int b, cudaStream_t cs) { return record_top(pls[b], p[b], f[b], 1, cs); }, {});
            continue;
        }
        if (!batched) {   // spline level between SR levels, fp32 generator, or a multi-pass ratio: per grid
            r = per_grid(2, [&](int b, cudaStream_t cs) { return prolong_level(pls[b], l, 1, cs); }, {});
            continue;
        }
        // one generator launch over the SR grids' windows -> srbuf + b nf^2, then per grid mean + add
        const int nc = p0->sides[l];
        const double log_lo = std::log10(p0->cfg.p_min), span = std::log10(p0->cfg.p_max) - log_lo;
        cudaGraph_t sg = nullptr;
        MGSR_CUDA_TRY(cudaGraphCreate(&sg, 0));
        const double *const *csl = cs_dev + size_t(l) * B;
        r = capture_into(sg, G.cap, [&](cudaStream_t cs) {
            return launch_sr_pass_tc_batch(p0->gen, csl, B, list, count, nc, log_lo, span, srbuf, srws, srws_bytes, cs,
                                           p0->cfg.precision != MGSR_PREC_BF16);
        });
        cudaGraphNode_t n_sr;
        if (!r) MGSR_CUDA_TRY(cudaGraphAddChildGraphNode(&n_sr, body, &join, 1, sg));
        cudaGraphDestroy(sg);
        if (r) break;
        const int64_t nf = 2LL * nc;
        join = n_sr;
        r = per_grid(2, [&](int b, cudaStream_t cs) { return sr_add_level(pls[b], l, srbuf + size_t(b) * nf * nf, cs); }, {});
    }
    if (!r && stop > 0 && sr_lev[1])   // after an SR top prolongation: the logging pass
        r = per_grid(2, [&](int b, cudaStream_t cs) { return record_finalize(pls[b], p[b], f[b], cs); }, {});
    // the handle table, and the per-kind node counts into the controller's parameters (uniform across grids)
    if (!r) MGSR_CUDA_TRY(cudaMemcpy(hdev, hh.data(), sizeof(cudaGraphConditionalHandle) * hh.size(), cudaMemcpyHostToDevice));
    for (int k = 0; k < 3 && !r; ++k) {
        nu[k] = hused[k * B];
        for (int b = 1; b < B; ++b)
            if (hused[k * B + b] != nu[k]) { set_error("batch: uneven conditional nodes"); r = MGSR_E_UNSUPPORTED; }
    }
    if (!r) MGSR_CUDA_TRY(cudaGraphKernelNodeSetParams(n_pre, &kp_pre));
    const double *const *stats_c = stats_dev;
    void *a_post[] = {&state, &active, &B_, &stats_c, &rec, &nit, &tol_, &sth, &hw};
    kp.func = reinterpret_cast<void *>(k_batch_post);
    kp.kernelParams = a_post;
    if (!r) MGSR_CUDA_TRY(cudaGraphAddKernelNode(&n_post, body, &join, 1, &kp));
    if (!r) {
        cudaError_t e = cudaGraphInstantiate(&G.exec, g, 0);
        if (e != cudaSuccess) { set_error(std::string("batch graph instantiate: ") + cudaGetErrorString(e)); r = MGSR_E_CUDA; }
    }
    return r;
}

}  // namespace

extern "C" int mgsr_plan_solve_batch(mgsr_plan *const *plans, int32_t B, double *const *p, const double *const *f,
                                     int32_t mode, int32_t n_iter, double tol, double s_thres, int32_t cadence,
                                     int32_t first_sr, int32_t ngan_one, double *records_dev, int32_t *iterations_dev,
                                     void *stream) {
    if (!plans || !p || !f || !records_dev || !iterations_dev || B < 1 || B > 1024 || n_iter < 1 || mode < 0 ||
        mode > 2 || cadence < 1) {
        set_error("bad argument");
        return MGSR_E_BAD_ARG;
    }
    for (int b = 0; b < B; ++b) {
        if (!plans[b] || !p[b] || !f[b]) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
        const mgsr_plan *a = plans[0], *c = plans[b];
        if (c->sides != a->sides || c->gen != a->gen || c->cfg.precision != a->cfg.precision ||
            c->cfg.sr_level_mask != a->cfg.sr_level_mask || c->cfg.n_smooth != a->cfg.n_smooth ||
            c->cfg.coarse_sweeps != a->cfg.coarse_sweeps || c->cfg.p_min != a->cfg.p_min || c->cfg.p_max != a->cfg.p_max) {
            set_error("solve_batch: the plans must share one configuration and generator");
            return MGSR_E_BAD_ARG;
        }
        for (int k = 0; k < b; ++k)
            if (plans[k] == plans[b]) { set_error("solve_batch: a plan appears twice"); return MGSR_E_BAD_ARG; }
    }
    if (mode != 0 && !plans[0]->gen) { set_error("SR prolongation requires generator weights"); return MGSR_E_BAD_ARG; }
    if (plans[0]->sides[0] <= kSmallN) { set_error("solve_batch: grids of side <= 64 run per grid"); return MGSR_E_UNSUPPORTED; }
    if (graphs_disabled()) {
        set_error("the batched solve loop needs CUDA graphs (disabled by MGSR_NO_GRAPH or an attached profiler)");
        return MGSR_E_UNSUPPORTED;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<const void *> ids;
    for (int b = 0; b < B; ++b) { ids.push_back(plans[b]); ids.push_back(p[b]); ids.push_back(f[b]); }
    BatchKey key{ids, int(mode), int(n_iter), tol, s_thres, int(cadence), int(first_sr), int(ngan_one)};
    auto it = g_batches.find(key);
    if (it == g_batches.end()) {
        MGSR_CUDA_TRY(cudaStreamSynchronize(st));
        if (g_batches.size() >= 4) {   // bounded cache
            MGSR_CUDA_TRY(cudaDeviceSynchronize());
            for (auto &kv : g_batches) batch_free(kv.second);
            g_batches.clear();
        }
        BatchGraph G;
        std::vector<bool> mk(B);   // no event-record markers inside conditional bodies
        for (int b = 0; b < B; ++b) { mk[b] = plans[b]->capturing_markers; plans[b]->capturing_markers = false; }
        int r = build_batch(G, plans, B, p, f, mode, n_iter, tol, s_thres, cadence, first_sr, ngan_one);
        for (int b = 0; b < B; ++b) plans[b]->capturing_markers = mk[b];
        if (r) { batch_free(G); return r; }
        it = g_batches.emplace(key, G).first;
    }
    BatchGraph &G = it->second;
    MGSR_CUDA_TRY(cudaGraphLaunch(G.exec, st));
    MGSR_CUDA_TRY(cudaMemcpyAsync(records_dev, G.rec, 4 * sizeof(double) * size_t(B) * n_iter, cudaMemcpyDeviceToDevice, st));
    for (int b = 0; b < B; ++b)
        MGSR_CUDA_TRY(cudaMemcpyAsync(iterations_dev + b, G.state + 4 * b + 3, sizeof(int), cudaMemcpyDeviceToDevice, st));
    return MGSR_OK;
}

// drop the batched graphs that captured a plan's buffers (called by mgsr_plan_destroy)
void batch_forget(const mgsr_plan *pl) {
    bool any = false;
    for (auto &kv : g_batches)
        for (size_t i = 0; i < std::get<0>(kv.first).size(); i += 3)
            if (std::get<0>(kv.first)[i] == pl) any = true;
    if (!any) return;
    cudaDeviceSynchronize();
    for (auto it = g_batches.begin(); it != g_batches.end();) {
        bool hit = false;
        for (size_t i = 0; i < std::get<0>(it->first).size(); i += 3)
            if (std::get<0>(it->first)[i] == pl) hit = true;
        if (hit) { batch_free(it->second); it = g_batches.erase(it); }
        else ++it;
    }
}
