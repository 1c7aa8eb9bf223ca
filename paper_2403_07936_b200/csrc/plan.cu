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

// correction(rhs_l, l) of solver.py:181-190; leaves the gauge-fixed result in d[l].
int correction(mgsr_plan *pl, int l, int use_sr, cudaStream_t st) {
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
    if ((r = correction(pl, l + 1, use_sr, st))) return r;
    // d[l] = (d[l] - d_mean) + up  (in place: elementwise)
    const double *bshift = n <= kSmallN ? nullptr : d_mean(pl, l);
    return prolong_into(pl, l + 1, use_sr, pl->d[l], bshift, pl->d[l], nullptr, st);
}

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
    const double *bshift = n <= kSmallN ? nullptr : sc(pl, SC_S_MEAN);
    if ((r = prolong_into(pl, 1, use_sr, pl->S, bshift, pl->S, sc(pl, SC_OUT_MEAN), st))) return r;
    r = launch_finalize(pl->S, sc(pl, SC_OUT_MEAN), p, fs, n, sc(pl, SC_ACC), sc(pl, SC_STATS), slot(pl, 0), st);
    if (r) return r;
    if (mk) MGSR_CUDA_TRY(cudaEventRecordWithFlags(pl->cap_ev[5], st, cudaEventRecordExternal));
    return MGSR_OK;
}

}  // namespace

extern "C" int mgsr_plan_create(const mgsr_plan_config *cfg, const mgsr_gen *gen, mgsr_plan **out) {
    if (!cfg || !out) { set_error("bad argument"); return MGSR_E_BAD_ARG; }
    if (cfg->n_smooth < 1 || cfg->coarse_sweeps < 1) { set_error("sweep counts must be positive"); return MGSR_E_BAD_ARG; }
    if (cfg->r_min < 2 || cfg->r_min % 2) { set_error("r_min must be an even integer >= 2"); return MGSR_E_BAD_ARG; }
    if (!valid_precision(cfg->precision)) { set_error("precision must be one of fp32, bf16, fp16"); return MGSR_E_BAD_ARG; }
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

extern "C" int mgsr_plan_destroy(mgsr_plan *pl) {
    if (!pl) return MGSR_OK;
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
