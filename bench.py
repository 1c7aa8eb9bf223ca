#!/usr/bin/env python
"""Benchmark: V-cycles/s (and GUpdates/s) of the 4096^2 V-cycle with GAN
prolongation on B200 -- BASELINE.json config 4.

Workload (``config.workload``): periodic 4096^2 grid, N_step=1 ladder
4096 -> 8 (10 levels), N_smooth=2, coarse_sweeps=10, SR ("GAN") prolongation
at the 3 finest prolongations (2048->4096, 1024->2048, 512->1024; 1,369,100
windows of 6x6), Keys spline below; generator = reference architecture, B=8
residual blocks; weights: the reference's trained-weights slot (pkg/artifacts)
is empty, so BASELINE's "trained weights if present" is filled by
artifacts/trained_b8.mgsr, produced by the reference's own documented
training pipeline (artifacts/PROVENANCE.md); ``--weights he`` selects the
seeded He-normal init (``random_weights(8, 0)``).  Speed does not depend on
the weights; the fp16 field parity bar (1e-2 relL2) does: trained weights
meet it, He-init weights amplify operand rounding (2e-2).
fp16 tcgen05 operands with fp32 accumulation; fp64 stencils.  RHS: seeded Gaussian
random field k^-5/3 + 32 blobs scaled to p_rms = 1e-4 (in the SR band).
A step = one V-cycle + the solve loop's logging pass (diff and residual
norms), one CUDA-graph launch.  Inputs (134 MB per fp64 grid) exceed the
126 MB L2, so no explicit flush is needed.

Multi-GPU: the path does not shard (one grid per GPU) ->
replicas only: each rank runs its own seeded replica, value = sum over ranks
of cycles / max-over-ranks time ("scaling": "weak").

``--impl reference`` times the reference's own CPU implementation (compiled
from its sources into oracle/_ref) on a bounded sample per step and projects
the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "V-cycles/s and GUpdates/s at 4096² (GAN prolong) on 1 B200; % HBM / tensor roofline"
UNIT = "V-cycles/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--mode", default="gan", choices=["gan", "spline"])
    ap.add_argument("--precision", default="fp16", choices=["fp16", "bf16", "fp32"])
    ap.add_argument("--sr-levels", type=int, default=3)
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--weights", default="trained", choices=["trained", "he"])
    ap.add_argument("--n-smooth", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    # launch-path self-test (CPU, gloo): every rank fakes its timed region; exercises the torchrun
    # self-launch, the rendezvous, the max-over-ranks reduction and the whole-job value
    ap.add_argument("--plumbing-test", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def self_launch(args) -> None:
    """``--gpus N`` (N > 1) outside torchrun: re-exec this script under torch.distributed.run with
    one rank per GPU (127.0.0.1 rendezvous) and exit with its status.  NCCL's INIT lines (the
    communicator setup over NVLink) go to stderr, so stdout stays the single JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    if not args.plumbing_test:
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    sys.exit(subprocess.call(cmd, env=env))


# ---------------------------------------------------------------------------
# algorithmic work model; credits only executed work

def window_macs(blocks: int, kept_px: int) -> int:
    head = 36 * 64 * 81            # 3 identical input channels folded -> 81 taps executed
    body = 2 * blocks * 36 * 64 * 576
    post = 36 * 64 * 576
    up = 36 * 256 * 576
    tail = kept_px * 3 * 64 * 81   # tail evaluated only at the stitched (kept) pixels
    return head + body + post + up + tail


def pass_flops(nc: int, blocks: int) -> float:
    """FLOPs of one ratio-2 SR pass on an nc x nc coarse grid (stitch_plan bands)."""
    npos = nc // 2 - 2
    tot = 0
    for side_i in range(npos):
        ri = 8 if side_i in (0, npos - 1) else 4
        if npos == 1:
            ri = 12
        for side_j in range(npos):
            rj = 8 if side_j in (0, npos - 1) else 4
            if npos == 1:
                rj = 12
            tot += window_macs(blocks, ri * rj)
    return 2.0 * tot


def pass_flops_fast(nc: int, blocks: int) -> float:
    npos = nc // 2 - 2
    inner = max(npos - 2, 0)
    n_int, n_edge, n_corner = inner * inner, 4 * inner, 4
    return 2.0 * (n_int * window_macs(blocks, 16) + n_edge * window_macs(blocks, 32)
                  + n_corner * window_macs(blocks, 64))


def gs_bytes(n: int, fused_rc: bool = True) -> float:
    """Compulsory bytes of the finest temporally blocked GS launch: read p, f; write p
    (+ the injected coarse residual)."""
    return n * n * (24.0 + (2.0 if fused_rc else 0.0))


# ---------------------------------------------------------------------------
# clocks sampling during the timed region

class Clocks:
    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def weights_path(kind: str, blocks: int):
    path = os.path.join(ROOT, "artifacts", f"trained_b{blocks}.mgsr")
    return path if kind == "trained" and os.path.exists(path) else None


def bench_weights(kind: str, blocks: int, srmodel_mod):
    """MGSR1 trained weights (artifacts/) or the seeded He-normal init; same loader API in the
    reference's srmodel and ours."""
    path = weights_path(kind, blocks)
    return srmodel_mod.load_weights(path) if path else srmodel_mod.random_weights(blocks, 0)


def load_traffic(mode):
    """ncu dram bytes per launch of the dominant kernel, if a capture summary is committed."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(mode)
    except OSError:
        return None


# ---------------------------------------------------------------------------
# workload

def make_inputs(n: int, seed: int, mode: str):
    from paper_2403_07936_b200 import datagen
    f = datagen.grf_blobs_rhs(n, seed=seed, kmax=min(256.0, n / 4))
    f = datagen.scale_to_p_rms(f, 1e-4)
    rng = __import__("numpy").random.default_rng(seed)
    p0 = rng.uniform(-1e-4, 1e-4, size=(n, n))
    return f - f.mean(), p0 - p0.mean()


def reduce_max(x: float, dist, device) -> float:
    """Max over ranks (the timing rule: a multi-GPU number is the slowest rank's)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_value(steps: int, ms_max: float, world: int) -> float:
    """Whole-job V-cycles/s of `world` independent replicas (weak scaling, replicas only)."""
    return steps / (ms_max / 1e3) * world


def replica_seed(rank: int) -> int:
    """Each replica solves its own seeded right-hand side."""
    return 1000 + rank


def run_mine(args, rank: int, world: int, dist):
    import numpy as np
    import torch

    from paper_2403_07936_b200 import _lib, ops, srmodel
    from paper_2403_07936_b200.solver import RunConfig, VCyclePlan

    torch.cuda.set_device(rank % max(torch.cuda.device_count(), 1))
    dev = torch.device("cuda")
    n = args.n
    cfg = RunConfig(N_step=1, r_min=8, N_smooth=args.n_smooth, coarse_sweeps=10)
    weights = bench_weights(args.weights, args.blocks, srmodel) if args.mode == "gan" else None
    op = "sr" if args.mode == "gan" else "spline"
    plan = VCyclePlan(n, cfg, weights, precision=args.precision, sr_levels=args.sr_levels)
    f_np, p_np = make_inputs(n, replica_seed(rank), args.mode)
    f = torch.from_numpy(f_np).to(dev)
    p = torch.from_numpy(p_np).to(dev)
    lib = _lib.load()

    clk = Clocks(torch.cuda.current_device())
    clk.__enter__()
    for _ in range(args.warmup):
        plan.cycle(p, f, op)
    torch.cuda.synchronize()
    kernels_per_cycle = int(lib.mgsr_plan_kernel_nodes(plan.handle, 1 if op == "sr" else 0))

    # ---- device-resident timed region (also records in-graph kernel events) ----
    _lib.check(lib.mgsr_plan_timing_enable(plan.handle, args.steps))
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wait = time.time()
    while not clk.rows and time.time() - t_wait < 5.0:   # sampler running before the timed region
        time.sleep(0.05)
    clk.rows.clear()
    if True:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            plan.cycle(p, f, op)
        e1.record(st)
        torch.cuda.synchronize()
        time.sleep(0.15)   # let the 100 ms sampler see the tail of the region
        clk.__exit__()
        if dist is not None:
            dist.barrier()
    ms_total = e0.elapsed_time(e1)
    import ctypes
    kms = (ctypes.c_double * 3)()
    cnt = ctypes.c_int32()
    _lib.check(lib.mgsr_plan_timing_read(plan.handle, kms, ctypes.byref(cnt)))
    gen_ms, gs_ms, cyc_ms = float(kms[0]), float(kms[1]), float(kms[2])
    stats = plan.stats.cpu().numpy()
    if not np.all(np.isfinite(stats)):
        raise RuntimeError(f"non-finite cycle statistics {stats}")

    # ---- end to end through the C ABI with pinned host buffers ----
    # Every step copies its inputs host -> device and reads its result back; uploads and readbacks run
    # on two copy streams (the PCIe directions overlap) and are double-buffered, so step i + 1's
    # upload and step i's readback overlap the V-cycles (the timed region still contains every copy).
    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(p_np).pin_memory()
        hf = torch.from_numpy(f_np).pin_memory()
        houts = [torch.empty_like(hp).pin_memory() for _ in range(2)]
        hstats = [torch.empty(2, dtype=torch.float64).pin_memory() for _ in range(2)]
        dps = [torch.empty_like(p) for _ in range(2)]
        dfs = [torch.empty_like(f) for _ in range(2)]
        dst = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in range(2)]
        use_sr = 1 if op == "sr" else 0
        for b in range(2):   # capture both buffer variants outside the timed region
            dps[b].copy_(p)
            dfs[b].copy_(f)
            ops.vcycle_(dps[b], dfs[b], plan.handle, use_sr, dst[b])
        torch.cuda.synchronize()
        cs = torch.cuda.Stream()      # uploads
        cs_dn = torch.cuda.Stream()   # readbacks: a separate stream, so the two PCIe directions overlap
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_read = [torch.cuda.Event() for _ in range(2)]
        k2 = max(1, min(args.steps, 5))
        if dist is not None:
            dist.barrier()
        e0.record(st)
        cs.wait_stream(st)
        cs_dn.wait_stream(st)

        def upload(i):
            b = i & 1
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(ev_read[b])   # the cycle that last used buffer b and its readback finished
                dps[b].copy_(hp, non_blocking=True)
                dfs[b].copy_(hf, non_blocking=True)
                ev_in[b].record(cs)

        upload(0)
        for i in range(k2):
            b = i & 1
            st.wait_event(ev_in[b])
            ops.vcycle_(dps[b], dfs[b], plan.handle, use_sr, dst[b])
            ev_done[b].record(st)
            if i + 1 < k2:
                upload(i + 1)
            with torch.cuda.stream(cs_dn):
                cs_dn.wait_event(ev_done[b])
                houts[b].copy_(dps[b], non_blocking=True)
                hstats[b].copy_(dst[b], non_blocking=True)
                ev_read[b].record(cs_dn)
        st.wait_stream(cs)
        st.wait_stream(cs_dn)
        e1.record(st)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        e2e = (k2, e2e_ms, 2 * 8 * n * n, 8 * n * n + 16)

    ms_total = reduce_max(ms_total, dist, dev)
    if e2e is not None:
        e2e = (e2e[0], reduce_max(e2e[1], dist, dev), e2e[2], e2e[3])
    return dict(ms_total=ms_total, gen_ms=gen_ms, gs_ms=gs_ms, cyc_ms=cyc_ms, kernels=kernels_per_cycle,
                e2e=e2e, clocks=clk.summary(), stats=stats.tolist())


# ---------------------------------------------------------------------------
# CPU baseline: the reference compiled from its own sources (oracle/_ref)

SR_SAMPLE_NC = 68        # coarse side of the timed reference sr_prolong sample: (68/2 - 2)^2 = 1024 windows
SPLINE_SAMPLE_N = 2048   # side of the timed reference spline V-cycle


def cpu_reference_sample(n: int, blocks: int, mode: str, sr_levels: int, wkind: str = "trained"):
    """Time the reference on ONE bounded sample and project V-cycles/s at n^2: its
    spline v_cycle at 2048^2 scaled by work (n^2 / 2048^2), plus -- GAN mode -- its full
    sr_prolong (normalise, 1024 windows of 6x6, generator, stitch, denormalise) on a 68^2 coarse grid,
    per-window cost x the cycle's SR windows.  The reference arm and the cpu_baseline leg call this
    same function.  Returns (projected cycles/s, kind, sample description, sample wall seconds)."""
    import numpy as np
    import oracle
    ref = oracle.import_ref()
    kind = "reference" if ref is not None else "port"
    m = min(n, SPLINE_SAMPLE_N)
    f = _rhs(m)
    rng = np.random.default_rng(0)
    c = 1e-4 * _rhs(SR_SAMPLE_NC) + 1e-6 * rng.standard_normal((SR_SAMPLE_NC, SR_SAMPLE_NC))
    c -= c.mean()
    nwin_sample = (SR_SAMPLE_NC // 2 - 2) ** 2
    t_all = time.perf_counter()
    if kind == "reference":
        from mgsr import smoother, solver, srmodel
        from mgsr.grid import Grid, NormBounds
        w = bench_weights(wkind, blocks, srmodel)
        cfg = solver.RunConfig(N_step=1, r_min=8, N_smooth=2)
        t0 = time.perf_counter()
        solver.v_cycle(Grid(np.zeros((m, m))), smoother.PoissonProblem(Grid(f)), cfg, "spline")
        t_spline = time.perf_counter() - t0
        if mode == "gan":
            t0 = time.perf_counter()
            srmodel.sr_prolong(Grid(c), w, NormBounds(), 2)
            t_sr_sample = time.perf_counter() - t0
    else:
        from oracle import mgsr_oracle as orc
        path = weights_path(wkind, blocks)
        w = orc.read_mgsr1(path) if path else orc.random_weights(blocks, 0)
        t0 = time.perf_counter()
        orc.v_cycle(np.zeros((m, m)), f, orc.Config(N_step=1, r_min=8, N_smooth=2), "spline")
        t_spline = time.perf_counter() - t0
        if mode == "gan":
            t0 = time.perf_counter()
            orc.sr_prolong(c, w, orc.Bounds(), 2)
            t_sr_sample = time.perf_counter() - t0
    t_cycle = t_spline * (n * n) / (m * m)
    nw_total = 0
    if mode == "gan":
        for lev in range(1, sr_levels + 1):
            nc = n >> lev
            nw_total += (nc // 2 - 2) ** 2
        t_cycle += t_sr_sample / nwin_sample * nw_total
    sample = (f"reference v_cycle(spline) at {m}^2 scaled by work to {n}^2"
              + (f" + reference sr_prolong (B={blocks}) on a {SR_SAMPLE_NC}^2 coarse grid ({nwin_sample} windows), "
                 f"per-window cost x {nw_total} windows" if mode == "gan" else "") + " (projected)")
    return 1.0 / t_cycle, kind, sample, time.perf_counter() - t_all


def _rhs(m):
    import numpy as np
    x = 2 * np.pi * np.arange(m) / m
    f = np.outer(np.sin(3 * x), np.sin(5 * x)) + 0.3 * np.outer(np.cos(2 * x), np.sin(x))
    return f - f.mean()


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    ncpu = os.cpu_count() or 1
    vals = []
    kind, sample = "reference", ""
    walls = []
    for i in range(args.warmup + args.steps):
        cyc, kind, sample, wall = cpu_reference_sample(args.n, args.blocks, args.mode, args.sr_levels, wkind=args.weights)
        if i >= args.warmup:
            vals.append(cyc)
            walls.append(wall)
    v = sum(vals) / len(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": ncpu, "kind": kind, "sample": sample,
                         "projected": True, "sample_wall_s": sum(walls) / len(walls)},
        "projected": True,
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gupdates_per_s": v * args.n * args.n / 1e9,
    }
    print(json.dumps(line), flush=True)


def workload_config(args):
    wl = (f"periodic {args.n}^2 Poisson V-cycle, N_step=1 ladder {args.n}->8, N_smooth={args.n_smooth}, "
          f"coarse_sweeps=10, " + (f"SR prolongation at the {args.sr_levels} finest levels (B={args.blocks}, "
                                   f"{args.precision} tcgen05 operands / fp32 accumulate), spline below"
                                   if args.mode == "gan" else "spline prolongation at all levels"))
    return {"workload": wl, "grid": args.n, "levels": len(_sides(args.n)), "mode": args.mode,
            "precision": args.precision if args.mode == "gan" else "fp64",
            "generator_blocks": args.blocks, "sr_levels": args.sr_levels if args.mode == "gan" else 0,
            "weights": ("trained" if weights_path(args.weights, args.blocks) else "he_init") if args.mode == "gan"
            else None,
            "parallelism": f"replicas x{int(os.environ.get('WORLD_SIZE', args.gpus))}", "l2": "inputs (134 MB/grid) exceed L2; no flush"}


def _sides(n):
    s = [n]
    while s[-1] > 8:
        s.append(s[-1] // 2)
    return s


def run_plumbing(args, rank: int, world: int, dist):
    """--plumbing-test: the multi-rank bookkeeping of run_mine without a GPU (fake per-rank times)."""
    import torch
    ms = 100.0 + 10.0 * rank
    dev = torch.device("cpu")
    return dict(ms_total=reduce_max(ms, dist, dev), gen_ms=0.0, gs_ms=0.0, cyc_ms=0.0, kernels=0,
                e2e=(1, reduce_max(ms, dist, dev), 0, 0), clocks={"sm_mhz": None, "sm_max_mhz": None,
                                                               "reasons": ["plumbing-test"]}, stats=[])


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "mine":
        self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
        run_reference_arm(args, rank, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        if args.plumbing_test:
            tdist.init_process_group("gloo")
        else:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            tdist.init_process_group("nccl")
        dist = tdist
    res = (run_plumbing if args.plumbing_test else run_mine)(args, rank, world, dist)
    if rank == 0 and args.plumbing_test:
        print(json.dumps({"metric": METRIC, "value": replica_value(args.steps, res["ms_total"], world),
                          "unit": UNIT, "n_gpus": world, "steps": args.steps, "ms_per_step": res["ms_total"] / args.steps,
                          "config": workload_config(args), "plumbing_test": True}), flush=True)
    elif rank == 0:
        peaks, peak_kind = measured_peaks()
        n = args.n
        cyc_s = replica_value(args.steps, res["ms_total"], world)
        if args.mode == "gan":
            flops = pass_flops_fast(n // 2, args.blocks)
            ach = flops / (res["gen_ms"] / 1e3) / 1e12 if res["gen_ms"] > 0 else 0.0
            peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
            roof = {"bound": "tensor", "kernel": "finest-level SR generator (2048->4096, "
                                                 f"{(n // 4 - 2) ** 2} windows)",
                    "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "peak_kind": f"{peak_kind} bf16 sustained (kernel timed inside the cycle)",
                    "algorithmic_flop_per_launch": flops, "launch_ms": res["gen_ms"],
                    "traffic": load_traffic("gan")}
        else:
            b = gs_bytes(n)
            ach = b / (res["gs_ms"] / 1e3) / 1e9 if res["gs_ms"] > 0 else 0.0
            peak = peaks.get("hbm_gbs")
            roof = {"bound": "hbm", "kernel": f"finest-level temporally blocked GS ({args.n_smooth} sweeps "
                                              "+ fused residual injection)",
                    "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "peak_kind": f"{peak_kind} HBM copy", "algorithmic_bytes_per_launch": b,
                    "launch_ms": res["gs_ms"], "traffic": load_traffic("spline")}
        line = {
            "metric": METRIC, "value": cyc_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_total"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": f"f64+{args.precision}" if args.mode == "gan" else "f64",
            "data": "synthetic (seeded GRF k^-5/3 + blobs RHS); generator weights " + (
                "artifacts/trained_b%d.mgsr (reference training pipeline)" % args.blocks
                if weights_path(args.weights, args.blocks) else "seeded He-normal init"),
            "config": workload_config(args), "gupdates_per_s": cyc_s * n * n / 1e9,
            "roofline": roof, "clocks": res["clocks"],
            "gpu_launches": res["kernels"] * args.steps,
            "kernel_ms": {"generator_finest": res["gen_ms"], "gs_finest": res["gs_ms"], "cycle": res["cyc_ms"]},
        }
        if res["e2e"] is not None:
            k2, ms, bi, bo = res["e2e"]
            line["e2e"] = {"value": replica_value(k2, ms, world), "unit": UNIT, "h2d_bytes_per_step": bi,
                           "d2h_bytes_per_step": bo,
                           "path": "pinned host p,f -> torch.ops.mgsr.vcycle_ (C ABI mgsr_plan_vcycle) -> host p; "
                                   "uploads and readbacks on two copy streams, double-buffered across steps"}
        if not args.no_cpu_baseline:
            try:
                cyc, kind, sample, wall = cpu_reference_sample(n, args.blocks, args.mode, args.sr_levels,
                                                               wkind=args.weights)
                line["cpu_baseline"] = {"value": cyc, "unit": UNIT, "cores": os.cpu_count(), "kind": kind,
                                        "sample": sample, "projected": True, "sample_wall_s": wall}
            except Exception as exc:  # the baseline never blocks the GPU line
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                        "sample": f"failed: {exc}"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
