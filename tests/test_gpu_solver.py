"""GPU parity: the graph-launched V-cycle and the solve loop vs golden / oracle.

Bars (north_star / SURVEY §8(d)): one spline V-cycle within 1e-12 relative;
residual-norm histories matching (<= 1e-12 early, <= 1e-6 late -- the spread
the reference shows against itself), the same iteration count to tol, and
identical operator/latch sequences in hybrid mode.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu


def cfg_(**kw):
    from paper_2403_07936_b200.solver import RunConfig
    base = dict(N_step=1, r_min=8, N_smooth=2)
    base.update(kw)
    return RunConfig(**base)


def test_v_cycle_spline_golden(cuda, golden):
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    out = solver.v_cycle(Grid(golden["vc_p"]), PoissonProblem(Grid(golden["vc_f"])), cfg_(N_smooth_pre=2), "spline")
    assert rel(out.data, golden["vc_spline_out"]) < 1e-12


@pytest.mark.parametrize("n,nsm", [(256, 2), (1024, 2), (1024, 5), (2048, 3), (4096, 2)])
def test_v_cycle_spline_large_vs_oracle(cuda, orc, n, nsm):
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    f = orc.sine_modes_rhs(n, 1)
    p0 = orc.initial_iterate(n, orc.Config())
    exp = orc.v_cycle(p0, f, orc.Config(N_step=1, r_min=8, N_smooth=nsm), "spline")
    got = solver.v_cycle(Grid(p0), PoissonProblem(Grid(f)), cfg_(N_smooth=nsm), "spline").data
    assert rel(got, exp) < 1e-12


def test_v_cycle_nstep4_ladder(cuda, orc):
    """Paper-fiducial N_step = 4 ladder (192 -> 12, ratio 16)."""
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    f = orc.sine_modes_rhs(192, 2)
    p0 = orc.initial_iterate(192, orc.Config())
    exp = orc.v_cycle(p0, f, orc.Config(N_step=4, r_min=12, N_smooth=4), "spline")
    got = solver.v_cycle(Grid(p0), PoissonProblem(Grid(f)), cfg_(N_step=4, r_min=12, N_smooth=4), "spline").data
    assert rel(got, exp) < 1e-12


def test_solve_spline_history_golden(cuda, golden):
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    p, log = solver.solve(PoissonProblem(Grid(golden["solve64_f"])), cfg_())
    ref = golden["solve64_log"]
    assert log.iterations == len(ref)
    got = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    assert rel_l2(got[:2], ref[:2]) < 1e-12
    assert (np.abs(got - ref) / ref).max() < 1e-6
    assert np.abs(p.data - golden["solve64_p"]).max() < 1e-13


def test_solve_spline_1024_matches_oracle(cuda, orc):
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    f = orc.sine_modes_rhs(1024, 0)
    p_ref, log_ref = orc.solve(f, orc.Config(N_step=1, r_min=8, N_smooth=2))
    p, log = solver.solve(PoissonProblem(Grid(f)), cfg_())
    assert log.iterations == log_ref.iterations
    a = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    b = np.array([[r.diff_norm, r.residual_norm] for r in log_ref.records])
    assert (np.abs(a - b) / b).max() < 1e-6
    assert rel(p.data, p_ref) < 1e-9


def test_solve_matches_discrete_oracle(cuda, orc):
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    f = orc.sine_modes_rhs(256, 3)
    p, log = solver.solve(PoissonProblem(Grid(f)), cfg_())
    assert log.converged(1e-10)
    assert np.sqrt(np.mean((p.data - orc.spectral_solution(f)) ** 2)) < 1e-8


def test_solve_hybrid_schedule_golden(cuda, golden, golden_meta):
    """Latched hybrid: identical operator and latch sequences, same iteration count."""
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    cfg = cfg_(mode="hybrid", N_GAN=1.0, S_thres=2.27e-4)
    p, log = solver.solve(PoissonProblem(Grid(golden["hyb64_f"])), cfg, srmodel.random_weights(1, 0), precision="fp32")
    assert [r.operator for r in log.records] == golden_meta["hyb64_ops"]
    assert [r.switch_latched for r in log.records] == golden_meta["hyb64_latched"]
    got = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    assert rel_l2(got, golden["hyb64_log"]) < 1e-4


def test_v_cycle_sr_golden(cuda, golden):
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    out = solver.v_cycle(Grid(golden["vc_sr_p"]), PoissonProblem(Grid(golden["vc_sr_f"])), cfg_(N_smooth_pre=2),
                         "sr", srmodel.random_weights(2, 0), precision="fp32")
    assert rel_l2(out.data, golden["vc_sr_out"]) < 1e-4


def test_sr_requires_weights(cuda):
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    f = np.zeros((32, 32))
    with pytest.raises(ValueError, match="weights"):
        solver.v_cycle(Grid(f), PoissonProblem(Grid(f)), cfg_(), "sr")


@pytest.mark.parametrize("sr_levels,bar", [(1, 1e-2)])
def test_v_cycle_sr_fp16_vs_oracle(cuda, orc, sr_levels, bar):
    """SR V-cycle (trained weights, SR at the finest prolongation) through the tensor-core path vs
    the fp64 oracle's whole cycle.  With SR at several levels every prolongation is held to the
    field bar separately (test_vcycle_sr_levels_each_prolongation_vs_oracle): the cycle output
    compounds their errors."""
    import os
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    from conftest import ROOT
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b4.mgsr"))
    f = orc.scale_to_p_rms(orc.sine_modes_rhs(128, 0), 1e-4)
    p0 = orc.initial_iterate(128, orc.Config()) * 0.1
    ow = orc.Weights(dict(w.tensors), w.num_residual_blocks, w.tanh_scale)
    nlev = len(orc.level_sides(128, 1, 8))
    lops = None if sr_levels is None else [None] + ["sr" if l <= sr_levels else "spline" for l in range(1, nlev)]
    exp = orc.v_cycle(p0, f, orc.Config(N_step=1, r_min=8, N_smooth=2), "sr", ow, level_ops=lops)
    got = solver.v_cycle(Grid(p0), PoissonProblem(Grid(f)), cfg_(), "sr", w, precision="fp16",
                         sr_levels=sr_levels).data
    assert rel_l2(got, exp) < bar


def test_solve_hybrid_fp16_matches_fp32_schedule(cuda, orc):
    """Latched hybrid solve at 256^2 with the tensor-core generator: same operator/latch
    sequence and iteration count as the fp32 path, converged to tol."""
    import os
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    from conftest import ROOT
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    f = orc.scale_to_p_rms(orc.sine_modes_rhs(256, 0), 1e-4)
    cfg = cfg_(mode="hybrid", N_GAN=1.0, S_thres=5e-4)
    _, l32 = solver.solve(PoissonProblem(Grid(f)), cfg, w, precision="fp32")
    _, l16 = solver.solve(PoissonProblem(Grid(f)), cfg, w, precision="fp16")
    assert [r.operator for r in l16.records] == [r.operator for r in l32.records]
    assert l16.iterations == l32.iterations and l16.converged(1e-10)


@pytest.mark.parametrize("mode,n", [("spline", 64), ("spline", 256), ("hybrid", 256)])
def test_resident_solve_matches_host_loop(cuda, orc, mode, n):
    """The single-launch device loop (WHILE conditional graph node, mgsr_plan_solve) runs the
    same cycles as the per-cycle host loop: identical histories, operators, latches and count."""
    import os
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    from conftest import ROOT
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr")) if mode == "hybrid" else None
    f = orc.scale_to_p_rms(orc.sine_modes_rhs(n, 0), 1e-4)
    cfg = cfg_(mode=mode, N_GAN=1.0, S_thres=5e-4)
    p_a, la = solver.solve(PoissonProblem(Grid(f)), cfg, w, resident=True, precision="fp32")
    p_b, lb = solver.solve(PoissonProblem(Grid(f)), cfg, w, resident=False, precision="fp32")
    assert la.iterations == lb.iterations
    assert [r.operator for r in la.records] == [r.operator for r in lb.records]
    assert [r.switch_latched for r in la.records] == [r.switch_latched for r in lb.records]
    a = np.array([[r.diff_norm, r.residual_norm] for r in la.records])
    b = np.array([[r.diff_norm, r.residual_norm] for r in lb.records])
    assert np.array_equal(a, b)
    assert np.array_equal(p_a.data, p_b.data)


@pytest.mark.parametrize("batched,precision,n,sr_levels", [(False, "fp32", 128, None), (True, "fp32", 128, None),
                                                         (True, "fp16", 128, None), (True, "fp16", 256, 3)])
def test_solve_batch_matches_single_solves(cuda, orc, batched, precision, n, sr_levels):
    """Multi-RHS solves give exactly the single-solve results: one plan + stream each (batched=False),
    or all solve loops in lockstep in one graph launch with one generator launch per SR level across
    the RHS that prolong by SR in that iteration (batched=True; fp16 = the batched tensor-core launch).
    The right-hand sides differ in scale and spectrum, so their latches and stopping iterations differ."""
    import os
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    from conftest import ROOT
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    fs = [orc.scale_to_p_rms(orc.sine_modes_rhs(n, 0), 1e-4), orc.scale_to_p_rms(orc.grf_blobs_rhs(n, seed=1, kmax=n / 8), 3e-4),
          orc.scale_to_p_rms(orc.sine_modes_rhs(n, 2), 3e-2)]
    cfg = cfg_(mode="hybrid", N_GAN=1.0, S_thres=5e-4)
    batch = solver.solve_batch([PoissonProblem(Grid(f)) for f in fs], cfg, w, precision=precision, sr_levels=sr_levels,
                               batched=batched)
    iters = []
    for f, (pb, lb) in zip(fs, batch):
        ps, ls = solver.solve(PoissonProblem(Grid(f)), cfg, w, precision=precision, sr_levels=sr_levels)
        assert lb.iterations == ls.iterations and lb.converged(1e-10)
        assert [r.operator for r in lb.records] == [r.operator for r in ls.records]
        assert [r.switch_latched for r in lb.records] == [r.switch_latched for r in ls.records]
        assert [r.diff_norm for r in lb.records] == [r.diff_norm for r in ls.records]
        assert np.array_equal(pb.data, ps.data)
        iters.append(ls.iterations)
    print(f"\nsolve_batch batched={batched} {precision} n={n}: iterations {iters}")


@pytest.mark.parametrize("n,seed,pmax", [(16, 0, 1e-3), (64, 3, 1e-3), (256, 0, 2.5e-2), (2048, 11, 1e-3)])
def test_device_initial_iterate_bitwise(cuda, n, seed, pmax):
    """mgsr_initial_iterate == numpy default_rng(seed).uniform(-p_max, p_max) - mean, bit for bit."""
    from paper_2403_07936_b200 import solver
    cfg = solver.RunConfig(seed=seed, p_max=pmax)
    exp = solver.initial_iterate(n, cfg)
    got = solver.initial_iterate_device(n, cfg).cpu().numpy()
    assert np.array_equal(got, exp)


def test_default_config_ladder_3072_vs_oracle(cuda, orc):
    """The reference's default RunConfig (N_step=4, r_min=12, N_smooth=20) at 3072^2: ladder
    [3072, 192, 12] with ratio-16 spline prolongations and 20-sweep smoothing (chunked K=4 register
    tiles).  Two V-cycles against the CPU oracle."""
    from paper_2403_07936_b200 import datagen, solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    n = 3072
    f = datagen.grf_blobs_rhs(n, seed=0, kmax=n / 8)
    ocfg = orc.Config(N_step=4, r_min=12, N_smooth=20)
    p = orc.initial_iterate(n, orc.Config())
    exp = orc.v_cycle(orc.v_cycle(p, f, ocfg, "spline"), f, ocfg, "spline")
    cfg = cfg_(N_step=4, r_min=12, N_smooth=20)
    got = solver.v_cycle(solver.v_cycle(Grid(p), PoissonProblem(Grid(f)), cfg, "spline"),
                         PoissonProblem(Grid(f)), cfg, "spline").data
    assert rel(got, exp) < 1e-12


def test_solve_non_power_of_two_side_uses_host_start(cuda, orc):
    """Sides whose n*n is not a power of two keep the host draw of the seeded start (the device
    draw needs numpy's perfect pairwise tree); the history still matches the oracle."""
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    assert not solver._device_start_ok(96)
    f = orc.sine_modes_rhs(96, 4)
    p_ref, log_ref = orc.solve(f, orc.Config(N_step=1, r_min=12, N_smooth=2))
    p, log = solver.solve(PoissonProblem(Grid(f)), cfg_(r_min=12))
    assert log.iterations == log_ref.iterations
    a = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    b = np.array([[r.diff_norm, r.residual_norm] for r in log_ref.records])
    assert (np.abs(a - b) / b).max() < 1e-6


def _sr_dumps(plan, levels, torch):
    """Attach the plan's per-level SR dump (mgsr_debug_plan_sr_dump): {level: (c, sr_raw)} device buffers."""
    import ctypes
    from paper_2403_07936_b200 import _lib
    lib = _lib.load()
    lib.mgsr_debug_plan_sr_dump.restype = ctypes.c_int
    lib.mgsr_debug_plan_sr_dump.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
    out = {}
    for l in levels:
        nc, nf = plan.sides[l], plan.sides[l - 1]
        c = torch.zeros((nc, nc), dtype=torch.float64, device="cuda")
        s = torch.zeros((nf, nf), dtype=torch.float64, device="cuda")
        _lib.check(lib.mgsr_debug_plan_sr_dump(plan.handle, l, c.data_ptr(), s.data_ptr()))
        out[l] = (c, s)
    return out


@pytest.mark.parametrize("weights,n,sr_levels", [("trained_b8", 256, 3), ("trained_b4", 256, 3),
                                                ("trained_b4", 128, None)])
def test_vcycle_sr_levels_each_prolongation_vs_oracle(cuda, orc, weights, n, sr_levels):
    """The bench's cycle shape (SR at the 3 finest prolongations, spline below, fp16 tensor cores) at
    256^2, and SR at every level (128 -> 8, the reference's own "sr" cycle): inside the captured graph
    each SR prolongation's input correction and output are dumped, and EACH level's output is checked
    against the fp64 oracle's sr_prolong of that same input at the north-star 1e-2 relL2 bar."""
    import os
    from paper_2403_07936_b200 import solver, srmodel
    from conftest import ROOT
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", f"{weights}.mgsr"))
    ow = orc.Weights(dict(w.tensors), w.num_residual_blocks, w.tanh_scale)
    f = orc.scale_to_p_rms(orc.grf_blobs_rhs(n, seed=2, kmax=n / 4), 1e-4)
    p0 = orc.initial_iterate(n, orc.Config()) * 0.1
    plan = solver.VCyclePlan(n, cfg_(), w, precision="fp16", sr_levels=sr_levels)
    nsr = len(plan.sides) - 1 if sr_levels is None else sr_levels
    dumps = _sr_dumps(plan, range(1, nsr + 1), cuda)
    p, fd = plan.load(p0, f)
    plan.cycle(p, fd, "sr")
    cuda.cuda.synchronize()
    for l, (c, s) in dumps.items():
        c = c.cpu().numpy()
        got = s.cpu().numpy()
        got = got - got.mean()
        exp = orc.sr_prolong(c, ow, orc.Bounds(), 2)
        assert np.abs(c).max() > 0, l
        assert rel_l2(got, exp) < 1e-2, (l, rel_l2(got, exp))


def test_bench_cycle_4096_each_sr_level_vs_oracle_sampled(cuda, orc):
    """BASELINE config 4 exactly as bench.py runs it (4096^2, 10 levels, SR at the 3 finest
    prolongations, trained B=8, fp16 tensor cores, bench RHS and start): each of the three SR
    prolongations of the captured cycle (n_c = 2048, 1024, 512) is dumped and checked against the
    fp64 oracle on 96 seeded sampled windows per level (corners and edges included) at 1e-2."""
    import os
    import sys
    from paper_2403_07936_b200 import solver, srmodel
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    import bench
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    ow = orc.Weights(dict(w.tensors), w.num_residual_blocks, w.tanh_scale)
    n = 4096
    f, p0 = bench.make_inputs(n, bench.replica_seed(0), "gan")
    plan = solver.VCyclePlan(n, cfg_(coarse_sweeps=10), w, precision="fp16", sr_levels=3)
    dumps = _sr_dumps(plan, (1, 2, 3), cuda)
    p, fd = plan.load(p0, f)
    plan.cycle(p, fd, "sr")
    cuda.cuda.synchronize()
    b = orc.Bounds()
    for l, (c, s) in dumps.items():
        c = c.cpu().numpy()
        got = s.cpu().numpy()
        nc = c.shape[0]
        npos = nc // 2 - 2
        rng = np.random.default_rng(100 + l)
        picks = {(0, 0), (0, npos - 1), (npos - 1, 0), (npos - 1, npos - 1), (0, npos // 3), (npos // 2, 0)}
        while len(picks) < 96:
            picks.add(tuple(int(x) for x in rng.integers(1, npos - 1, size=2)))
        sample = [i * npos + j for i, j in sorted(picks)]
        qf = orc.sr_pass(orc.normalize(c, b), ow, 1, sample=sample)
        m = ~np.isnan(qf)
        exp = orc.denormalize(qf[m], np.sign(qf[m]), b)
        assert m.sum() >= 96 * 16
        assert rel_l2(got[m], exp) < 1e-2, (l, rel_l2(got[m], exp))


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_config3_hybrid_1024_matches_reference_fixture(cuda, orc, golden_dir, precision):
    """BASELINE config 3 (1024^2, GRF + blobs, latched hybrid, trained B=8) against the REFERENCE's
    own solve (tests/golden/make_config3_golden.py -> config3_hybrid.npz): the same iteration count,
    operator and latch sequences, the converged field, and the residual / diff histories."""
    import json
    import os
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    from conftest import ROOT
    fx = np.load(os.path.join(golden_dir, "config3_hybrid.npz"))
    meta = json.load(open(os.path.join(golden_dir, "config3_hybrid_meta.json")))
    f = orc.scale_to_p_rms(orc.grf_blobs_rhs(1024, seed=0, kmax=256.0), 1e-4)
    assert np.allclose([f.sum(), np.abs(f).sum(), (f * f).sum()], fx["f_checksum"], rtol=1e-12, atol=1e-12)
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    cfg = cfg_(mode="hybrid", N_GAN=1.0, S_thres=5e-4)
    p, log = solver.solve(PoissonProblem(Grid(f)), cfg, w, precision=precision)
    assert log.iterations == meta["iterations"]
    assert [r.operator for r in log.records] == meta["operators"]
    assert [r.switch_latched for r in log.records] == meta["latched"]
    hist = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    ref = fx["log"]
    relh = np.abs(hist - ref) / ref
    print(f"\nconfig3 {precision}: history rel diff per iteration {relh.max(axis=1)}")
    bar = 1e-4 if precision == "fp32" else 5e-3     # measured 1.8e-5 / 1.7e-3 (generator operand precision)
    assert relh.max() < bar
    sub = p.data[::16, ::16]
    assert rel_l2(sub, fx["p_sub"]) < 1e-8


@pytest.mark.parametrize("precision,bar", [("fp32", 1e-4), ("fp16", 1e-2)])
def test_default_config_sr_vcycle_vs_oracle(cuda, orc, precision, bar):
    """The reference's default RunConfig (N_step=4, r_min=12, N_smooth=20) with SR prolongation at
    192^2: ladder [192, 12], one ratio-16 SR prolongation (two ratio-4 passes) of the 12^2 correction,
    on the tensor cores for fp16.  One V-cycle against the CPU oracle (trained B=8 weights)."""
    import os
    from paper_2403_07936_b200 import datagen, solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    from conftest import ROOT
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    n = 192
    f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(n, seed=2, kmax=24.0), 1e-4)
    p = orc.initial_iterate(n, orc.Config()) * 0.1
    ocfg = orc.Config(N_step=4, r_min=12, N_smooth=20)
    ow = orc.Weights({k: v for k, v in w.tensors.items()}, w.num_residual_blocks, w.tanh_scale)
    exp = orc.v_cycle(p, f, ocfg, "sr", orc.quantize_f32(ow))
    cfg = cfg_(N_step=4, r_min=12, N_smooth=20)
    got = solver.v_cycle(Grid(p), PoissonProblem(Grid(f)), cfg, "sr", w, precision=precision).data
    err = rel_l2(got - got.mean(), exp - exp.mean())
    print(f"default-config SR V-cycle {precision}: relL2 {err:.3e}")
    assert err < bar, err


def test_solve_batch_default_config_ratio16_matches_single(cuda, orc):
    """Batched solves with the reference's default ladder (N_step=4, r_min=12: [192, 12], one ratio-16 SR
    prolongation = two ratio-4 tensor-core passes, run per grid inside the batched graph) equal the single
    solves bitwise."""
    import os
    from paper_2403_07936_b200 import solver, srmodel
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    from conftest import ROOT
    w = srmodel.load_weights(os.path.join(ROOT, "artifacts", "trained_b8.mgsr"))
    n = 192
    fs = [orc.scale_to_p_rms(orc.grf_blobs_rhs(n, seed=s, kmax=24.0), 1e-4) for s in range(2)]
    cfg = cfg_(N_step=4, r_min=12, N_smooth=20, mode="hybrid", N_GAN=1.0, S_thres=5e-4, N_iter=40)
    batch = solver.solve_batch([PoissonProblem(Grid(f)) for f in fs], cfg, w, precision="fp16", batched=True)
    for f, (pb, lb) in zip(fs, batch):
        ps, ls = solver.solve(PoissonProblem(Grid(f)), cfg, w, precision="fp16")
        assert lb.iterations == ls.iterations
        assert [r.operator for r in lb.records] == [r.operator for r in ls.records]
        assert [r.diff_norm for r in lb.records] == [r.diff_norm for r in ls.records]
        assert np.array_equal(pb.data, ps.data)
