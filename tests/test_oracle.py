"""CPU: pin the oracle restatement against the reference's own outputs.

``tests/golden/golden.npz`` was produced by running the reference itself
(tests/golden/make_golden.py); when ``oracle/_ref`` (the reference compiled
from its own sources) is present the oracle is also compared live.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel, rel_l2


@pytest.mark.parametrize("n", [8, 16, 64])
def test_gs_matches_reference_bitwise(golden, orc, n):
    p = golden[f"gs{n}_p"].copy()
    orc.gs_sweeps(p, golden[f"gs{n}_f"], (2 * np.pi / n) ** 2, 3)
    assert np.array_equal(p, golden[f"gs{n}_out"])          # Cython backend, sequential mean
    q = golden[f"gs{n}_p"].copy()
    orc.gs_sweeps(q, golden[f"gs{n}_f"], (2 * np.pi / n) ** 2, 3, use_c=False)
    assert np.abs(q - golden[f"gs{n}_out_numpy"]).max() < 1e-15


def test_laplacian(golden, orc):
    out = orc.laplacian(golden["lap9_p"], 1.0 / (2 * np.pi / 9) ** 2)
    assert np.abs(out - golden["lap9_out"]).max() < 1e-12


def test_residual_restrict(golden, orc):
    assert rel(orc.residual(golden["res_p"], golden["res_f"]), golden["res_out"]) < 1e-14
    assert np.array_equal(orc.restrict(golden["res_p"], 2), golden["restrict_out"])
    assert np.array_equal(orc.restrict(golden["res_p"], 4, subtract_mean=False), golden["restrict4_raw"])


@pytest.mark.parametrize("s", [2, 4, 8, 16])
def test_spline(golden, orc, s):
    assert rel(orc.spline_prolong(golden[f"spline{s}_c"], s), golden[f"spline{s}_out"]) < 1e-14


def test_keys_known_answers(orc):
    # half-way row (-1/16, 9/16, 9/16, -1/16), coincident rows identity, partition of unity
    # (reference tests/test_transfer.py:57-78)
    w = orc.prolong_taps(2)
    assert np.array_equal(w[0], [0.0, 1.0, 0.0, 0.0])
    assert np.array_equal(w[1], [-0.0625, 0.5625, 0.5625, -0.0625])
    for s in (4, 8, 16):
        assert np.allclose(orc.prolong_taps(s).sum(axis=1), 1.0, atol=1e-15)


def test_restrict_prolong_identity(orc):
    c = np.random.default_rng(3).standard_normal((12, 12))
    for s in (2, 4, 8, 16):
        assert np.abs(orc.restrict(orc.spline_prolong(c, s), s, subtract_mean=False) - c).max() < 1e-13


def test_normalize(golden, orc):
    b = orc.Bounds()
    q = orc.normalize(golden["norm_in"], b)
    assert np.array_equal(q, golden["norm_q"])
    assert np.array_equal(orc.denormalize(q, np.sign(golden["norm_in"]), b), golden["norm_back"])


def test_generator(golden, orc):
    w1 = orc.random_weights(1, 3)
    for key in ("6", "8"):
        y = orc.forward_batch(w1, golden[f"gen_b1_x{key}"][None])[0]
        assert rel(y, golden[f"gen_b1_y{key}"]) < 1e-12
    y = orc.forward_batch(orc.random_weights(8, 0), golden["gen_b8_x6"][None])[0]
    assert rel(y, golden["gen_b8_y6"]) < 1e-12


def test_sr_prolong(golden, orc):
    w2 = orc.random_weights(2, 0)
    b = orc.Bounds()
    assert rel(orc.sr_prolong(golden["sr_c16"], w2, b, 2), golden["sr2_out"]) < 1e-12
    assert rel(orc.sr_prolong(golden["sr_c12"], w2, b, 4), golden["sr4_out"]) < 1e-12
    assert rel(orc.sr_prolong(golden["sr_c16"], orc.nn_weights(), b, 2), golden["srnn2_out"]) < 1e-12


def test_stitch_covers_each_cell_once(orc):
    # reference tests/test_srmodel.py:336-355
    for n in (6, 8, 14, 32):
        cover = np.zeros((n, n), dtype=int)
        for iw, jw, li, hi, lj, hj in orc.stitch_plan(n):
            cover[iw + li:iw + hi, jw + lj:jw + hj] += 1
        assert (cover == 1).all()


def test_v_cycle(golden, orc):
    cfg = orc.Config(N_step=1, r_min=8, N_smooth=2, N_smooth_pre=2)
    out = orc.v_cycle(golden["vc_p"], golden["vc_f"], cfg, "spline")
    assert rel(out, golden["vc_spline_out"]) < 1e-13
    out = orc.v_cycle(golden["vc_sr_p"], golden["vc_sr_f"], cfg, "sr", orc.random_weights(2, 0))
    assert rel(out, golden["vc_sr_out"]) < 1e-11


def test_solve_spline_history(golden, orc):
    p, log = orc.solve(golden["solve64_f"], orc.Config(N_step=1, r_min=8, N_smooth=2))
    ref = golden["solve64_log"]
    assert log.iterations == len(ref)
    got = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    assert rel_l2(got[:3], ref[:3]) < 1e-12
    assert np.abs(got - ref).max() / ref.max() < 1e-6
    assert np.abs(p - golden["solve64_p"]).max() < 1e-14


def test_solve_hybrid_schedule(golden, golden_meta, orc):
    cfg = orc.Config(N_step=1, r_min=8, N_smooth=2, mode="hybrid", N_GAN=1.0, S_thres=2.27e-4)
    p, log = orc.solve(golden["hyb64_f"], cfg, orc.random_weights(1, 0))
    assert [r.operator for r in log.records] == golden_meta["hyb64_ops"]
    assert [r.switch_latched for r in log.records] == golden_meta["hyb64_latched"]
    got = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    assert rel_l2(got, golden["hyb64_log"]) < 1e-8


def test_oracle_against_live_reference(orc):
    """When oracle/_ref (the compiled reference) is importable, compare a full V-cycle live."""
    import oracle
    ref = oracle.import_ref()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from mgsr import smoother, solver
    from mgsr.grid import Grid
    f = orc.sine_modes_rhs(128, 7)
    p0 = orc.initial_iterate(128, orc.Config())
    cfg = orc.Config(N_step=1, r_min=8, N_smooth=3)
    mine = orc.v_cycle(p0, f, cfg, "spline")
    theirs = solver.v_cycle(Grid(p0), smoother.PoissonProblem(Grid(f)),
                            solver.RunConfig(N_step=1, r_min=8, N_smooth=3), "spline").data
    assert rel(mine, theirs) < 1e-13


def test_oracle_generator_matches_reference_trainer_fixtures(orc):
    """The oracle's generator (srmodel.py restatement) replays the reference TRAINER's recorded torch
    forward passes (tests/golden/make_trainer_fixtures.py, PROVENANCE.md:11-19) for both trained weight
    files within the reference's own trainer-parity bar (test_acceptance.py:247-263: 1e-4)."""
    import os
    from conftest import GOLDEN, ROOT
    fx = np.load(os.path.join(GOLDEN, "trainer_fixtures.npz"))
    for b in (4, 8):
        w = orc.read_mgsr1(os.path.join(ROOT, "artifacts", f"trained_b{b}.mgsr"))
        got = orc.forward_batch(w, fx[f"b{b}_inputs"].astype(np.float64))
        assert np.abs(got - fx[f"b{b}_outputs"]).max() < 1e-4, b
