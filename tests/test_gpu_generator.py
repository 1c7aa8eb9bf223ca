"""GPU parity: generator inference and windowed SR prolongation.

Bar (north_star): GAN-prolonged fields within 1e-2 relative L2 of the
reference's generator; the fp32 CUDA-core path is held much tighter.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel, rel_l2

pytestmark = pytest.mark.gpu


def test_generator_forward_golden(cuda, golden):
    from paper_2403_07936_b200 import srmodel
    w1 = srmodel.random_weights(1, 3)
    for key in ("6", "8"):
        y = srmodel.generator_forward(w1, golden[f"gen_b1_x{key}"])
        assert rel(y, golden[f"gen_b1_y{key}"]) < 1e-5
    y = srmodel.generator_forward(srmodel.random_weights(8, 0), golden["gen_b8_x6"])
    assert rel(y, golden["gen_b8_y6"]) < 1e-3   # saturated tanh, fp32 vs fp64


def test_generator_nn_weights_exact(cuda):
    """Crafted weights = exact x2 nearest-neighbour upsampler (srmodel.py:361-387)."""
    from paper_2403_07936_b200 import srmodel
    x = np.random.default_rng(0).uniform(-1, 1, (3, 6, 6))
    y = srmodel.generator_forward(srmodel.make_nearest_neighbor_weights(), x)
    exp = np.repeat(np.repeat(x, 2, axis=1), 2, axis=2)
    assert np.abs(y - exp).max() < 1e-6


def test_sr_prolong_fp32_golden(cuda, golden):
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w2 = srmodel.random_weights(2, 0)
    out = srmodel.sr_prolong(Grid(golden["sr_c16"]), w2, NormBounds(), 2, precision="fp32")
    assert rel_l2(out.data, golden["sr2_out"]) < 1e-4
    out = srmodel.sr_prolong(Grid(golden["sr_c12"]), w2, NormBounds(), 4, precision="fp32")
    assert rel_l2(out.data, golden["sr4_out"]) < 1e-4
    out = srmodel.sr_prolong(Grid(golden["sr_c16"]), srmodel.make_nearest_neighbor_weights(), NormBounds(), 2, precision="fp32")
    assert rel(out.data, golden["srnn2_out"]) < 1e-5


@pytest.mark.parametrize("s,nc", [(2, 46), (4, 22)])
def test_fp32_row_tiled_kernels_bitwise_equal_one_pixel_kernels(cuda, monkeypatch, s, nc):
    """The row-tiled fp32 kernels (k_conv_rows / k_conv_tail_rows, sides 6 and 12) keep the accumulation
    order of the one-pixel kernels they replaced: the whole pass is bitwise identical (partial CTAs included:
    441 and 81 windows are not multiples of the windows per CTA)."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    rng = np.random.default_rng(7)
    c = (10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)
    c -= c.mean()
    w = srmodel.random_weights(2, 5)
    new = srmodel.sr_prolong(Grid(c), w, NormBounds(), s, precision="fp32").data
    monkeypatch.setenv("MGSR_F32_LEGACY", "1")
    old = srmodel.sr_prolong(Grid(c), w, NormBounds(), s, precision="fp32").data
    assert np.array_equal(new, old)


def test_fp32_row_tiled_kernels_deterministic(cuda):
    """Repeated fp32 passes are bitwise identical (staging, stage barriers and the shared-memory epilogue of the
    row-tiled kernels carry no race): ratio 4 at n_c = 100 (2304 windows, 12x12 second application)."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    rng = np.random.default_rng(11)
    c = (10.0 ** rng.uniform(-7, -3.5, (100, 100))) * np.where(rng.random((100, 100)) < 0.5, -1, 1)
    c -= c.mean()
    w = srmodel.random_weights(8, 0)
    ref = srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp32").data
    for _ in range(3):
        assert np.array_equal(srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp32").data, ref)


@pytest.mark.parametrize("s", [8, 16])
def test_sr_prolong_two_pass_ratios(cuda, orc, s):
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    from conftest import ROOT  # noqa: F401
    c = orc.scale_to_p_rms(orc.sine_modes_rhs(12, 4), 1e-4)[:12, :12]
    c = c - c.mean()
    w = srmodel.random_weights(1, 2)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), s, precision="fp32").data
    exp = orc.sr_prolong(c, orc.random_weights(1, 2), orc.Bounds(), s)
    assert rel_l2(got, exp) < 1e-3


def test_sr_prolong_fp32_vs_oracle_256(cuda, orc):
    """Full field at n_c = 128 (3844 windows), trained-like in-band input."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    c = orc.scale_to_p_rms(orc.sine_modes_rhs(128, 5), 1e-4)
    w = srmodel.random_weights(8, 0)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp32").data
    exp = orc.sr_prolong(c, orc.quantize_f32(orc.random_weights(8, 0)), orc.Bounds(), 2)
    assert rel_l2(got, exp) < 1e-3


def test_sr_ratio_errors(cuda):
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = srmodel.random_weights(1, 0)
    with pytest.raises(ValueError, match="unsupported SR ratio"):
        srmodel.sr_prolong(Grid(np.ones((8, 8))), w, NormBounds(), 3)
    with pytest.raises(ValueError, match=">= 6"):
        srmodel.sr_prolong(Grid(np.ones((4, 4))), w, NormBounds(), 2)


# ---------------------------------------------------------------------------
# tensor-core (tcgen05) megakernel: fp16 / bf16 operands, fp32 accumulation

def _fields(nc):
    from paper_2403_07936_b200 import datagen
    rng = np.random.default_rng(0)
    noise = (10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)
    f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(nc, seed=3, kmax=nc / 8), 1e-5)
    return {"noise": noise, "smooth": datagen.spectral_solution(f)}


def _trained(blocks):
    import os
    from paper_2403_07936_b200 import srmodel
    from conftest import ROOT
    return srmodel.load_weights(os.path.join(ROOT, "artifacts", f"trained_b{blocks}.mgsr"))


def _oracle_weights(orc, w):
    return orc.Weights({k: v for k, v in w.tensors.items()}, w.num_residual_blocks, w.tanh_scale)


@pytest.mark.parametrize("blocks", [4, 8])
def test_tc_fp16_field_parity_trained(cuda, orc, blocks):
    """North-star bar: GAN-prolonged field within 1e-2 relL2 of the reference generator (the fp64
    CPU oracle on the MGSR1 weights), full field at n_c = 64, noise and smooth inputs."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(blocks)
    ow = _oracle_weights(orc, w)
    for name, c in _fields(64).items():
        exp = orc.sr_prolong(c, ow, orc.Bounds(), 2)
        got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
        assert rel_l2(got, exp) < 1e-2, name


def test_tc_fp16_field_parity_he_init_smooth(cuda, orc):
    """Seeded He-init B=8 (BASELINE's fallback weights) on a smooth correction field, vs the oracle."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = srmodel.random_weights(8, 0)
    c = _fields(64)["smooth"]
    exp = orc.sr_prolong(c, _oracle_weights(orc, w), orc.Bounds(), 2)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
    assert rel_l2(got, exp) < 1e-2


def test_tc_bf16_vs_fp16_error_ordering(cuda):
    """bf16 (7-bit mantissa) is measurably worse than fp16 (10-bit) at the same speed; record both."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(8)
    c = _fields(128)["noise"]
    ref = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp32").data
    e16 = rel_l2(srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data, ref)
    eb = rel_l2(srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="bf16").data, ref)
    assert e16 < eb < 2e-2


def test_tc_vs_oracle_full_field(cuda, orc):
    """Full field against the fp64 CPU oracle on MGSR1-quantised trained weights (n_c = 64)."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(4)
    c = _fields(64)["smooth"]
    ow = orc.Weights({k: v for k, v in w.tensors.items()}, w.num_residual_blocks, w.tanh_scale)
    exp = orc.sr_prolong(c, ow, orc.Bounds(), 2)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
    assert rel_l2(got, exp) < 1e-2


@pytest.mark.parametrize("nc", [6, 8, 10, 16])
def test_tc_edge_windows_and_tiny_grids(cuda, orc, nc):
    """Grids whose windows are all (or mostly) edge windows exercise the exact fallback tail;
    every fine cell is written (stitch coverage) and matches the fp64 oracle."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(4)
    c = _fields(nc)["noise"]
    exp = orc.sr_prolong(c, _oracle_weights(orc, w), orc.Bounds(), 2)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
    assert np.all(np.isfinite(got))
    assert rel_l2(got, exp) < 1e-2


def test_tc_nn_weights_upsampler(cuda, orc):
    """Crafted nearest-neighbour weights: the generator copies q; the field returns to the
    input values at the coincident fine cells up to operand rounding (fp16 head), vs the oracle."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    c = _fields(32)["noise"]
    w = srmodel.make_nearest_neighbor_weights()
    exp = orc.sr_prolong(c, _oracle_weights(orc, w), orc.Bounds(), 2)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
    assert rel_l2(got, exp) < 1e-2


def test_tc_deterministic(cuda):
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(8)
    c = _fields(256)["smooth"]
    a = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
    b = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
    assert np.array_equal(a, b)


@pytest.mark.parametrize("weights", ["trained_b8", "trained_b4", "he_b1"])
@pytest.mark.parametrize("nc", [12, 40])
def test_tc_ratio4_pass_vs_oracle(cuda, orc, weights, nc):
    """A ratio-4 SR pass on the tensor cores (first application on 6x6 windows with the full 12x12x3
    output, second on 12x12 windows of 3 distinct channels, kept 8x8 fine pixels; srmodel.py:443-487)
    against the fp64 CPU oracle, full field, at the north-star 1e-2 relL2 bar.  nc = 12 is the paper
    ladder's 12 -> 48 first pass (16 windows, 12 of them edge windows).  Measured 1.7e-3 .. 4.3e-3
    (tests/precision_r4.py; the oracle with fp16-rounded conv operands lands within 10% of the same)."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = {"trained_b8": lambda: _trained(8), "trained_b4": lambda: _trained(4),
         "he_b1": lambda: srmodel.random_weights(1, 3)}[weights]()
    c = _fields(max(nc, 16))["smooth"][:nc, :nc]
    c = c - c.mean()
    exp = orc.sr_prolong(c, orc.quantize_f32(_oracle_weights(orc, w)), orc.Bounds(), 4)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp16").data
    assert got.shape == exp.shape
    assert rel_l2(got, exp) < 1e-2, rel_l2(got, exp)


@pytest.mark.parametrize("s,nc", [(8, 16), (16, 12)])
def test_tc_two_pass_ratios_per_pass_vs_oracle(cuda, orc, s, nc):
    """Ratios 8 (x4 then x2) and 16 (x4 then x4) on the tensor cores: the composed prolongation equals
    the two passes run one after the other through the public API (bitwise), and each pass matches the
    fp64 oracle's pass on the same input at the 1e-2 bar.  The end-to-end fp16 error of the composition
    is the reference algorithm's own sensitivity to operand rounding (the second pass re-normalises the
    first pass's output logarithmically): the oracle run with fp16-rounded conv operands shows 7e-3 ..
    6e-2 on these fields (tests/precision_r4.py), so the composition is
    pinned per pass, not end to end."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(8)
    ow = orc.quantize_f32(_oracle_weights(orc, w))
    c = _fields(16)["smooth"][:nc, :nc]
    c = c - c.mean()
    full = srmodel.sr_prolong(Grid(c), w, NormBounds(), s, precision="fp16").data
    mid = srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp16").data
    last = srmodel.sr_prolong(Grid(mid), w, NormBounds(), s // 4, precision="fp16").data
    assert np.allclose(full, last, rtol=1e-12, atol=0.0), float(np.abs(full - last).max())
    e1 = rel_l2(mid, orc.sr_prolong(c, ow, orc.Bounds(), 4))
    e2 = rel_l2(last, orc.sr_prolong(mid, ow, orc.Bounds(), s // 4))
    assert e1 < 1e-2 and e2 < 1e-2, (e1, e2)


def test_tc_ratio4_pass_vs_fp32_generator_larger(cuda):
    """A ratio-4 pass at n_c = 128 (3844 windows: many groups per CTA pair, interior and edge windows):
    fp16 tensor cores against the fp32 CUDA-core generator (itself pinned to the oracle by
    test_sr_prolong_fp32_golden) at the 1e-2 bar, and bitwise repeatable."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(8)
    c = _fields(128)["smooth"]
    ref = srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp32").data
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp16").data
    assert rel_l2(got, ref) < 1e-2, rel_l2(got, ref)
    again = srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp16").data
    assert np.array_equal(got, again)


@pytest.mark.parametrize("weights", ["trained", "he_init"])
def test_tc_bench_size_pass_vs_oracle_sampled_windows(cuda, orc, weights):
    """The bench's finest pass at full size (n_c = 2048, 1,044,484 windows): the fp16 tensor-core
    field (before the per-pass mean subtraction, via mgsr_debug_tc_pass) against the fp64 CPU
    oracle on 256 seeded sampled windows -- corners, edge windows and interior windows -- within the
    north-star 1e-2 relL2 bar.  Weights: trained B=8, and the seeded He-init B=8 the bench uses."""
    import ctypes
    from paper_2403_07936_b200 import _lib, datagen, srmodel
    nc = 2048
    w = _trained(8) if weights == "trained" else srmodel.random_weights(8, 0)
    f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(nc, seed=5, kmax=256.0), 1e-4)
    c = datagen.spectral_solution(f)
    lib = _lib.load()
    lib.mgsr_debug_tc_pass.restype = ctypes.c_int
    lib.mgsr_debug_tc_pass.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_void_p]
    dc = cuda.from_numpy(c).cuda()
    fine = cuda.empty((2 * nc, 2 * nc), dtype=cuda.float64, device="cuda")
    _lib.check(lib.mgsr_debug_tc_pass(w.device_handle(), dc.data_ptr(), nc, 1e-10, 1e-3, fine.data_ptr(), None, -1,
                                      1, cuda.cuda.current_stream().cuda_stream))
    got = fine.cpu().numpy()
    npos = nc // 2 - 2
    rng = np.random.default_rng(11)
    picks = {(0, 0), (0, npos - 1), (npos - 1, 0), (npos - 1, npos - 1), (0, 517), (npos - 1, 3), (700, 0)}
    while len(picks) < 256:
        picks.add(tuple(int(x) for x in rng.integers(1, npos - 1, size=2)))
    sample = [i * npos + j for i, j in sorted(picks)]
    ow = orc.Weights({k: v for k, v in w.tensors.items()}, w.num_residual_blocks, w.tanh_scale)
    b = orc.Bounds()
    qf = orc.sr_pass(orc.normalize(c, b), ow, 1, sample=sample)
    m = ~np.isnan(qf)
    exp = orc.denormalize(qf[m], np.sign(qf[m]), b)
    assert m.sum() >= 256 * 16
    # north-star bar for both weight sets (measured 7.1e-3 He-init; the
    # He-init error is a handful of sign flips of saturated tanh outputs, see the full-field test below)
    assert rel_l2(got[m], exp) < 1e-2


@pytest.mark.parametrize("weights", ["trained", "he_init"])
def test_tc_bench_size_full_field_vs_fp32_generator(cuda, weights):
    """The whole bench-size field (n_c = 2048, 1,044,484 windows, 16.8M fine cells): fp16 tensor cores
    vs the fp32 CUDA-core generator (itself pinned to the fp64 oracle: test_sr_prolong_fp32_golden,
    test_sr_prolong_fp32_vs_oracle_256) at the north-star 1e-2 bar.  Measured 2.6e-3 (trained) and
    1.7e-3 (He-init)."""
    from paper_2403_07936_b200 import datagen, srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    nc = 2048
    w = _trained(8) if weights == "trained" else srmodel.random_weights(8, 0)
    f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(nc, seed=5, kmax=256.0), 1e-4)
    c = datagen.spectral_solution(f)
    ref = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp32").data
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp16").data
    assert rel_l2(got, ref) < 1e-2


def test_tc_generator_depths(cuda, orc):
    """Residual-block counts other than 4/8: B=1 runs on the tensor cores within the bar; B=16 (the
    deepest whose constants fit the kernel's shared memory) runs; B=17 is refused loudly, never run
    on a fallback."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    c = _fields(32)["smooth"]
    w1 = srmodel.random_weights(1, 3)
    exp = orc.sr_prolong(c, _oracle_weights(orc, w1), orc.Bounds(), 2)
    got = srmodel.sr_prolong(Grid(c), w1, NormBounds(), 2, precision="fp16").data
    assert rel_l2(got, exp) < 1e-2
    # B=16 with the crafted nearest-neighbour network (a He-init network this deep amplifies fp16
    # operand rounding to ~4% of its tanh output, so it would test the weights, not the kernel)
    w16 = srmodel.make_nearest_neighbor_weights(16)
    exp = orc.sr_prolong(c, _oracle_weights(orc, w16), orc.Bounds(), 2)
    got = srmodel.sr_prolong(Grid(c), w16, NormBounds(), 2, precision="fp16").data
    assert rel_l2(got, exp) < 1e-2
    w17 = srmodel.random_weights(17, 0)
    with pytest.raises(ValueError, match="too deep"):
        srmodel.sr_prolong(Grid(c), w17, NormBounds(), 2, precision="fp16")


@pytest.mark.parametrize("blocks", [4, 8])
def test_generator_forward_matches_reference_trainer_fixtures(cuda, blocks):
    """generator_forward replays the reference trainer's recorded forward passes (torch fp32, eval
    mode; tests/golden/make_trainer_fixtures.py) within the reference's trainer-parity bar 1e-4."""
    import os
    from paper_2403_07936_b200 import srmodel
    from conftest import GOLDEN
    fx = np.load(os.path.join(GOLDEN, "trainer_fixtures.npz"))
    w = _trained(blocks)
    for x, y in zip(fx[f"b{blocks}_inputs"], fx[f"b{blocks}_outputs"]):
        got = srmodel.generator_forward(w, x.astype(np.float64))
        assert np.abs(got - y).max() < 1e-4


@pytest.mark.parametrize("nc", [6, 8, 10, 14, 26])
def test_tc_ratio4_pass_tiny_and_ragged_grids(cuda, orc, nc):
    """Ratio-4 passes where every window is an edge window (nc = 6: one window; 8: 2 x 2) and where the
    window count leaves the last 2-window group of the second application half full (nc = 10, 14, 26):
    fp16 tensor cores against the fp64 oracle at the 1e-2 bar (trained B=8)."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(8)
    c = _fields(32)["smooth"][:nc, :nc]
    c = c - c.mean()
    exp = orc.sr_prolong(c, orc.quantize_f32(_oracle_weights(orc, w)), orc.Bounds(), 4)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp16").data
    assert rel_l2(got, exp) < 1e-2, rel_l2(got, exp)


def test_tc_ratio4_pass_bf16_operands(cuda, orc):
    """The bf16-operand instantiations of the ratio-4 kernels (V = 1, 2 with F16 = false) run and stay within
    their operand format's error (bf16 has 8x coarser mantissas than fp16: DESIGN.md "Operand precision"),
    and fp16 is the more accurate of the two."""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = _trained(8)
    c = _fields(40)["smooth"][:40, :40]
    c = c - c.mean()
    exp = orc.sr_prolong(c, orc.quantize_f32(_oracle_weights(orc, w)), orc.Bounds(), 4)
    eb = rel_l2(srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="bf16").data, exp)
    e16 = rel_l2(srmodel.sr_prolong(Grid(c), w, NormBounds(), 4, precision="fp16").data, exp)
    print(f"\nratio-4 pass relL2: bf16 {eb:.2e}, fp16 {e16:.2e}")
    assert e16 < eb < 5e-2


@pytest.mark.parametrize("weights", ["trained_b8", "trained_b4", "he_b1"])
@pytest.mark.parametrize("s,nc", [(8, 16), (8, 40), (16, 12), (16, 24)])
def test_mixed_two_pass_ratios_vs_oracle(cuda, orc, weights, s, nc):
    """precision="mixed" (the default): x8 / x16 prolongations with the first ratio-4 pass on the fp32 CUDA
    cores and the second pass (16x the windows) on the fp16 tensor cores, end to end against the fp64 oracle
    at the north-star 1e-2 bar.  (fp16 throughout lands at 5e-2 on these fields: the second pass amplifies
    the first pass's operand rounding; the reverse split -- first fp16, second exact -- shows the same
    4.8e-2 in the CPU emulation, the forward one 1.8e-3.)"""
    from paper_2403_07936_b200 import srmodel
    from paper_2403_07936_b200.grid import Grid, NormBounds
    w = {"trained_b8": lambda: _trained(8), "trained_b4": lambda: _trained(4),
         "he_b1": lambda: srmodel.random_weights(1, 3)}[weights]()
    c = _fields(max(nc, 16))["smooth"][:nc, :nc]
    c = c - c.mean()
    exp = orc.sr_prolong(c, orc.quantize_f32(_oracle_weights(orc, w)), orc.Bounds(), s)
    got = srmodel.sr_prolong(Grid(c), w, NormBounds(), s).data     # default precision: mixed
    assert rel_l2(got, exp) < 1e-2, rel_l2(got, exp)
