"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``mgsr`` -- preferring the Cython-compiled
build in ``oracle/_ref`` (the reference's default "auto" backend when its
extension is built), else the pure-Python tree under /root/reference -- runs
the hot-path functions on small seeded inputs and writes ``golden.npz``
(plus the reference's own trainer fixtures copied from the regenerated
artifacts when available).  The fixtures travel with the repo; the GPU box
never needs /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def load_reference():
    import oracle
    ref = oracle.import_ref()
    if ref is None:
        sys.path.insert(0, "/root/reference/pkg/src")
        import mgsr  # noqa: F401
    import mgsr
    return mgsr


def main() -> None:
    mgsr = load_reference()
    from mgsr import kernels, smoother, solver, srmodel, transfer
    from mgsr.grid import Grid, NormBounds, _denormalize_array, _normalize_array
    from mgsr.kernels import numpy_backend
    from oracle import mgsr_oracle as orc

    g: dict[str, np.ndarray] = {}
    meta = {"backend": kernels.active_backend()}
    rng = np.random.default_rng(1234)

    # --- stencil kernels (kernels/_stencil.pyx) ---
    for n in (8, 16, 64):
        p = rng.standard_normal((n, n)); p -= p.mean()
        f = rng.standard_normal((n, n)); f -= f.mean()
        h2 = (2 * np.pi / n) ** 2
        out = p.copy(); kernels.gs_sweeps(out, f, h2, 3)
        outn = p.copy(); numpy_backend.gs_sweeps(outn, f, h2, 3)
        g[f"gs{n}_p"], g[f"gs{n}_f"], g[f"gs{n}_out"], g[f"gs{n}_out_numpy"] = p, f, out, outn
    p9 = rng.standard_normal((9, 9))
    g["lap9_p"], g["lap9_out"] = p9, kernels.laplacian(p9, 1.0 / (2 * np.pi / 9) ** 2)

    # --- residual / restrict / spline (smoother.py, transfer.py) ---
    p = rng.standard_normal((32, 32)); f = rng.standard_normal((32, 32)); f -= f.mean()
    g["res_p"], g["res_f"] = p, f
    g["res_out"] = smoother.residual(Grid(p), smoother.PoissonProblem(Grid(f))).data
    g["restrict_out"] = transfer.restrict(Grid(p), 2).data
    g["restrict4_raw"] = transfer.restrict(Grid(p), 4, subtract_mean=False).data
    for s in (2, 4, 8, 16):
        c = rng.standard_normal((8, 8))
        g[f"spline{s}_c"], g[f"spline{s}_out"] = c, transfer.spline_prolong(Grid(c), s).data

    # --- normalisation (grid.py:103-114) ---
    vals = np.concatenate([rng.standard_normal(64) * 10.0 ** rng.uniform(-12, -1, 64), [0.0, 1e-10, -1e-3]])
    q, sg = _normalize_array(vals, NormBounds())
    g["norm_in"], g["norm_q"], g["norm_back"] = vals, q, _denormalize_array(q, sg, NormBounds())

    # --- generator (srmodel.py) ---
    w1 = srmodel.random_weights(1, 3)
    x6 = rng.uniform(-1, 1, (3, 6, 6))
    x8 = rng.uniform(-1, 1, (3, 8, 8))
    g["gen_b1_x6"], g["gen_b1_y6"] = x6, srmodel.generator_forward(w1, x6)
    g["gen_b1_x8"], g["gen_b1_y8"] = x8, srmodel.generator_forward(w1, x8)
    w8 = srmodel.random_weights(8, 0)
    x6b = np.repeat(rng.uniform(-1, 1, (1, 6, 6)), 3, axis=0)
    g["gen_b8_x6"], g["gen_b8_y6"] = x6b, srmodel.generator_forward(w8, x6b)

    # --- windowed SR prolongation (srmodel.py:443-487) ---
    from conftest_shim import in_band_values
    c16 = in_band_values((16, 16), 5); c16 -= c16.mean()
    w2 = srmodel.random_weights(2, 0)
    g["sr_c16"] = c16
    g["sr2_out"] = srmodel.sr_prolong(Grid(c16), w2, NormBounds(), 2).data
    c12 = in_band_values((12, 12), 6); c12 -= c12.mean()
    g["sr_c12"], g["sr4_out"] = c12, srmodel.sr_prolong(Grid(c12), w2, NormBounds(), 4).data
    nn = srmodel.make_nearest_neighbor_weights()
    g["srnn2_out"] = srmodel.sr_prolong(Grid(c16), nn, NormBounds(), 2).data

    # --- V-cycle / solve (solver.py) ---
    f32 = orc.sine_modes_rhs(32, 0)
    cfg = solver.RunConfig(N_step=1, r_min=8, N_smooth=2, N_smooth_pre=2)
    prob = smoother.PoissonProblem(Grid(f32))
    p0 = orc.initial_iterate(32, orc.Config(N_step=1, r_min=8, N_smooth=2))
    g["vc_f"], g["vc_p"] = f32, p0
    g["vc_spline_out"] = solver.v_cycle(Grid(p0), prob, cfg, "spline").data
    f32s = orc.scale_to_p_rms(f32, 1e-4)
    probs = smoother.PoissonProblem(Grid(f32s))
    p0s = orc.initial_iterate(32, orc.Config()) * 0.1
    g["vc_sr_f"], g["vc_sr_p"] = f32s, p0s
    g["vc_sr_out"] = solver.v_cycle(Grid(p0s), probs, cfg, "sr", w2).data

    f64 = orc.sine_modes_rhs(64, 0)
    cfg1 = solver.RunConfig(N_step=1, r_min=8, N_smooth=2)
    p, log = solver.solve(smoother.PoissonProblem(Grid(f64)), cfg1)
    g["solve64_f"], g["solve64_p"] = f64, p.data
    g["solve64_log"] = np.array([[r.diff_norm, r.residual_norm] for r in log.records])

    f64s = orc.scale_to_p_rms(f64, 1e-4)
    cfg2 = solver.RunConfig(N_step=1, r_min=8, N_smooth=2, mode="hybrid", N_GAN=1.0, S_thres=2.27e-4)
    p, log = solver.solve(smoother.PoissonProblem(Grid(f64s)), cfg2, srmodel.random_weights(1, 0))
    g["hyb64_f"], g["hyb64_p"] = f64s, p.data
    g["hyb64_log"] = np.array([[r.diff_norm, r.residual_norm] for r in log.records])
    meta["hyb64_ops"] = [r.operator for r in log.records]
    meta["hyb64_latched"] = [bool(r.switch_latched) for r in log.records]

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"wrote {len(g)} arrays; backend={meta['backend']}")


if __name__ == "__main__":
    sys.path.insert(0, HERE)
    main()
