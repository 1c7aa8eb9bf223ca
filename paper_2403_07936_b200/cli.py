"""``mgsr``-compatible command line over the B200 path (``python -m paper_2403_07936_b200.cli``).

Mirrors the reference CLI's user-facing contract (cli.py:1-6, 314-393): the same subcommands
``solve`` / ``sweep`` / ``spectrum`` / ``bench`` / ``datagen`` (kinds ``mode`` and ``turb``), the same
flags and JSON RunConfig with flag overrides, ``MGSR_SEED``, the same CSV columns and summary
line, and the same exit codes (0 converged / ok, 2 usage or configuration error, 3 iteration
budget exhausted).  What changes is where the work runs:

* ``solve`` runs ``solver.solve`` (device-resident loop, one graph launch for the whole solve);
  ``--precision`` / ``--sr-levels`` select the generator path and the per-level SR mask.
* ``sweep`` does not fan solves out over processes (cli.py:237-241): tasks that share a grid side
  and configuration go to ``solver.solve_batch`` together (concurrent on one GPU).  ``--jobs`` is
  accepted for compatibility; the rows are identical and sorted the same way.
* ``bench`` times the ``cuda`` kernel backend's ``gs_sweeps`` / ``laplacian`` (cli.py:268-311) with
  host arrays (the plugin call, copies included) and with device tensors.
* ``datagen --kind windows`` writes the generator trainer's corpus (MGWP), which is outside the
  V-cycle path; it raises a configuration error here.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

from . import srmodel, transfer
from .grid import Grid, read_grid, write_grid
from .smoother import PoissonProblem
from .solver import RunConfig, solve, solve_batch

SWEEP_COLUMNS = ("param", "value", "replicate", "rhs_id", "iters_to_converge", "converged", "final_diff")
SWEEP_PARAMS = ("N_smooth", "N_GAN", "S_thres", "N_grid", "k_peak")
PRECISIONS = ("fp32", "bf16", "fp16", "mixed")


class CliError(Exception):
    """A usage / configuration problem: exit code 2."""


def _seed_from_env() -> int:
    raw = os.environ.get("MGSR_SEED", "0")
    try:
        return int(raw)
    except ValueError:
        raise CliError(f"MGSR_SEED must be an integer, got {raw!r}") from None


def _config(path: str | None, **overrides) -> RunConfig:
    if path is None:
        cfg = RunConfig(seed=_seed_from_env())
    else:
        try:
            text = Path(path).read_text()
        except FileNotFoundError:
            raise CliError(f"config file not found: {path}") from None
        try:
            cfg = RunConfig.from_json(text)
        except (json.JSONDecodeError, ValueError, TypeError) as exc:
            raise CliError(f"bad config: {exc}") from None
    given = {k: v for k, v in overrides.items() if v is not None}
    if not given:
        return cfg
    try:
        return replace(cfg, **given)
    except ValueError as exc:
        raise CliError(f"bad config override: {exc}") from None


def _rhs(path: str) -> PoissonProblem:
    try:
        g = read_grid(path)
    except FileNotFoundError:
        raise CliError(f"RHS file not found: {path}") from None
    except ValueError as exc:
        raise CliError(f"bad RHS file {path}: {exc}") from None
    return PoissonProblem(f=g.mean_subtracted())


def _weights_for(cfg: RunConfig):
    if cfg.mode == "spline":
        return None
    if cfg.weights is None:
        raise CliError(f"mode {cfg.mode!r} requires --weights")
    try:
        return srmodel.load_weights(cfg.weights)
    except (FileNotFoundError, ValueError) as exc:
        raise CliError(f"bad weights file {cfg.weights}: {exc}") from None


def cmd_solve(a) -> int:
    cfg = _config(a.config, N_iter=a.n_iter, N_smooth=a.n_smooth, N_GAN=a.n_gan, S_thres=a.s_thres, tol=a.tol,
                  mode=a.mode, weights=a.weights, seed=a.seed)
    prob = _rhs(a.rhs)
    w = _weights_for(cfg)
    try:
        p, log = solve(prob, cfg, w, precision=a.precision, sr_levels=a.sr_levels)
    except ValueError as exc:
        raise CliError(str(exc)) from None
    if a.out_grid:
        write_grid(p, a.out_grid)
    if a.out_log:
        log.write_csv(a.out_log)
    ops = [r.operator for r in log.records]
    ok = log.converged(cfg.tol)
    print(f"iterations={log.iterations} converged={ok} final_diff={log.final_diff:.3e} "
          f"spline={ops.count('spline')} sr={ops.count('sr')}")
    return 0 if ok else 3


def _resample(f: Grid, n: int) -> Grid:
    """RHS onto side n: Keys prolongation up, injection down (the reference's sweep resampling)."""
    if n == f.n:
        return f
    big, small = (n, f.n) if n > f.n else (f.n, n)
    ratio = big // small
    if ratio * small != big:
        raise CliError(f"cannot resample {f.n} -> {n}")
    out = transfer.spline_prolong(f, ratio) if n > f.n else transfer.restrict(f, ratio)
    return out.mean_subtracted()


def _values(param: str, raw: str) -> list:
    conv = int if param in ("N_smooth", "N_grid", "k_peak") else float
    vals = [conv(t.strip()) for t in raw.split(",") if t.strip()]
    if not vals:
        raise CliError("--values must list at least one value")
    return vals


def cmd_sweep(a) -> int:
    if a.param not in SWEEP_PARAMS:
        raise CliError(f"--param must be one of {SWEEP_PARAMS}, got {a.param!r}")
    if a.replicates < 1:
        raise CliError("--replicates must be >= 1")
    vals = _values(a.param, a.values)
    base = _config(a.config, seed=a.seed)
    # task = (value, replicate, rhs_id, f, cfg); grouped below by (side, cfg) for batched solves
    tasks = []
    if a.param == "k_peak":
        if base.N_grid is None:
            raise CliError("k_peak sweeps need N_grid in the config")
        from .spectral import turbulent_source
        for v in vals:
            for rep in range(a.replicates):
                f, _, _ = turbulent_source(base.N_grid, v, base.seed + rep, p_rms=a.p_rms)
                tasks.append((v, rep, f"kpeak{v}", f, replace(base, N_grid=None)))
    else:
        if not a.rhs:
            raise CliError("--rhs is required for this sweep parameter")
        grids = {Path(p).stem: _rhs(p).f for p in (t.strip() for t in a.rhs.split(",")) if p}
        for v in vals:
            cfg_v = replace(base, N_grid=None) if a.param == "N_grid" else replace(base, **{a.param: v}, N_grid=None)
            for rid, f in grids.items():
                fv = _resample(f, v) if a.param == "N_grid" else f
                for rep in range(a.replicates):
                    tasks.append((v, rep, rid, fv, cfg_v))
    groups: dict = {}
    for i, (v, rep, rid, f, cfg) in enumerate(tasks):
        cfg_r = replace(cfg, seed=cfg.seed + rep)
        groups.setdefault((f.n, cfg_r.to_json()), []).append((i, PoissonProblem(f=f.mean_subtracted()), cfg_r))
    rows = [None] * len(tasks)
    for (_, _), items in groups.items():
        cfg = items[0][2]
        w = _weights_for(cfg)
        try:
            res = solve_batch([pr for _, pr, _ in items], cfg, w, precision=a.precision, sr_levels=a.sr_levels)
        except ValueError as exc:
            raise CliError(str(exc)) from None
        for (i, _, cfg_i), (_, log) in zip(items, res):
            v, rep, rid, _, _ = tasks[i]
            ok = log.converged(cfg_i.tol)
            iters = None
            if ok:
                iters = log.iterations * cfg_i.N_smooth / 20.0 if a.scale_iters else log.iterations
            rows[i] = (a.param, v, rep, rid, iters, int(ok), log.final_diff)
    rows.sort(key=lambda r: (str(r[0]), float(r[1]), int(r[2]), str(r[3])))
    with open(a.out, "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(SWEEP_COLUMNS)
        wr.writerows(rows)
    print(f"wrote {a.out} ({len(rows)} rows)")
    return 0


def cmd_spectrum(a) -> int:
    from .spectral import power_spectrum
    try:
        g = read_grid(a.infile)
    except (FileNotFoundError, ValueError) as exc:
        raise CliError(f"bad grid file {a.infile}: {exc}") from None
    sp = power_spectrum(g, peak_normalize=a.peak_normalize)
    with open(a.out, "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(("k", "power"))
        wr.writerows((int(k), f"{p:.17e}") for k, p in zip(sp.k, sp.power))
    print(f"wrote {a.out} ({len(sp.k)} bins)")
    return 0


def _best(fn, repeats: int, sync=None) -> float:
    best = float("inf")
    for _ in range(repeats):
        t0 = time.perf_counter()
        fn()
        if sync:
            sync()
        best = min(best, time.perf_counter() - t0)
    return best


def cmd_bench(a) -> int:
    from . import _lib, kernels
    torch = _lib.require_cuda()
    sizes = [int(t) for t in a.sizes.split(",") if t.strip()]
    rng = np.random.default_rng(0)
    rows = []
    for n in sizes:
        f = rng.standard_normal((n, n))
        f -= f.mean()
        h2 = (2.0 * np.pi / n) ** 2
        p = np.zeros((n, n))
        host_gs = _best(lambda: kernels.gs_sweeps(p, f, h2, a.sweeps), a.repeats)
        host_lap = _best(lambda: kernels.laplacian(p, 1.0 / h2), a.repeats)
        rows.append((n, "cuda-host", host_gs / a.sweeps * 1e3, host_lap * 1e3))
        pd, fd = torch.zeros((n, n), dtype=torch.float64, device="cuda"), torch.from_numpy(f).cuda()
        sync = torch.cuda.synchronize
        dev_gs = _best(lambda: kernels.gs_sweeps(pd, fd, h2, a.sweeps), a.repeats, sync)
        dev_lap = _best(lambda: kernels.laplacian(pd, 1.0 / h2), a.repeats, sync)
        rows.append((n, "cuda-device", dev_gs / a.sweeps * 1e3, dev_lap * 1e3))
    print(f"{'n':>6} {'backend':>12} {'ms/sweep':>10} {'ms/laplacian':>13}")
    for n, name, g, lap in rows:
        print(f"{n:>6} {name:>12} {g:>10.3f} {lap:>13.3f}")
    if a.out:
        with open(a.out, "w", newline="") as fh:
            wr = csv.writer(fh)
            wr.writerow(("n", "backend", "gs_ms_per_sweep", "laplacian_ms"))
            wr.writerows(rows)
    return 0


def cmd_datagen(a) -> int:
    from . import spectral
    seed = a.seed if a.seed is not None else _seed_from_env()
    stem = Path(a.out)
    stem = stem.with_suffix("") if stem.suffix == ".mgg" else stem
    if a.kind == "mode":
        if a.mode_k is None:
            raise CliError("--mode-k is required for --kind mode")
        p, f = spectral.single_mode_field(a.n, a.mode_k)
        write_grid(f, f"{stem}_f.mgg")
        write_grid(p, f"{stem}_p.mgg")
        print(f"wrote {stem}_f.mgg and {stem}_p.mgg (n={a.n}, k={a.mode_k})")
        return 0
    if a.kind == "turb":
        f, flow, p = spectral.turbulent_source(a.n, a.k_peak, seed, p_rms=a.p_rms)
        for tag, g in (("f", f), ("p", p), ("u", flow.u), ("v", flow.v)):
            write_grid(g, f"{stem}_{tag}.mgg")
        print(f"wrote {stem}_{{f,p,u,v}}.mgg (n={a.n}, k_peak={a.k_peak}, seed={seed})")
        return 0
    raise CliError("--kind windows builds the generator trainer's corpus, which is not part of the V-cycle path")


def _common_solver_flags(sp):
    sp.add_argument("--precision", choices=PRECISIONS, default=None,
                    help="generator path for SR prolongations (default MGSR_PRECISION or mixed: tcgen05 tensor cores "
                         "with an exact first pass for x8/x16; fp16/bf16: tensor cores throughout; fp32: the exact "
                         "CUDA-core mode)")
    sp.add_argument("--sr-levels", type=int, default=None,
                    help="SR only at the N finest prolongations (spline below); default: every level")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="mgsr-b200", description="Multigrid Poisson solver with spline or "
                                 "super-resolution prolongation on a B200")
    sub = ap.add_subparsers(dest="command", required=True)
    s = sub.add_parser("solve", help="solve laplace(p) = f from an MGG1 file")
    s.add_argument("--rhs", required=True)
    s.add_argument("--config", default=None)
    s.add_argument("--weights", default=None)
    s.add_argument("--mode", choices=("spline", "sr", "hybrid"), default=None)
    for flag, typ in (("--n-iter", int), ("--n-smooth", int), ("--n-gan", float), ("--s-thres", float),
                      ("--tol", float), ("--seed", int)):
        s.add_argument(flag, type=typ, default=None)
    s.add_argument("--out-grid", default=None)
    s.add_argument("--out-log", default=None)
    _common_solver_flags(s)
    s.set_defaults(fn=cmd_solve)
    s = sub.add_parser("sweep", help="parameter sweep over repeated solves")
    s.add_argument("--param", required=True)
    s.add_argument("--values", required=True)
    s.add_argument("--replicates", type=int, default=1)
    s.add_argument("--rhs", default=None)
    s.add_argument("--config", default=None)
    s.add_argument("--p-rms", type=float, default=None)
    s.add_argument("--scale-iters", action="store_true")
    s.add_argument("--jobs", type=int, default=1, help="accepted for compatibility (solves are batched on the GPU)")
    s.add_argument("--seed", type=int, default=None)
    s.add_argument("--out", required=True)
    _common_solver_flags(s)
    s.set_defaults(fn=cmd_sweep)
    s = sub.add_parser("spectrum", help="radial power spectrum of a grid")
    s.add_argument("--in", dest="infile", required=True)
    s.add_argument("--peak-normalize", action="store_true")
    s.add_argument("--out", required=True)
    s.set_defaults(fn=cmd_spectrum)
    s = sub.add_parser("bench", help="time the cuda kernel backend")
    s.add_argument("--sizes", default="96,192,384")
    s.add_argument("--sweeps", type=int, default=20)
    s.add_argument("--repeats", type=int, default=3)
    s.add_argument("--out", default=None)
    s.set_defaults(fn=cmd_bench)
    s = sub.add_parser("datagen", help="generate synthetic problems")
    s.add_argument("--kind", choices=("mode", "turb", "windows"), required=True)
    s.add_argument("--n", type=int, required=True)
    s.add_argument("--mode-k", type=int, default=None)
    s.add_argument("--k-peak", type=int, default=8)
    s.add_argument("--p-rms", type=float, default=None)
    s.add_argument("--count", type=int, default=1000)
    s.add_argument("--fields", type=int, default=50)
    s.add_argument("--seed", type=int, default=None)
    s.add_argument("--out", required=True)
    s.set_defaults(fn=cmd_datagen)
    return ap


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (CliError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
