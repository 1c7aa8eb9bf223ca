"""CPU: host logic of the package and the C ABI boundary (no compute calls)."""

from __future__ import annotations

import ctypes
import os
import re
import struct

import numpy as np
import pytest

from conftest import ROOT


def header_symbols() -> list[str]:
    text = open(os.path.join(ROOT, "include", "mgsr_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mgsr_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    from paper_2403_07936_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 17
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert lib.mgsr_version().startswith(b"mgsr_b200")
    assert lib.mgsr_workspace_bytes(4096) > 0


def test_plan_config_layout_matches_header():
    from paper_2403_07936_b200 import _lib
    # int64 n; 4 x int32; 2 x double; int32 precision; uint32 mask
    assert ctypes.sizeof(_lib.PlanConfig) == 8 + 16 + 16 + 8


def test_runconfig_mirrors_reference():
    from paper_2403_07936_b200.solver import RunConfig
    c = RunConfig()
    assert (c.N_iter, c.r_min, c.N_smooth_pre, c.N_smooth, c.N_step, c.N_GAN, c.S_thres, c.tol, c.mode,
            c.coarse_sweeps) == (300, 12, 10, 20, 4, 1.0, 1e-10, 1e-10, "spline", 10)
    with pytest.raises(ValueError, match="unknown config keys"):
        RunConfig.from_json('{"N_iter": 3, "bogus": 1}')
    with pytest.raises(ValueError, match="must be one of"):
        RunConfig(mode="gan")
    with pytest.raises(ValueError, match="even integer"):
        RunConfig(r_min=7)
    assert RunConfig.from_json(RunConfig(N_iter=7).to_json()) == RunConfig(N_iter=7)


@pytest.mark.parametrize("n,step,rmin,expected", [
    (4096, 1, 8, [4096, 2048, 1024, 512, 256, 128, 64, 32, 16, 8]),
    (192, 4, 12, [192, 12]),
    (3072, 4, 12, [3072, 192, 12]),
    (64, 1, 8, [64, 32, 16, 8]),
])
def test_level_sides(n, step, rmin, expected, orc):
    from paper_2403_07936_b200.solver import level_sides
    assert level_sides(n, step, rmin) == expected == orc.level_sides(n, step, rmin)


def test_level_sides_errors():
    from paper_2403_07936_b200.solver import level_sides
    with pytest.raises(ValueError, match="must exceed"):
        level_sides(12, 1, 12)
    with pytest.raises(ValueError, match="no valid ladder"):
        level_sides(100, 1, 12)


def test_schedule_matches_oracle(orc):
    from paper_2403_07936_b200.solver import schedule_operator
    for n_gan in (0.25, 0.5, 1.0, 2.0, 3.0, 7.6):
        for latched in (False, True):
            for it in range(1, 30):
                assert schedule_operator(it, n_gan, latched) == orc.schedule_operator(it, n_gan, latched)
    with pytest.raises(ValueError):
        schedule_operator(0, 1.0, False)


def test_weights_roundtrip_and_errors(tmp_path):
    from paper_2403_07936_b200 import srmodel
    w = srmodel.random_weights(2, 5)
    path = tmp_path / "w.mgsr"
    srmodel.save_weights(w, path)
    back = srmodel.load_weights(path)
    for k, v in w.tensors.items():
        assert np.array_equal(back.tensors[k], v.astype(np.float32).astype(np.float64))
    nn = srmodel.make_nearest_neighbor_weights()
    srmodel.save_weights(nn, tmp_path / "nn.mgsr")
    assert srmodel.load_weights(tmp_path / "nn.mgsr").tanh_scale == 1e6
    blob = path.read_bytes()
    (tmp_path / "bad.mgsr").write_bytes(b"NOPE" + blob[4:])
    with pytest.raises(srmodel.WeightsMagicError, match="bad magic"):
        srmodel.load_weights(tmp_path / "bad.mgsr")
    (tmp_path / "trunc.mgsr").write_bytes(blob[: len(blob) // 2])
    with pytest.raises(srmodel.WeightsTruncatedError, match="bytes"):
        srmodel.load_weights(tmp_path / "trunc.mgsr")
    (tmp_path / "trail.mgsr").write_bytes(blob + b"\0")
    with pytest.raises(srmodel.WeightsShapeError, match="trailing"):
        srmodel.load_weights(tmp_path / "trail.mgsr")
    ver = bytearray(blob)
    ver[4:8] = struct.pack("<I", 9)
    (tmp_path / "ver.mgsr").write_bytes(bytes(ver))
    with pytest.raises(srmodel.WeightsVersionError, match="version"):
        srmodel.load_weights(tmp_path / "ver.mgsr")
    for sub in (srmodel.WeightsMagicError, srmodel.WeightsVersionError, srmodel.WeightsShapeError,
                srmodel.WeightsTruncatedError):
        assert issubclass(sub, srmodel.WeightsError) and issubclass(sub, ValueError)


def test_random_weights_match_oracle(orc):
    from paper_2403_07936_b200 import srmodel
    w = srmodel.random_weights(8, 0)
    o = orc.random_weights(8, 0)
    for k in o.tensors:
        assert np.array_equal(w.tensors[k], o.tensors[k])


def test_window_plan_matches_oracle(orc):
    from paper_2403_07936_b200 import srmodel
    for n in (6, 8, 16, 30):
        mine = [(a, b, s1.start, s1.stop, s2.start, s2.stop) for a, b, s1, s2 in srmodel.stitch_plan(n)]
        assert mine == orc.stitch_plan(n)
    with pytest.raises(ValueError, match=">= 6"):
        srmodel.window_positions(4)
    with pytest.raises(ValueError, match="even"):
        srmodel.window_positions(7)


def test_backend_selector_rejects_unknown(monkeypatch):
    import importlib
    import subprocess
    import sys
    code = "import paper_2403_07936_b200.kernels"
    env = dict(os.environ, MGSR_BACKEND="numpy", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode != 0 and "MGSR_BACKEND" in r.stderr
    from paper_2403_07936_b200 import kernels
    assert kernels.active_backend() == "cuda"


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_07936_b200 import kernels
    p = np.zeros((8, 8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        kernels.gs_sweeps(p, p.copy(), 1.0, 1)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2403_07936_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f


def test_replicas_gloo_world2(tmp_path):
    """bench.py --gpus 2 host logic on CPU: two gloo ranks (127.0.0.1), max-over-ranks
    time, whole-job value = replicas x steps / max time, distinct seeded inputs per rank."""
    import json
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PYTHONPATH=ROOT)
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_replica_worker.py"),
                                       str(tmp_path)], env=env))
    for pr in procs:
        assert pr.wait(timeout=240) == 0
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(2)]
    for r in res:
        assert r["ms"] == 150.0                        # the slower rank's time, on every rank
        assert abs(r["value"] - 2 * 10 / 0.150) < 1e-9
        assert abs(r["f_mean"]) < 1e-12                # mean-free RHS
    d = res[0]["digests"]
    assert d == res[1]["digests"] and d[0] != d[1]     # each replica solves its own RHS


@pytest.mark.parametrize("n_gan", [0.25, 0.5, 1.0, 2.0, 3.0, 1.5])
def test_device_schedule_matches_schedule_operator(n_gan):
    """The operator rule k_solve_pre evaluates on device (cadence, first_sr, N_GAN == 1; see
    mgsr_plan_solve) reproduces schedule_operator (solver.py:122-144) for every iteration and latch."""
    from paper_2403_07936_b200.solver import _cadence, schedule_operator
    cad, first_sr, one = _cadence(n_gan)

    def device_rule(it, latched):   # mirror of k_solve_pre for mode = hybrid
        if latched:
            sr = not first_sr
        elif one:
            sr = bool(it & 1)
        else:
            sr = bool(first_sr) if it % cad != 0 else not first_sr
        return "sr" if sr else "spline"

    for latched in (False, True):
        for it in range(1, 40):
            assert device_rule(it, latched) == schedule_operator(it, n_gan, latched)


def test_solve_batch_rejects_mixed_sizes():
    from paper_2403_07936_b200 import solver
    from paper_2403_07936_b200.grid import Grid
    from paper_2403_07936_b200.smoother import PoissonProblem
    a = PoissonProblem(Grid(np.zeros((16, 16))))
    b = PoissonProblem(Grid(np.zeros((32, 32))))
    with pytest.raises(ValueError, match="same side"):
        solver.solve_batch([a, b], solver.RunConfig())


# ---- the algorithm of mgsr_initial_iterate (csrc/rng.cu), restated with Python integers and
# checked against numpy: PCG64 jump-ahead + XSL-RR output + uniform, and the pairwise mean ----

_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1


def _pcg_advance(state, delta, inc):
    cur_mult, cur_plus, acc_mult, acc_plus = _PCG_MULT, inc, 1, 0
    while delta > 0:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & _M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & _M128
        cur_plus = ((cur_mult + 1) * cur_plus) & _M128
        cur_mult = (cur_mult * cur_mult) & _M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & _M128


def _pcg_draw(state, inc):
    state = (state * _PCG_MULT + inc) & _M128
    x = ((state >> 64) ^ state) & ((1 << 64) - 1)
    rot = state >> 122
    return state, ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)


@pytest.mark.parametrize("seed", [0, 7, 12345])
def test_pcg64_jump_ahead_matches_numpy_stream(seed):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s0, inc = int(st["state"]), int(st["inc"])
    ref = np.random.default_rng(seed).uniform(-1e-3, 1e-3, size=4096)
    for off in (0, 1, 127, 128, 1000, 4095):   # a thread's leaf starts at a jump-ahead offset
        s = _pcg_advance(s0, off, inc)
        _, u = _pcg_draw(s, inc)
        d = (u >> 11) * (1.0 / 9007199254740992.0)
        assert -1e-3 + (1e-3 - (-1e-3)) * d == ref[off]


@pytest.mark.parametrize("n", [16, 64, 256, 1024])
def test_pairwise_leaf_tree_equals_numpy_mean(n):
    a = np.random.default_rng(n).uniform(-1e-3, 1e-3, size=(n, n))
    leaves = a.reshape(-1, 16, 8)             # 128 values per leaf, 8 interleaved accumulators
    r = leaves[:, 0, :].copy()
    for k in range(1, 16):
        r = r + leaves[:, k, :]
    s = ((r[:, 0] + r[:, 1]) + (r[:, 2] + r[:, 3])) + ((r[:, 4] + r[:, 5]) + (r[:, 6] + r[:, 7]))
    while s.size > 1:
        s = s[0::2] + s[1::2]
    assert (0.0 + s[0]) / (n * n) == a.mean()


def test_solve_batch_distributed_gloo_world2(tmp_path):
    """Config 5 across ranks (replicas only): round-robin shards, results gathered in input order on
    every rank, each RHS solved exactly once."""
    import json
    import socket
    import subprocess
    import sys
    from paper_2403_07936_b200 import solver
    assert solver.shard_indices(5, 0, 2) == [0, 2, 4] and solver.shard_indices(5, 1, 2) == [1, 3]
    with pytest.raises(ValueError):
        solver.shard_indices(4, 2, 2)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), PYTHONPATH=ROOT)
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_shard_worker.py"),
                                       str(tmp_path)], env=env))
    for pr in procs:
        assert pr.wait(timeout=240) == 0
    res = [json.load(open(tmp_path / f"shard{r}.json")) for r in range(2)]
    assert sorted(res[0]["seen"] + res[1]["seen"]) == [0, 1, 2, 3, 4]
    for r in res:
        assert r["order"] == [0.0, 1.0, 2.0, 3.0, 4.0]
        assert r["solved_by"] == [0.0, 1.0, 0.0, 1.0, 0.0]


def test_bench_gpus2_self_launch_gloo():
    """`python bench.py --gpus 2` outside torchrun re-executes itself under torch.distributed.run with
    two ranks (127.0.0.1 rendezvous); the line reports n_gpus 2 and the whole-job value from the
    slower rank's time (plumbing self-test: gloo, fake per-rank times 100 / 110 ms)."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing-test",
                          "--steps", "4", "--warmup", "3"], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "replicas x2"
    assert abs(d["value"] - 2 * 4 / 0.110) < 1e-9


def test_custom_op_fake_kernels():
    """The torch.library ops carry fake (meta) kernels: shapes propagate under FakeTensorMode without the
    CUDA library or a GPU."""
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode
    from paper_2403_07936_b200 import ops  # noqa: F401
    with FakeTensorMode():
        p = torch.empty(64, 64, dtype=torch.float64)
        assert torch.ops.mgsr.laplacian(p, 1.0).shape == (64, 64)
        assert torch.ops.mgsr.residual(p, p).shape == (64, 64)
        assert torch.ops.mgsr.restrict(p, 4, True).shape == (16, 16)
        assert torch.ops.mgsr.spline_prolong(p, 4).shape == (256, 256)
        assert torch.ops.mgsr.sr_prolong(p, 0, 16, 1e-10, 1e-3, 2).shape == (1024, 1024)
        x = torch.empty(5, 3, 6, 6, dtype=torch.float64)
        assert torch.ops.mgsr.generator_forward(x, 0).shape == (5, 3, 12, 12)
