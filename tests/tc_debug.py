"""Bring-up harness (GPU): per-layer comparison of the tcgen05 generator against
a torch fp32 reference of the same windows.  Not collected by pytest.

    python tests/tc_debug.py [nc] [blocks]
"""

from __future__ import annotations

import ctypes
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_07936_b200 import _lib, srmodel  # noqa: E402


def conv(x, w):
    k = w.shape[-1]
    return F.conv2d(F.pad(x, (k // 2,) * 4, mode="replicate"), w)


def bn(x, t, pre):
    g, b, m, v = (torch.tensor(t[f"{pre}.{s}"], dtype=torch.float32, device="cuda")[None, :, None, None]
                  for s in ("gamma", "beta", "mean", "var"))
    return g * (x - m) / torch.sqrt(v + 1e-5) + b


def prelu(x, a):
    a = torch.tensor(a, dtype=torch.float32, device="cuda")[None, :, None, None]
    return torch.where(x > 0, x, a * x)


def torch_layers(w, x):
    t = {k: v for k, v in w.tensors.items()}
    T = lambda k: torch.tensor(t[k], dtype=torch.float32, device="cuda")  # noqa: E731
    outs = []
    y = prelu(conv(x, T("head.conv.weight")), t["head.prelu.alpha"])
    outs.append(y)
    skip = y
    for i in range(w.num_residual_blocks):
        z = prelu(bn(conv(y, T(f"res{i}.conv1.weight")), t, f"res{i}.bn1"), t[f"res{i}.prelu.alpha"])
        outs.append(z)
        y = y + bn(conv(z, T(f"res{i}.conv2.weight")), t, f"res{i}.bn2")
        outs.append(y)
    y = bn(conv(y, T("post.conv.weight")), t, "post.bn") + skip
    outs.append(y)
    up = F.pixel_shuffle(conv(y, T("up.conv.weight")), 2)
    u = prelu(up, t["up.prelu.alpha"])
    outs.append(u)
    out = conv(u, T("tail.conv.weight")) + T("tail.conv.bias")[None, :, None, None]
    s = w.tanh_scale
    return outs, s * torch.tanh(out / s)


F16 = 0


def main():
    global F16
    nc = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
    F16 = 1 if prec == "fp16" else 0
    blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    lib = _lib.load()
    lib.mgsr_debug_tc_pass.restype = ctypes.c_int
    lib.mgsr_debug_tc_pass.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
    w = srmodel.random_weights(blocks, 0)
    rng = np.random.default_rng(0)
    c = (10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)
    dc = torch.from_numpy(c).cuda()
    npos = nc // 2 - 2
    nw = npos * npos
    # q windows
    q = np.clip((np.log10(np.abs(c)) + 10) / 7, 0, 1) * np.sign(c)
    X = np.stack([q[2 * (k // npos):2 * (k // npos) + 6, 2 * (k % npos):2 * (k % npos) + 6] for k in range(nw)])
    x = torch.from_numpy(np.repeat(X[:, None], 3, axis=1)).float().cuda()
    ref_layers, ref_out = torch_layers(w, x)
    h = w.device_handle()
    nl = 2 * blocks + 1
    fine = torch.zeros((2 * nc, 2 * nc), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for L in range(nl + 2):
        size = nw * (144 if L == nl + 1 else 36) * 64
        dbg = torch.full((size,), float("nan"), dtype=torch.float32, device="cuda")
        _lib.check(lib.mgsr_debug_tc_pass(h, dc.data_ptr(), nc, 1e-10, 1e-3, fine.data_ptr(), dbg.data_ptr(), L, F16, st))
        torch.cuda.synchronize()
        side = 12 if L == nl + 1 else 6
        got = dbg.view(nw, side, side, 64).permute(0, 3, 1, 2)
        ref = ref_layers[L]
        err = float((got - ref).norm() / ref.norm())
        nan = int(torch.isnan(got).sum())
        print(f"layer {L:2d}: relL2 {err:.3e}  nan {nan}  max|ref| {float(ref.abs().max()):.3e}", flush=True)
    # final field vs fp32 SIMT path
    from paper_2403_07936_b200.grid import Grid, NormBounds
    a = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision=prec).data
    b = srmodel.sr_prolong(Grid(c), w, NormBounds(), 2, precision="fp32").data
    print(f"sr_prolong {prec} vs fp32: relL2 {np.linalg.norm(a - b) / np.linalg.norm(b):.3e}  "
          f"nan {int(np.isnan(a).sum())}")


if __name__ == "__main__":
    main()
