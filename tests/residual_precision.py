"""Bring-up (CPU): generator-output error of fp16 operands with an fp32 vs an fp16 residual stream,
against fp64 (oracle conv2d), trained and He-init B=8 weights.  Not collected by pytest."""
import os, sys
import numpy as np
ROOT = "/root/repo"; sys.path.insert(0, ROOT)
from oracle import mgsr_oracle as O
from paper_2403_07936_b200 import srmodel, datagen
r16 = lambda a: a.astype(np.float16).astype(np.float64)
def bnfold(t, pre):
    g, b, m, v = (t[f"{pre}.{s}"] for s in ("gamma", "beta", "mean", "var"))
    sc = g / np.sqrt(v + 1e-5); return sc, b - sc * m
def fwd(t, B, x, mode):
    R = (lambda a: a) if mode == "exact" else r16
    conv = lambda y, w: O.conv2d(R(y), R(w))
    y = O._prelu(O.conv2d(R(x), R(t["head.conv.weight"])), t["head.prelu.alpha"])
    skip = y.astype(np.float32).astype(np.float64) if mode != "exact" else y
    for i in range(B):
        s1, h1 = bnfold(t, f"res{i}.bn1"); s2, h2 = bnfold(t, f"res{i}.bn2")
        z = O._prelu(conv(y, t[f"res{i}.conv1.weight"] * s1[:, None, None, None]) + h1[None, :, None, None], t[f"res{i}.prelu.alpha"])
        d = conv(z, t[f"res{i}.conv2.weight"] * s2[:, None, None, None]) + h2[None, :, None, None]
        y = (r16(y) if mode == "f16res" else y) + d
    s, h = bnfold(t, "post.bn")
    y = conv(y, t["post.conv.weight"] * s[:, None, None, None]) + h[None, :, None, None] + skip
    y = O._prelu(O.pixel_shuffle(conv(y, t["up.conv.weight"])), t["up.prelu.alpha"])
    y = conv(y, t["tail.conv.weight"]) + t["tail.conv.bias"][None, :, None, None]
    return np.tanh(y)
rng = np.random.default_rng(0); nc = 64
noise = (10.0 ** rng.uniform(-7, -3.5, (nc, nc))) * np.where(rng.random((nc, nc)) < 0.5, -1, 1)
f = datagen.scale_to_p_rms(datagen.grf_blobs_rhs(nc, seed=3, kmax=nc / 8), 1e-5)
smooth = datagen.spectral_solution(f)
def windows(c):
    q = np.sign(c) * np.clip((np.log10(np.abs(c)) + 10) / 7, 0, 1)
    pos = range(0, nc - 5, 4)
    w = np.stack([q[i:i + 6, j:j + 6] for i in pos for j in pos])
    return np.repeat(w[:, None], 3, axis=1)
for wn, w in (("he", srmodel.random_weights(8, 0)), ("trained", srmodel.load_weights(ROOT + "/artifacts/trained_b8.mgsr"))):
    t = {k: np.asarray(v, dtype=np.float64) for k, v in w.tensors.items()}
    for inn, c in (("noise", noise), ("smooth", smooth)):
        x = windows(c)
        ex = fwd(t, 8, x, "exact")
        out = []
        for m in ("f32res", "f16res"):
            g = fwd(t, 8, x, m)
            out.append(f"{m} {np.linalg.norm(g - ex) / np.linalg.norm(ex):.3e}")
        print(wn, inn, *out, flush=True)
