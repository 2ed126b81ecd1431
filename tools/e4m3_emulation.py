"""Error of the split-precision variants of the fast mode's hidden layers, emulated on the
CPU (numpy + torch's float8_e4m3fn / float16 casts, float64 everywhere else) for a 256-wide
fixture near its surface (|f| < 0.05):

  1term   A_hi.W_hi                       (fp16 operands)
  2term   A_hi.W_hi + A_lo.W_hi
  e4m3    A_hi.W_hi + [fp8(A) | fp8(A_lo 2^11)] . [fp8(W_lo 2^11) ; fp8(W_hi)] / 2^11
          (the engine's E4M3 correction MMA, mlp_tc.cuh tc_split8)
  3term   A_hi.W_hi + A_lo.W_hi + A_hi.W_lo   (fp16 split)

    python tools/e4m3_emulation.py [torus3_256x3 torus_w30_256x3 ...]

Printed: |f - f64| p50 / p99 / p99.9 / max over the near-surface points (DESIGN.md,
Arithmetic modes: 4.8e-6 p99.9 for e4m3 on torus3_256x3, 9.1e-6 on torus_w30_256x3).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2201_09147_b200.manifest import load_sdfnet  # noqa: E402


def f16(x):
    return torch.from_numpy(x).to(torch.float16).to(torch.float64).numpy()


def f8(x):
    return torch.from_numpy(x).to(torch.float8_e4m3fn).to(torch.float64).numpy()


def evaluate(layers, omega, p, mode):
    h = np.sin(omega * (layers[0][0] @ p + layers[0][1][:, None]))
    for w, b in layers[1:-1]:
        wo = omega * w
        if mode == "f64":
            z = wo @ h
        else:
            a = h.astype(np.float32).astype(np.float64)
            wh, ah = f16(wo), f16(a)
            wl, al = f16(wo - wh), f16(a - ah)
            if mode == "1term":
                z = wh @ ah
            elif mode == "2term":
                z = wh @ ah + wh @ al
            elif mode == "3term":
                z = wh @ ah + wh @ al + wl @ ah
            else:
                s = 2.0 ** 11
                z = wh @ ah + (f8((wo - wh) * s) @ f8(a) + f8(wh) @ f8((a - ah) * s)) / s
        h = np.sin(z + omega * b[:, None])
    return (layers[-1][0] @ h + layers[-1][1][:, None])[0]


def main(names):
    for name in names:
        net = load_sdfnet(os.path.join(ROOT, "assets", name + ".sdfnet"))
        layers = list(net.layers())
        rng = np.random.default_rng(1)
        p = rng.uniform(-1.2, 1.2, (3, 400000))
        f = evaluate(layers, net.omega0, p, "f64")
        near = np.abs(f) < 0.05
        p, f = p[:, near][:, :20000], f[near][:20000]
        print(f"{name}: {p.shape[1]} near-surface points")
        for mode in ("1term", "2term", "e4m3", "3term"):
            d = np.abs(evaluate(layers, net.omega0, p, mode) - f)
            print(f"  {mode:6s} |df| p50 {np.median(d):.2e} p99 {np.percentile(d, 99):.2e} "
                  f"p99.9 {np.percentile(d, 99.9):.2e} max {d.max():.2e}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["torus3_256x3", "torus_w30_256x3"])
