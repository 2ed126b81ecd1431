"""Fixture generator: the nested SIREN sequences the parity tests and bench.py render.

The reference ships no weights (proj/assets/build_assets.sh only), so the
benchmark scenes are produced here, once, and committed under assets/:

  torus_w30.nest      64x1 > 128x2 > 256x3, omega0 = 30, torus R=0.6 r=0.3   (configs 1-3)
  blend4d_w30.nest    4-input 64x1 > 128x2, sphere r=0.7 -> torus blend       (config 5)

Fitting uses PyTorch on the CPU (Adam, plain MSE on exact SDF targets, the SIREN init of
mlp::random_init, mlp.cpp:63-88).  The nets are *inputs* to the render path: parity is
defined on identical weights, so the trainer is only a way to get realistic surfaces.
Certification is done by the REFERENCE library (oracle/_ref/libnsdf_ref.so):
estimate_sup_diff per member against the analytic shape, Prop-2 thresholds, empirical
verify_nesting, and save_params/save_manifest write the reference's own .sdfnet/.nest
formats (io.cpp:15-36, manifest.cpp:96-104) — exactly what fit_sequence does after
fitting (fit.cpp:262-298).

Usage:  python tools/make_fixtures.py [--steps N] [--only torus|blend]
"""
from __future__ import annotations

import argparse
import ctypes
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import refshim  # noqa: E402  (test infrastructure: the reference library)

R_MAJOR, R_MINOR, R_SPHERE = 0.6, 0.3, 0.7


def torus_sdf(p):
    s = torch.sqrt(p[:, 0] ** 2 + p[:, 2] ** 2)
    return torch.sqrt((s - R_MAJOR) ** 2 + p[:, 1] ** 2) - R_MINOR


def sphere_sdf(p):
    return torch.linalg.norm(p, dim=1) - R_SPHERE


def torus_surface(n, g):
    u = torch.rand(n, generator=g) * 2 * math.pi
    v = torch.rand(n, generator=g) * 2 * math.pi
    pts = torch.stack([(R_MAJOR + R_MINOR * torch.cos(v)) * torch.cos(u), R_MINOR * torch.sin(v),
                       (R_MAJOR + R_MINOR * torch.cos(v)) * torch.sin(u)], 1)
    nrm = torch.stack([torch.cos(v) * torch.cos(u), torch.sin(v), torch.cos(v) * torch.sin(u)], 1)
    return pts, nrm


def sphere_surface(n, g):
    d = torch.randn(n, 3, generator=g)
    d = d / torch.linalg.norm(d, dim=1, keepdim=True)
    return d * R_SPHERE, d


def sample(n, g, sdf_fn, surface_fn, t=None):
    """Uniform box [-1.2,1.2]^3, near-surface gaussian shells, and a sparse far field out to
    the standard camera (2,1.5,2) so the march through extrapolation stays sane."""
    nu, ns, nf = int(0.35 * n), int(0.45 * n), n - int(0.35 * n) - int(0.45 * n)
    pu = (torch.rand(nu, 3, generator=g) * 2 - 1) * 1.2
    ps, nrm = surface_fn(ns, g)
    sig = torch.where(torch.rand(ns, 1, generator=g) < 0.5, torch.tensor(0.01), torch.tensor(0.08))
    ps = ps + nrm * torch.randn(ns, 1, generator=g) * sig
    pf = (torch.rand(nf, 3, generator=g) * 2 - 1) * 3.5
    p = torch.cat([pu, ps, pf], 0)
    return p, sdf_fn(p)


class Siren(torch.nn.Module):
    def __init__(self, width, hidden, input_dim, omega0, seed, first_scale=1.0):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        dims = [input_dim] + [width] * (hidden + 1) + [1]
        self.omega0 = omega0
        self.layers = torch.nn.ModuleList()
        for i in range(len(dims) - 1):
            lin = torch.nn.Linear(dims[i], dims[i + 1])
            fan_in = dims[i]
            # mlp.cpp:71-74; coarse nets start the first layer at a lower frequency
            # (first_scale < 1) so a 64-wide sine net can fit a smooth SDF at omega0 = 30.
            bound = first_scale / fan_in if i == 0 else math.sqrt(6.0 / fan_in) / omega0
            with torch.no_grad():
                lin.weight.uniform_(-bound, bound, generator=g)
                bb = 1.0 / math.sqrt(fan_in)
                lin.bias.uniform_(-bb, bb, generator=g)
            self.layers.append(lin)

    def forward(self, x):
        for lin in self.layers[:-1]:
            x = torch.sin(self.omega0 * lin(x))
        return self.layers[-1](x)

    def packed(self):
        rows, cols, chunks = [], [], []
        for lin in self.layers:
            w = lin.weight.detach().double().numpy()
            rows.append(w.shape[0])
            cols.append(w.shape[1])
            chunks += [w.reshape(-1), lin.bias.detach().double().numpy()]
        return np.array(rows, np.int32), np.array(cols, np.int32), np.concatenate(chunks)


def fit(width, hidden, input_dim, omega0, steps, batch, seed, sdf_fn, surface_fn, lr=1e-4, first_scale=1.0):
    torch.manual_seed(seed)
    net = Siren(width, hidden, input_dim, omega0, seed, first_scale)
    opt = torch.optim.Adam(net.parameters(), lr=lr)
    sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, steps, eta_min=lr * 0.05)
    g = torch.Generator().manual_seed(seed + 1)
    t0 = time.time()
    for it in range(steps):
        if input_dim == 4:
            tt = torch.rand(batch, 1, generator=g)
            p, _ = sample(batch, g, sphere_sdf, sphere_surface if it % 2 == 0 else torus_surface)
            y = (1 - tt[:, 0]) * sphere_sdf(p) + tt[:, 0] * torus_sdf(p)  # BlendTimeField, field.cpp:242-244
            x = torch.cat([p, tt], 1)
        else:
            x, y = sample(batch, g, sdf_fn, surface_fn)
        loss = torch.mean((net(x)[:, 0] - y) ** 2)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        sched.step()
        if it % 500 == 0 or it == steps - 1:
            print(f"  {width}x{hidden} step {it} loss {loss.item():.3e} ({time.time() - t0:.0f}s)", flush=True)
    return net


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--only", default="")
    ap.add_argument("--threads", type=int, default=6)
    args = ap.parse_args()
    torch.set_num_threads(args.threads)
    out = os.path.join(ROOT, "assets")
    os.makedirs(out, exist_ok=True)
    ref = refshim.load()

    if args.only in ("", "torus"):
        names = []
        for i, (w, k, fs, sm) in enumerate([(64, 1, 0.7, 1.3), (128, 2, 0.5, 1.0), (256, 3, 1.0, 1.3)]):
            steps = int(args.steps * sm)
            net = fit(w, k, 3, 30.0, steps, args.batch, 31 + 1000 * i, torus_sdf, torus_surface, first_scale=fs)
            rows, cols, packed = net.packed()
            path = os.path.join(out, f"torus_w30_{w}x{k}.sdfnet")
            refshim.save_params(ref, rows, cols, packed, 0, 30.0, 3, path)
            names.append(path)
        eps, deltas, viol = refshim.certify(ref, names, [f"{w}x{k}" for w, k in [(64, 1), (128, 2), (256, 3)]],
                                            "torus:R=0.6,r=0.3", os.path.join(out, "torus_w30.nest"),
                                            n_uniform=200000, n_surface=200000, verify=1000000)
        print("torus eps", eps, "deltas", deltas, "violations", viol)

    if args.only in ("", "blend"):
        names = []
        for i, (w, k) in enumerate([(64, 1), (128, 2)]):
            net = fit(w, k, 4, 30.0, args.steps, args.batch, 51 + 1000 * i, None, None, first_scale=0.5)
            rows, cols, packed = net.packed()
            path = os.path.join(out, f"blend4d_w30_{w}x{k}.sdfnet")
            refshim.save_params(ref, rows, cols, packed, 0, 30.0, 4, path)
            names.append(path)
        refshim.write_time_manifest(names, [f"{w}x{k}" for w, k in [(64, 1), (128, 2)]],
                                    os.path.join(out, "blend4d_w30.nest"), ref)


if __name__ == "__main__":
    main()
