"""Quick GPU check of the tcgen05 fast modes against the FP32 oracle mode (debug aid)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from conftest import random_net
from paper_2201_09147_b200.engine import Context
from paper_2201_09147_b200.manifest import load_sdfnet

ctx = Context(0, "fp32")
modes = {m: Context(0, m) for m in ("fp16", "fp16low")}
nets = [("r64x1", random_net(64, 1, seed=3)), ("r128x2", random_net(128, 2, seed=4)), ("r256x3", random_net(256, 3, seed=5))]
for n in ["64x1", "128x2", "256x3"]:
    p = os.path.join(ROOT, f"assets/torus_w30_{n}.sdfnet")
    if os.path.exists(p):
        nets.append((n, load_sdfnet(p)))
rng = np.random.default_rng(0)
for name, net in nets:
    pts = rng.uniform(-1, 1, (3, 5000)).astype(np.float32)
    d0, g0 = ctx.eval_grad(ctx.upload(net), pts)
    for mname, c in modes.items():
        h1 = c.upload(net)
        t0 = time.time()
        d1 = c.eval(h1, pts)
        _, g1 = c.eval_grad(h1, pts)
        dt = time.time() - t0
        n0 = g0 / np.linalg.norm(g0, axis=0); n1 = g1 / np.linalg.norm(g1, axis=0)
        ang = np.degrees(np.arccos(np.clip((n0 * n1).sum(0), -1, 1)))
        print(f"{name:7s} {mname:8s}: |df| max {np.abs(d1-d0).max():.3e} p99 {np.percentile(np.abs(d1-d0),99):.3e}  "
              f"grad rel max {np.max(np.linalg.norm(g1-g0,axis=0)/np.linalg.norm(g0,axis=0)):.3e}  "
              f"normal deg max {ang.max():.3f} p99.9 {np.percentile(ang,99.9):.3f}  ({dt*1e3:.1f} ms)", flush=True)
