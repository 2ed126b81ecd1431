"""Certification benchmark: the drop-in library's verify_nesting /
estimate_sup_diff (neural fields on the device FP64 path) vs the reference's own functions
on all host cores, same manifest and seeds; plus the FP64 evaluator's raw throughput.

    python tools/certbench.py [--samples 1000000] [--sup 500000] [--no-ref]
Prints one JSON line.  The reference leg uses oracle/_ref (test infrastructure).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--samples", type=int, default=1000000)
ap.add_argument("--sup", type=int, default=500000, help="n_uniform = n_surface")
ap.add_argument("--no-ref", action="store_true")
args = ap.parse_args()

from paper_2201_09147_b200 import certify  # noqa: E402
from paper_2201_09147_b200.engine import Context  # noqa: E402
from paper_2201_09147_b200.manifest import load_sdfnet  # noqa: E402

man = os.path.join(ROOT, "assets", "torus_w30.nest")
net256 = "weights:" + os.path.join(ROOT, "assets", "torus_w30_256x3.sdfnet")
torus = "torus:R=0.6,r=0.3"
line = {"workload": f"verify_nesting(torus_w30.nest 64x1>128x2>256x3, {args.samples} samples, seed 7); "
                    f"estimate_sup_diff(256x3 vs analytic torus, {args.sup}+{args.sup} samples, seed 1)"}

# FP64 evaluator throughput (256x3, fwd and fwd+grad, 1M points)
ctx = Context(0, "fp32")
net = load_sdfnet(os.path.join(ROOT, "assets", "torus_w30_256x3.sdfnet"))
h = ctx.upload(net)
pts = np.random.default_rng(0).uniform(-1, 1, (3, 1 << 20))
for grad in (False, True):
    ctx.eval_f64(h, pts[:, :4096], want_grad=grad)
    t0 = time.perf_counter()
    ctx.eval_f64(h, pts, want_grad=grad)
    dt = time.perf_counter() - t0
    flop = 2 * (net.macs_normal() if grad else net.macs_forward()) * pts.shape[1]
    line["f64_eval_grad" if grad else "f64_eval"] = {"points": pts.shape[1], "s": dt, "Mpoints_per_s": pts.shape[1] / dt / 1e6,
                                                     "TFLOP_per_s_f64": flop / dt / 1e12,
                                                     "note": "host arrays in/out, H2D+D2H included"}
ctx.close()

certify.verify_nesting(man, samples=100000)  # warm-up (uploads, allocations)
t0 = time.perf_counter()
v = certify.verify_nesting(man, samples=args.samples, seed=7, max_recorded=1000)
line["gpu_verify_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
s = certify.sup_diff(net256, torus, n_uniform=args.sup, n_surface=args.sup, seed=1)
line["gpu_sup_s"] = time.perf_counter() - t0
line["verify"] = {k: v[k] for k in ("samples_total", "checked", "violation_count")}
line["sup"] = {"raw_max": s["raw_max"], "eps": s["eps"]}

if not args.no_ref:
    from oracle import refshim
    refshim.set_backend("avx2")
    t0 = time.perf_counter()
    vr = refshim.verify_nesting(man, samples=args.samples, seed=7, max_recorded=1000)
    line["ref_verify_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sr = refshim.sup_diff(net256, torus, n_uniform=args.sup, n_surface=args.sup, seed=1)
    line["ref_sup_s"] = time.perf_counter() - t0
    line["ref_cores"] = refshim.worker_threads()
    line["identical"] = bool(vr["checked"] == v["checked"] and vr["violation_count"] == v["violation_count"] and
                             sr["raw_max"] == s["raw_max"] and np.array_equal(sr["argmax"], s["argmax"]))
    line["speedup_verify"] = line["ref_verify_s"] / line["gpu_verify_s"]
    line["speedup_sup"] = line["ref_sup_s"] / line["gpu_sup_s"]
print(json.dumps(line))
