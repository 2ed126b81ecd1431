"""Training benchmark: trainer::fit_mlp through the drop-in library
(device FP64) vs the reference trainer on all host cores, same training set, config and seed;
the results are compared bit for bit.

    python tools/trainbench.py [--arch 256x3] [--n 100000] [--epochs 3] [--no-ref]
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
ap.add_argument("--arch", default="256x3")
ap.add_argument("--n", type=int, default=100000, help="n_uniform = n_surface")
ap.add_argument("--epochs", type=int, default=3)
ap.add_argument("--no-ref", action="store_true")
args = ap.parse_args()

from paper_2201_09147_b200 import train  # noqa: E402
from paper_2201_09147_b200.abi import TrainConfigC  # noqa: E402

torus = "torus:R=0.6,r=0.3"
pts, tg, vp, vt = train.sample_training_set(torus, args.n, args.n, 0.01, 10000, seed=1)
cfg = TrainConfigC(epochs=args.epochs, batch_size=8192, learning_rate=0.3, warmup_epochs=100)
train.fit_mlp("16x1", pts[:, :5000], tg[:5000], vp, vt, TrainConfigC(epochs=1))  # warm-up
t0 = time.perf_counter()
pa, la, ra = train.fit_mlp(args.arch, pts, tg, vp, vt, cfg, seed=7)
gpu_s = time.perf_counter() - t0
w, k = (int(x) for x in args.arch.split("x"))
macs = 3 * w + k * w * w + w
flop_epoch = pts.shape[1] * 2 * macs * 3 + pts.shape[1] * 2 * macs  # fwd + 2x bwd per minibatch, + full-batch loss
line = {"workload": f"fit_mlp({args.arch}, {2 * args.n} points torus, {args.epochs} epochs, batch 8192)",
        "gpu_s": gpu_s, "gpu_s_per_epoch": gpu_s / args.epochs,
        "gpu_TFLOP_per_s_f64": flop_epoch * args.epochs / gpu_s / 1e12, "final_loss": ra.final_loss}
if not args.no_ref:
    from oracle import refshim
    refshim.set_backend("avx2")
    t0 = time.perf_counter()
    pb, lb, rb = refshim.fit_mlp(args.arch, pts, tg, vp, vt, cfg, seed=7)
    line["ref_s"] = time.perf_counter() - t0
    line["ref_cores"] = refshim.worker_threads()
    line["speedup"] = line["ref_s"] / gpu_s
    line["identical"] = bool(np.array_equal(pa.view(np.uint64), pb.view(np.uint64)) and
                             np.array_equal(la.view(np.uint64), lb.view(np.uint64)))
print(json.dumps(line))
