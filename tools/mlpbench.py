"""Microbenchmark of the MLP tiles alone (eval op, contiguous points): evals/s per net/mode."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2201_09147_b200.engine import Context
from paper_2201_09147_b200.manifest import load_sdfnet

k = int(os.environ.get("K", 2_000_000))
pts = (torch.rand(3, k, device="cuda") * 2 - 1).contiguous()
out = torch.empty(k, device="cuda")
grad = torch.empty(3, k, device="cuda")
for mode in sys.argv[1:] or ["fp16", "fp16low", "fp32"]:
    ctx = Context(0, mode)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)
    for n in ["64x1", "128x2", "256x3"]:
        h = ctx.upload(load_sdfnet(os.path.join(ROOT, f"assets/torus_w30_{n}.sdfnet")))
        for g in (False, True):
            kk = k if not g else k // 4
            for _ in range(3):
                ctx.eval_grad_device(h, pts.data_ptr(), 3, kk, 0.0, out.data_ptr(), grad.data_ptr() if g else 0)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            for _ in range(10):
                ctx.eval_grad_device(h, pts.data_ptr(), 3, kk, 0.0, out.data_ptr(), grad.data_ptr() if g else 0)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            w = int(n.split("x")[0]); hid = int(n.split("x")[1])
            macs = 3 * w + hid * w * w + w
            if g:
                macs += 3 * (hid * w * w + 2 * w) + 3 * w
            sines = (hid + 1) * w
            mufu_bound_ms = kk * sines / (16 * 148 * 1.965e9) * 1e3 * (1 if not g else 1)
            print(f"{mode:8s} {n:6s} {'grad' if g else 'fwd ':4s}: {kk/ms/1e3:8.1f} Meval/s  {ms*1e3:8.1f} us  "
                  f"{2*macs*kk/ms/1e9:7.1f} TFLOP/s  MUFU-bound {mufu_bound_ms*1e3:7.1f} us", flush=True)
    ctx.close()
