"""Convergence of the speed setting per fixture: 1080p renders (fast mode, device buffers)
at several budget tuples of a nested sequence — hit count, image MSE against the generous
(40,40,40) render (as `nsdf bench` reports MSE against its baseline row) and ms/frame.

    python tools/budget_scan.py assets/torus_w30.nest [more.nest ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera  # noqa: E402
from paper_2201_09147_b200.engine import Context, DeviceSequence  # noqa: E402
from paper_2201_09147_b200.manifest import load_manifest  # noqa: E402

BUDGETS = [tuple(int(x) for x in b.split(",")) for b in os.environ.get("NSDF_SCAN_BUDGETS", "20,5,5;20,10,10;40,20,20;40,40,40").split(";")]


def scan(path, w=1920, h=1080):
    seq = load_manifest(path)
    m = len(seq.members)
    c = Context(0, "fp16")
    s = torch.cuda.Stream()
    c.set_stream(s.cuda_stream)
    ds = DeviceSequence(c, seq)
    cam = standard_camera(w, h)
    n = w * h
    rgb, depth = torch.zeros(3 * n, device="cuda"), torch.zeros(n, device="cuda")
    mask = torch.zeros(n, dtype=torch.uint8, device="cuda")
    out = []
    imgs = {}
    for b in BUDGETS:
        b = tuple(b[:m]) if m <= 3 else b
        cfg = TraceConfig(b)
        with torch.cuda.stream(s):
            for _ in range(2):
                c.render_device(ds.levels(), cam, cfg, ShadeConfig(specular=0.3), rgb.data_ptr(), depth.data_ptr(),
                                mask.data_ptr())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            for _ in range(5):
                c.render_device(ds.levels(), cam, cfg, ShadeConfig(specular=0.3), rgb.data_ptr(), depth.data_ptr(),
                                mask.data_ptr())
            e1.record(s)
            torch.cuda.synchronize()
        imgs[b] = rgb.cpu().numpy().copy()
        out.append({"budgets": b, "hits": int(mask.sum().item()), "ms": e0.elapsed_time(e1) / 5})
    ref = imgs[out[-1]["budgets"]]
    for r in out:
        r["mse_vs_40"] = float(np.mean((imgs[r["budgets"]].astype(np.float64) - ref) ** 2))
        r["hits_vs_40"] = r["hits"] / max(out[-1]["hits"], 1)
    c.close()
    return {"manifest": path, "deltas": seq.deltas, "rows": out}


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps(scan(p)), flush=True)
