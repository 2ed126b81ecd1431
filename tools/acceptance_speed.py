"""The reference's acceptance criterion 7 (acceptance_main.cpp:295-333) on the B200: coarse
first is faster — fine@40 >= 4x coarse@40 and multiscale (30,30) faster than fine@60 — timed
with CUDA events over device-framebuffer renders (fast mode), at 256x256 and 1920x1080.

    python tools/acceptance_speed.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera  # noqa: E402
from paper_2201_09147_b200.engine import Context, DeviceSequence  # noqa: E402
from paper_2201_09147_b200.manifest import load_manifest  # noqa: E402


def time_render(ctx, levels, cam, budgets, reps=10):
    n = cam.width * cam.height
    rgb, depth = torch.zeros(3 * n, device="cuda"), torch.zeros(n, device="cuda")
    mask = torch.zeros(n, dtype=torch.uint8, device="cuda")
    cfg, shade = TraceConfig(budgets), ShadeConfig()
    for _ in range(2):
        ctx.render_device(levels, cam, cfg, shade, rgb.data_ptr(), depth.data_ptr(), mask.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        ctx.render_device(levels, cam, cfg, shade, rgb.data_ptr(), depth.data_ptr(), mask.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    seq = load_manifest(os.path.join(ROOT, "assets", "torus_w30.nest"))
    ctx = Context(0, "fp16")
    stream = torch.cuda.Stream()  # the engine's launch stream; the events are recorded on it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    coarse = DeviceSequence(ctx, seq.subsequence([0])).levels()
    fine = DeviceSequence(ctx, seq.subsequence([2])).levels()
    multi = DeviceSequence(ctx, seq.subsequence([0, 2])).levels()
    out = {}
    for w, h in ((256, 256), (1920, 1080)):
        cam = standard_camera(w, h)
        t = {k: time_render(ctx, lv, cam, b) for k, (lv, b) in
             {"coarse@40": (coarse, (40,)), "fine@40": (fine, (40,)), "multi(30,30)": (multi, (30, 30)),
              "fine@60": (fine, (60,))}.items()}
        ok = t["fine@40"] >= 4 * t["coarse@40"] and t["multi(30,30)"] < t["fine@60"]
        out[f"{w}x{h}"] = t
        print(f"{w}x{h}: " + ", ".join(f"{k} {v:.3f} ms" for k, v in t.items()) +
              f"; fine/coarse {t['fine@40'] / t['coarse@40']:.2f} (floor 4) -> {'PASS' if ok else 'FAIL'}", flush=True)
    ctx.close()
    return out


if __name__ == "__main__":
    main()
