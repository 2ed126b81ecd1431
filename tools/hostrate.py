"""Host enqueue rate of render_device frames vs their GPU time (is the frame launch-bound?).

    python tools/hostrate.py
"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
from paper_2201_09147_b200.engine import Context, DeviceSequence
from paper_2201_09147_b200.manifest import load_manifest
cfgw = bench.CONFIGS[2]
seq = load_manifest(cfgw["manifest"]).subsequence(cfgw["members"])
w, h = cfgw["res"]; npix = w * h
cam = standard_camera(w, h); cfg = TraceConfig((20, 5, 5)); shade = ShadeConfig(specular=0.3)
lanes = []
for _ in range(5):
    c = Context(0, "fp16"); s = torch.cuda.Stream(); c.set_stream(s.cuda_stream); d = DeviceSequence(c, seq)
    fb = (torch.zeros(npix * 3, device="cuda"), torch.zeros(npix, device="cuda"), torch.zeros(npix, dtype=torch.uint8, device="cuda"))
    lanes.append((c, s, d.levels(), fb))
for world in (1, 8):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(100):
            c, s, lv, (r, d, m) = lanes[i % 5]
            c.render_device(lv, cam, cfg, shade, r.data_ptr(), d.data_ptr(), m.data_ptr(), 0, -1, 32, 0, world)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"N={world}: host enqueue {1e3*(t1-t0)/100:.3f} ms/frame, wall {1e3*(t2-t0)/100:.3f} ms/frame")
