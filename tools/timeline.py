"""Per-tile timeline of CTA 0 of every tcgen05 launch of one config-2 frame (NSDF_TC_TIMELINE).

    NSDF_TC_TIMELINE_BUILD=1 python -c "from paper_2201_09147_b200 import build; build.build_cuda(force=True)"
    NSDF_TC_TIMELINE=1 [NSDF_TC_TIMELINE_SKIP=first_tile] [NSDF_TL_ASSET=torus3] [NSDF_TL_BUDGETS=40,20,20] \
        python tools/timeline.py [width height]
(the instrumentation is compiled out of the normal build: rebuild without the variable after)
Columns (SM cycles from the tile's start): A0 before its fence, A0 arrive | per MMA layer: the
accumulator-complete wait returning, the epilogue's end | (trace) return, update, flush ||
refill done, vote done, next tile's start.  Then, per tile, the MMA issuer's waits for A0,
for A block rows (kready) and for streamed weights, and its whole tile loop.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NSDF_TC_TIMELINE", "1")
import torch  # noqa: E402

from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera  # noqa: E402
from paper_2201_09147_b200.engine import Context, DeviceSequence  # noqa: E402
from paper_2201_09147_b200.manifest import load_manifest  # noqa: E402

w, h = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1920, 1080)
asset = os.environ.get("NSDF_TL_ASSET", "torus3")  # the headline scene (bench config 2)
budgets = tuple(int(b) for b in os.environ.get("NSDF_TL_BUDGETS", "40,20,20").split(","))
seq = load_manifest(os.path.join(ROOT, "assets", asset + ".nest"))
ctx = Context(0, "fp16")
ds = DeviceSequence(ctx, seq)
n = w * h
rgb, depth, mask = torch.zeros(3 * n, device="cuda"), torch.zeros(n, device="cuda"), torch.zeros(n, dtype=torch.uint8, device="cuda")
ctx.render_device(ds.levels(), standard_camera(w, h), TraceConfig(budgets), ShadeConfig(specular=0.3),
                  rgb.data_ptr(), depth.data_ptr(), mask.data_ptr(), 0)
torch.cuda.synchronize()
ctx.close()
