"""Strong-scaling estimate of the tile scheduler on ONE GPU: for each world size N, every
rank's share of the frame (interleaved 32x32 tiles, tile t -> rank t % N) is rendered
alone, back to back, and the slowest rank's ms/frame is the N-GPU frame time without the
NCCL gather.  It does not emulate a multi-rank run (no rank waits on another); it measures
what each rank's GPU would have to do.

    python tools/shardsim.py [--config 2] [--inflight 5] [--tile 32] [--frames 30]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# frames in flight: pack short 256-wide level lists onto CTAs of >= 1536 rays (see bench.py)
os.environ.setdefault("NSDF_TC_MIN_ITEMS_256", "1536")

import torch

import bench
from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
from paper_2201_09147_b200.engine import Context, DeviceSequence
from paper_2201_09147_b200.manifest import load_manifest

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--inflight", type=int, default=5)
ap.add_argument("--frames", type=int, default=30)
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--tile", type=int, default=32)
ap.add_argument("--profile", action="store_true", help="per-level serial launch times of the slowest rank")
ap.add_argument("--balanced", action="store_true",
                help="cost-balanced tile owners (scheduler.balanced_tile_owners from one traced frame) instead of t % N")
args = ap.parse_args()

cfgw = bench.CONFIGS[args.config]
seq = load_manifest(cfgw["manifest"]).subsequence(cfgw["members"])
w, h = cfgw["res"]
npix = w * h
cam = standard_camera(w, h)
cfg = TraceConfig(tuple(int(b) for b in cfgw["budgets"].split(",")))
shade = ShadeConfig(specular=0.3)
src = 0 if cfgw["normals"] == "own" else 1
lanes = []
for _ in range(args.inflight):
    c = Context(0, "fp16")
    s = torch.cuda.Stream()
    c.set_stream(s.cuda_stream)
    d = DeviceSequence(c, seq)
    fb = (torch.zeros(npix * 3, device="cuda"), torch.zeros(npix, device="cuda"),
          torch.zeros(npix, dtype=torch.uint8, device="cuda"))
    lanes.append((c, s, d.levels(), fb))
main = lanes[0][1]


def run(rank, world, frames):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(main)
    for _, s, _, _ in lanes[1:]:
        s.wait_event(e0)
    for i in range(frames):
        c, s, lv, (r, d, m) = lanes[i % len(lanes)]
        c.render_device(lv, cam, cfg, shade, r.data_ptr(), d.data_ptr(), m.data_ptr(), src, -1, args.tile, rank, world)
    for _, s, _, _ in lanes[1:]:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / frames


costs = None
if args.balanced:
    from conftest_free_records import records_np  # noqa: E402  (tools-local copy of the HitRecord view)
    from paper_2201_09147_b200.scheduler import balanced_tile_owners, tile_costs  # noqa: E402
    rec = records_np(lanes[0][0].trace_image(lanes[0][2], cam, cfg)[0])
    costs = tile_costs(rec["iters"], rec["hit"], w, h, args.tile, [m.width for m in seq.members],
                       seq.members[-1].width if src == 0 else seq.members[-1].width)

base = None
for world in [int(x) for x in args.worlds.split(",")]:
    if costs is not None:
        owners = balanced_tile_owners(costs, world) if world > 1 else None
        for c, _, _, _ in lanes:
            c.set_tile_owners(owners)
    per = []
    for rank in range(world):
        run(rank, world, 3)
        per.append(run(rank, world, args.frames))
    t = max(per)
    if args.profile:
        c0 = lanes[0][0]
        c0.set_profiling(True)
        r, d, m = lanes[0][3]
        for _ in range(10):
            c0.render_device(lanes[0][2], cam, cfg, shade, r.data_ptr(), d.data_ptr(), m.data_ptr(), src, -1,
                             args.tile, per.index(t), world)
        torch.cuda.synchronize()
        p = c0.get_profile()
        c0.set_profiling(False)
        f = max(p.frames, 1)
        print(f"   serial: frame {p.frame_ms / f:.3f} ms, levels {[round(p.level_ms[j] / f, 3) for j in range(len(seq.members))]}"
              f", normals {p.normals_ms / f:.3f}, trace launches {p.trace_launches / f:.1f}, normal launches {p.normal_launches / f:.1f}")
    base = base or t
    print(f"config {args.config} N={world}: slowest rank {t:.3f} ms/frame (ranks {min(per):.3f}..{t:.3f}), "
          f"est. speed-up {base / t:.2f}x, {npix / t / 1e3:.0f} Mrays/s", flush=True)
for c, _, _, _ in lanes:
    c.close()
