"""GPU: the N>1 frame assembly through peer stores (scheduler.PeerFramebuffer, bench.py's
default for tile-sharded frames).  Two processes on one GPU, host sync over gloo: rank 0
owns the framebuffer ring and exports it (CUDA IPC), rank 1 maps it and renders its tiles
straight into rank 0's memory, rank 0 renders its own tiles into the same slot.  The kernels
of the two ranks never wait on each other (each rank synchronizes its own stream, then a
host barrier).  The assembled slot must equal the single-process frame bit for bit."""
import os
import tempfile

import numpy as np
import pytest

from conftest import ASSETS, ROOT

pytestmark = pytest.mark.gpu

NEST = os.path.join(ASSETS, "torus_w30.nest")
W, H = 200, 120


def _render_args():
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    return standard_camera(W, H), TraceConfig((20, 5, 5)), ShadeConfig(specular=0.3)


def _worker(rank, world, port, mode, tile, out_path):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    from paper_2201_09147_b200.scheduler import PeerFramebuffer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = Context(0, mode)
    ds = DeviceSequence(ctx, load_manifest(NEST))
    cam, cfg, shade = _render_args()
    pf = PeerFramebuffer(ctx, W, H, 2, rank, world)
    assert pf.ok, pf.reason
    for slot in range(2):  # two frames through the ring
        ctx.render_device(ds.levels(), cam, cfg, shade, *pf.ptrs(slot), tile_size=tile, tile_rank=rank,
                          tile_world=world)
        ctx.synchronize()
    dist.barrier()
    if rank == 0:
        n = W * H
        res = []
        for slot in range(2):
            rgb = np.empty(3 * n, np.float32)
            depth = np.empty(n, np.float32)
            mask = np.empty(n, np.uint8)
            pf.to_host(slot, rgb.ctypes.data, depth.ctypes.data, mask.ctypes.data)
            res += [rgb, depth, mask]
        np.savez(out_path, *res)
    dist.barrier()
    pf.close()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
@pytest.mark.parametrize("tile", [32, 16])
def test_peer_framebuffer_assembles_the_frame(mode, tile):
    import torch.multiprocessing as mp
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    if not os.path.exists(NEST):
        pytest.skip("fixture missing")
    out = tempfile.mktemp(suffix=".npz")
    port = 29500 + (os.getpid() % 2000)
    mp.start_processes(_worker, args=(2, port, mode, tile, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    os.unlink(out)
    ctx = Context(0, mode)
    ref = ctx.render(DeviceSequence(ctx, load_manifest(NEST)).levels(), *_render_args())
    ctx.close()
    for slot in range(2):
        rgb, depth, mask = (got[f"arr_{3 * slot + i}"] for i in range(3))
        assert np.array_equal(mask, np.asarray(ref[2]).reshape(-1).astype(np.uint8))
        assert np.array_equal(depth.view(np.uint32), np.asarray(ref[1], np.float32).reshape(-1).view(np.uint32))
        assert np.array_equal(rgb.view(np.uint32), np.asarray(ref[0], np.float32).reshape(-1).view(np.uint32))


def _cam(i):
    """A different view per frame (orbiting camera), so a slot overwritten too early shows."""
    import math
    from paper_2201_09147_b200.abi import Camera
    a = 0.6 + 0.35 * i
    return Camera((2.6 * math.cos(a), 1.2 + 0.1 * i, 2.6 * math.sin(a)), (0, 0, 0), (0, 1, 0), 45.0, W, H)


def _ring_worker(rank, world, port, n_frames, out_path):
    import sys
    import time
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    from paper_2201_09147_b200.scheduler import PeerFramebuffer, PeerRing
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = Context(0, "fp16")
    lane = torch.cuda.Stream()
    ctx.set_stream(lane.cuda_stream)
    ds = DeviceSequence(ctx, load_manifest(NEST))
    pf = PeerFramebuffer(ctx, W, H, 2, rank, world)
    assert pf.ok, pf.reason
    ring = PeerRing(pf, 2)  # one frame in flight per rank: 2 slots, reused every other frame
    n = W * H
    frames = []
    for i in range(n_frames):
        ptrs = ring.begin(i, lane)
        ctx.render_device(ds.levels(), _cam(i), TraceConfig((20, 5, 5)), ShadeConfig(specular=0.3), *ptrs,
                          tile_size=16, tile_rank=rank, tile_world=world)
        ring.end(i, lane)
        if rank == 0:  # the e2e reader: frame i out of its slot as soon as its token completed
            ring.done(i).synchronize()
            time.sleep(0.05)  # a slow reader: rank 1 runs ahead and must wait for the slot
            rgb, depth, mask = np.empty(3 * n, np.float32), np.empty(n, np.float32), np.empty(n, np.uint8)
            pf.to_host(i % 2, rgb.ctypes.data, depth.ctypes.data, mask.ctypes.data)
            frames += [rgb, depth, mask]
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        np.savez(out_path, *frames)
    dist.barrier()
    pf.close()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_peer_ring_distinct_frames_through_reused_slots():
    """scheduler.PeerRing with a different camera per frame through more frames than slots
    (6 frames, 2 slots): rank 1 renders without host synchronisation of its own, rank 0 (a
    slow reader) reads every frame out of its slot after the frame's completion token; each
    read-back frame equals the single-process render of its own camera bit for bit.  On this
    one-GPU box the tokens go over gloo, whose all-reduce blocks the host, so rank 1 cannot get
    two frames ahead here and the slot-reuse edge (the ADVICE.md round-1 race) is not what
    keeps the frames apart; with NCCL's asynchronous tokens it is (PeerRing docstring)."""
    import torch.multiprocessing as mp
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    if not os.path.exists(NEST):
        pytest.skip("fixture missing")
    n_frames = 6
    out = tempfile.mktemp(suffix=".npz")
    port = 29500 + (os.getpid() % 2000) + 7
    mp.start_processes(_ring_worker, args=(2, port, n_frames, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    os.unlink(out)
    ctx = Context(0, "fp16")
    ds = DeviceSequence(ctx, load_manifest(NEST))
    try:
        for i in range(n_frames):
            ref = ctx.render(ds.levels(), _cam(i), TraceConfig((20, 5, 5)), ShadeConfig(specular=0.3))
            rgb, depth, mask = (got[f"arr_{3 * i + k}"] for k in range(3))
            assert np.array_equal(mask, np.asarray(ref[2]).reshape(-1).astype(np.uint8)), i
            assert np.array_equal(depth.view(np.uint32), np.asarray(ref[1], np.float32).reshape(-1).view(np.uint32)), i
            assert np.array_equal(rgb.view(np.uint32), np.asarray(ref[0], np.float32).reshape(-1).view(np.uint32)), i
    finally:
        ctx.close()


@pytest.mark.parametrize("shard", ["tiles", "frames", "animation"])
def test_bench_two_ranks_plumbing(shard):
    """bench.py's N > 1 path end to end (torchrun, 2 ranks, e2e to host) with both ranks on
    this one GPU over gloo (NSDF_BENCH_ONE_GPU=1): the JSON line carries the contract keys;
    tiles mode reports the peer assembly, frames mode the frame-sharded line plus the
    tile-sharded strong_scaling pass.  Plumbing only — not a measurement."""
    import json
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, NSDF_BENCH_ONE_GPU="1")
    env.pop("NSDF_MODE", None)  # conftest's oracle-mode default is not a bench --mode
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--no-alt"] +
                       (["--config", "5", "--width", "480", "--height", "270"] if shard == "animation"
                        else ["--shard", shard]),
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "e2e", "roofline", "clocks"):
        assert k in line
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    if shard == "animation":
        # config 5: the 120 frames round-robin over the ranks, e2e through the host-buffer API
        assert line["config"]["parallelism"] == "frames2" and line["steps"] == 60
        assert line["e2e"]["value"] > 0 and line["e2e"]["d2h_bytes_per_step"] == 480 * 270 * 17
    elif shard == "tiles":
        assert line["config"]["parallelism"] == "tiles2" and line["scaling"] == "strong"
        assert line["config"]["frame_assembly"].startswith("peer")
        assert line["strong_scaling"] is None
    else:
        assert line["config"]["parallelism"] == "frames2" and line["scaling"] == "weak"
        ss = line["strong_scaling"]
        assert ss["parallelism"] == "tiles2" and ss["value"] > 0 and ss["frame_assembly"].startswith("peer")
