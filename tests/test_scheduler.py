"""CPU, world_size 2 over gloo: the frame/tile scheduler's host logic — tile ownership
partitions the image exactly once, the weight broadcast reproduces the manifest, and the
packed-tile gather reassembles a frame bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ASSETS, ROOT


def test_tiles_partition_the_image():
    from paper_2201_09147_b200.scheduler import owned_pixels
    for (w, h, t, n) in [(1920, 1080, 64, 8), (37, 23, 8, 3), (5, 5, 64, 2), (100, 1, 7, 4)]:
        parts = [owned_pixels(w, h, t, r, n) for r in range(n)]
        allp = np.concatenate(parts)
        assert len(allp) == w * h and len(np.unique(allp)) == w * h


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, manifest, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_2201_09147_b200.scheduler import TileGather, broadcast_sequence, owned_pixels
    seq = broadcast_sequence(manifest if rank == 0 else None, world, rank, device="cpu")
    W, H, T = 50, 30, 8
    # each rank "renders" only its tiles: pixel value = a function of the pixel index
    rgb = torch.zeros(W * H * 3)
    depth = torch.zeros(W * H)
    mask = torch.zeros(W * H, dtype=torch.uint8)
    idx = torch.from_numpy(owned_pixels(W, H, T, rank, world))
    rgb.view(-1, 3)[idx] = torch.stack([idx.float(), idx.float() * 2, idx.float() * 3], 1)
    depth[idx] = idx.float() * 0.5
    mask[idx] = (idx % 3 == 0).to(torch.uint8)
    g = TileGather(W, H, T, rank, world, device="cpu")
    g(rgb, depth, mask)
    if rank == 0:
        all_idx = torch.arange(W * H).float()
        ok = bool(torch.equal(rgb.view(-1, 3)[:, 1], all_idx * 2) and torch.equal(depth, all_idx * 0.5) and
                  torch.equal(mask, (torch.arange(W * H) % 3 == 0).to(torch.uint8)))
        nets = [m for m in seq.members if hasattr(m, "packed")]
        out.put((ok, [float(n.packed.sum()) for n in nets], list(seq.deltas)))
    dist.destroy_process_group()


def test_gloo_world2_broadcast_and_gather():
    manifest = os.path.join(ASSETS, "torus_w30.nest")
    if not os.path.exists(manifest):
        pytest.skip("fixture missing")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, manifest, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, sums, deltas = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    from paper_2201_09147_b200.manifest import load_manifest
    seq = load_manifest(manifest)
    assert ok
    assert sums == [float(m.packed.sum()) for m in seq.members]
    assert deltas == list(seq.deltas)


class _ShmCtx:
    """Stand-in for engine.Context's shared-memory entry points on CPU: `alloc` is a POSIX
    shared-memory block, the 'IPC handle' its name, `ipc_open` attaches it in the peer
    process — so PeerFramebuffer's handle exchange, probe and verdict run unchanged."""

    def __init__(self, fail_open=False):
        from multiprocessing import shared_memory
        self._sm, self.fail_open, self.blocks = shared_memory, fail_open, {}

    def _addr(self, s):
        import ctypes
        a = ctypes.addressof(ctypes.c_char.from_buffer(s.buf))
        self.blocks[a] = s
        return a

    def alloc(self, n):
        return self._addr(self._sm.SharedMemory(create=True, size=n))

    def ipc_export(self, p):
        return self.blocks[p].name.encode().ljust(64, b"\0")

    def ipc_open(self, h):
        if self.fail_open:
            raise RuntimeError("peer mapping refused")
        return self._addr(self._sm.SharedMemory(name=h.rstrip(b"\0").decode()))

    def memcpy(self, dst, src, n):
        import ctypes
        ctypes.memmove(dst, src, n)

    def free(self, p):
        self.blocks.pop(p).unlink()

    def ipc_close(self, p):
        self.blocks.pop(p)


def _peer_worker(rank, world, port, fail, out):
    import ctypes
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_2201_09147_b200.scheduler import PeerFramebuffer, owned_pixels
    W, H, T = 50, 30, 8
    n = W * H
    pf = PeerFramebuffer(_ShmCtx(fail_open=fail and rank == 1), W, H, 2, rank, world)
    res = {"ok": pf.ok, "reason": pf.reason}
    if pf.ok:
        # each rank "renders" its tiles straight into rank 0's slot 1
        r, d, m = pf.ptrs(1)
        rgb = np.ctypeslib.as_array((ctypes.c_float * (3 * n)).from_address(r))
        depth = np.ctypeslib.as_array((ctypes.c_float * n).from_address(d))
        mask = np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(m))
        idx = owned_pixels(W, H, T, rank, world)
        rgb.reshape(-1, 3)[idx] = np.stack([idx, 2 * idx, 3 * idx], 1)
        depth[idx] = idx * 0.5
        mask[idx] = rank + 1
        dist.barrier()
        if rank == 0:
            hr, hd, hm = np.empty(3 * n, np.float32), np.empty(n, np.float32), np.empty(n, np.uint8)
            pf.to_host(1, hr.ctypes.data, hd.ctypes.data, hm.ctypes.data)
            a = np.arange(n)
            owner = np.empty(n, np.uint8)
            for q in range(world):
                owner[owned_pixels(W, H, T, q, world)] = q + 1
            res["frame"] = bool(np.array_equal(hr.reshape(-1, 3)[:, 2], 3.0 * a) and
                                np.array_equal(hd, a * 0.5) and np.array_equal(hm, owner))
        del rgb, depth, mask
        dist.barrier()
    if rank == 0:
        out.put(res)
    dist.barrier()
    pf.bases = []  # the shared blocks are released with the process
    dist.destroy_process_group()


@pytest.mark.parametrize("fail", [False, True])
def test_gloo_world2_peer_framebuffer(fail):
    """PeerFramebuffer over gloo: handles broadcast, probe verdict agreed by every rank, and
    (when mapping works) both ranks' tiles assembled in rank 0's slot; a rank that cannot map
    the ring makes every rank fall back (ok False with the reason)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, fail, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    if fail:
        assert not res["ok"] and res["reason"]
    else:
        assert res["ok"] and res["frame"], res


def test_owned_frames_partition_the_stream():
    from paper_2201_09147_b200.scheduler import owned_frames
    for world in (1, 2, 3, 8):
        parts = [owned_frames(120, r, world) for r in range(world)]
        assert sorted(sum(parts, [])) == list(range(120))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1


def _rate_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2201_09147_b200.scheduler import job_rate, owned_frames
    frames = owned_frames(7, rank, world)            # rank 0: 0,2,4,6; rank 1: 1,3,5
    ms = 10.0 * (rank + 1)                           # rank 1 is the slower one
    rate, job_ms = job_rate(1000.0 * len(frames), ms, world)
    out.put((rank, rate, job_ms))
    dist.destroy_process_group()


def test_gloo_world2_job_rate_is_max_over_ranks():
    """Frame-stream sharding accounting over gloo, world size 2: the job time is the slowest
    rank's, the units are every rank's frames (7 frames of 1000 units in 20 ms)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rate_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for _, rate, job_ms in got:
        assert job_ms == 20.0 and abs(rate - 7000.0 / 0.020) < 1e-6


def test_balanced_tile_owners_lpt():
    """Cost-balanced tile map (longest processing time first): every tile gets one rank in
    [0, world), the ranks' loads end within one tile's cost of each other, and the map is
    deterministic; tile_costs sums per-pixel work per row-major tile."""
    from paper_2201_09147_b200.scheduler import balanced_tile_owners, tile_costs
    rng = np.random.default_rng(5)
    costs = rng.gamma(0.5, 10.0, size=2040)
    for world in (2, 3, 8):
        owners = balanced_tile_owners(costs, world)
        assert owners.shape == costs.shape and owners.min() >= 0 and owners.max() < world
        loads = np.bincount(owners, weights=costs, minlength=world)
        assert loads.max() - loads.min() <= costs.max() + 1e-9
        static = np.bincount(np.arange(len(costs)) % world, weights=costs, minlength=world)
        assert loads.max() <= static.max() + 1e-9
        assert np.array_equal(owners, balanced_tile_owners(costs, world))
    W, H, T = 70, 33, 16
    iters = np.zeros((W * H, 8), np.uint16)
    iters[:, 0] = 2
    iters[5, 1] = 3
    hit = np.zeros(W * H, np.int32)
    hit[W * 20 + 40] = 1
    c = tile_costs(iters, hit, W, H, T, [64, 256], 256)
    assert c.shape == (5 * 3,)
    assert np.isclose(c.sum(), W * H * 2 * 47.0 + 3 * 997.0 + 4030.0)
    assert np.isclose(c[0], T * T * 2 * 47.0 + 3 * 997.0)
