"""Frame/tile scheduler across the GPUs of one node (north_star subsystem 5).

One process per GPU (torchrun), torch.distributed for the plumbing.  A stream of frames (an
animation, repeated views) shards whole frames — frame i on rank i % world (owned_frames),
no collective on the data path; the job's throughput is all ranks' units over the slowest
rank's time (job_rate: one MAX and one SUM all-reduce after the run).  A single frame is
split across the ranks instead, with only the collectives the north star names:
  * broadcast_sequence: rank 0 reads the .nest/.sdfnet files and broadcasts the packed
    weights once (one NCCL broadcast of a float64 buffer + the small metadata);
  * PeerFramebuffer (default): rank 0 owns a ring of framebuffers mapped into every rank
    (CUDA IPC); every rank renders the image tiles t with t % world == rank
    (nsdf_cuda_render_device) and its shading kernels store those pixels straight into rank
    0's framebuffer over NVLink — the gather is fused into the producing kernels; one 4-byte
    NCCL all-reduce per frame orders the frame's completion across the ranks;
  * TileGather (fallback when peer mapping is unavailable): rank 0 gathers the packed tile
    pixels with one NCCL gather.
Per-ray work is independent and partition-invariant (trace.hpp:69-70), so the
gathered frame is identical to a single-GPU render.  The host logic here is covered on
the CPU with gloo (tests/test_scheduler.py).
"""
from __future__ import annotations

from typing import Optional

import numpy as np


def owned_pixels(width: int, height: int, tile: int, rank: int, world: int, owners=None) -> np.ndarray:
    """Row-major pixel indices of the tiles this rank owns (tile index row-major): tile t is
    rank t % world's, or owners[t]'s with an explicit map (nsdf_cuda_set_tile_owners)."""
    tiles_x = (width + tile - 1) // tile
    ys, xs = np.divmod(np.arange(width * height, dtype=np.int64), width)
    t = (ys // tile) * tiles_x + xs // tile
    return np.nonzero((t % world if owners is None else np.asarray(owners)[t]) == rank)[0]


# Device time per evaluation of one ray at a level (picoseconds, B200, fast mode; bench.py
# per-kernel times of the config-2 frame): the weights of a tile's predicted cost.
EVAL_PS = {64: 47.0, 128: 187.0, 256: 997.0}
NORMAL_PS_PER_WIDTH = {64: 190.0, 128: 760.0, 256: 4030.0}


def tile_costs(iters: np.ndarray, hit: np.ndarray, width: int, height: int, tile: int, level_widths,
               normal_width: int) -> np.ndarray:
    """Predicted device time of every image tile (row-major) from a traced frame: per pixel,
    the evaluations it took at each level (HitRecord.iterations_used, W*H x levels) times the
    level's per-evaluation cost, plus the normal tile of a hit."""
    w = np.array([EVAL_PS.get(int(x), 1000.0 * (int(x) / 256.0) ** 2) for x in level_widths], np.float64)
    per_pixel = iters[:, :len(w)].astype(np.float64) @ w + hit.astype(np.float64) * NORMAL_PS_PER_WIDTH.get(
        int(normal_width), 4030.0)
    tiles_x = (width + tile - 1) // tile
    ys, xs = np.divmod(np.arange(width * height, dtype=np.int64), width)
    t = (ys // tile) * tiles_x + xs // tile
    n_tiles = tiles_x * ((height + tile - 1) // tile)
    return np.bincount(t, weights=per_pixel, minlength=n_tiles)


def balanced_tile_owners(costs: np.ndarray, world: int) -> np.ndarray:
    """Longest-processing-time assignment of tiles to ranks: tiles in decreasing predicted
    cost, each to the currently least-loaded rank (ties: lowest rank; equal costs keep the
    tile order) — the ranks' predicted loads end within one tile of each other."""
    import heapq
    order = np.argsort(-np.asarray(costs, np.float64), kind="stable")
    heap = [(0.0, r) for r in range(world)]
    owners = np.zeros(len(costs), np.int32)
    for t in order:
        load, r = heapq.heappop(heap)
        owners[t] = r
        heapq.heappush(heap, (load + float(costs[t]), r))
    return owners


def owned_frames(n_frames: int, rank: int, world: int) -> list:
    """Frame-stream sharding: frame i renders on rank i % world (nsdf_main.cpp:308-324 loops
    the frames in order; every frame is independent)."""
    return [i for i in range(n_frames) if i % world == rank]


def job_rate(units_per_rank: float, ms_rank: float, world: int, device=None) -> tuple:
    """Whole-job throughput of a sharded run: every rank processed `units_per_rank` units in
    `ms_rank` ms; the job time is the MAX over ranks (one all-reduce), the job's units the sum
    over ranks.  Returns (units/s over all ranks, job ms)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms_rank, units_per_rank], dtype=torch.float64, device=device or "cpu")
    if world > 1:
        mx = t[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        tot = t[1:].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        ms, units = float(mx.item()), float(tot.item())
    else:
        ms, units = float(t[0].item()), float(t[1].item())
    return units / (ms / 1e3), ms


def broadcast_sequence(manifest_path: Optional[str], world: int, rank: int, device=None):
    """Rank 0 loads the manifest and broadcasts the weights once; returns the Sequence."""
    from .manifest import Analytic, Net, Sequence, load_manifest

    if world == 1:
        return load_manifest(manifest_path)
    import torch
    import torch.distributed as dist

    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    meta = [None]
    blob = None
    if rank == 0:
        seq = load_manifest(manifest_path)
        members, chunks = [], []
        for m in seq.members:
            if isinstance(m, Analytic):
                members.append(("analytic", m.name, m.params))
            else:
                members.append(("net", m.rows.tolist(), m.cols.tolist(), m.activation, m.omega0, m.input_dim,
                                int(m.packed.size)))
                chunks.append(m.packed)
        total = int(sum(c.size for c in chunks))
        meta = [{"members": members, "deltas": seq.deltas, "labels": seq.labels, "td": seq.time_dependent,
                 "total": total, "prov": seq.provenance}]
        blob = torch.from_numpy(np.concatenate(chunks) if chunks else np.zeros(0)).to(device)
    dist.broadcast_object_list(meta, src=0)
    meta = meta[0]
    if rank != 0:
        blob = torch.empty(meta["total"], dtype=torch.float64, device=device)
    if meta["total"]:
        dist.broadcast(blob, src=0)
    host = blob.cpu().numpy()
    out, off = [], 0
    for m in meta["members"]:
        if m[0] == "analytic":
            out.append(Analytic(m[1], dict(m[2])))
        else:
            _, rows, cols, act, omega, idim, n = m
            out.append(Net(np.array(rows, np.int32), np.array(cols, np.int32), host[off:off + n].copy(), act, omega,
                           idim))
            off += n
    return Sequence(out, list(meta["deltas"]), list(meta["labels"]), meta["td"], manifest_path, meta["prov"])


class TileGather:
    """Packs this rank's tile pixels (rgb, depth, mask) and gathers them on rank 0.

    Per frame: one packing gather on every rank (a precomputed [n, 5] index into the flat
    rgb|depth|mask view), one NCCL gather, and on rank 0 one scatter per buffer for all
    remote ranks together (precomputed combined indices) — a handful of kernels, so rank 0's
    extra work does not grow with the world size."""

    def __init__(self, width: int, height: int, tile: int, rank: int, world: int, device=None, owners=None):
        import torch

        self.rank, self.world = rank, world
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        self.device = device
        idx = [torch.from_numpy(owned_pixels(width, height, tile, r, world, owners)) for r in range(world)]
        self.n = [int(i.numel()) for i in idx]
        self.n_max = max(self.n)
        self.idx = idx[rank].to(device)
        self.send = torch.zeros((self.n_max, 5), dtype=torch.float32, device=device)
        self.recv = None
        if rank == 0:
            self.recv_all = torch.zeros((world, self.n_max, 5), dtype=torch.float32, device=device)
            self.recv = list(self.recv_all.unbind(0))
            # rows of recv_all (flattened) holding remote pixels, and their pixel indices
            rows = [torch.arange(self.n[r]) + r * self.n_max for r in range(1, world)]
            self.remote_rows = torch.cat(rows).to(device) if rows else torch.zeros(0, dtype=torch.long, device=device)
            self.remote_pix = torch.cat(idx[1:]).to(device) if world > 1 else self.remote_rows
        self.host = None

    def __call__(self, rgb, depth, mask):
        import torch
        import torch.distributed as dist

        idx = self.idx
        n = idx.numel()
        self.send[:n] = torch.cat([rgb.view(-1, 3)[idx], depth[idx].unsqueeze(1), mask[idx].unsqueeze(1).float()], 1)
        dist.gather(self.send, self.recv if self.rank == 0 else None, dst=0)
        if self.rank == 0:
            self.rgb, self.depth, self.mask = rgb, depth, mask
            got = self.recv_all.view(-1, 5)[self.remote_rows]
            rgb.view(-1, 3)[self.remote_pix] = got[:, 0:3]
            depth[self.remote_pix] = got[:, 3]
            mask[self.remote_pix] = got[:, 4].to(mask.dtype)

    def to_host(self):
        """D2H of the assembled frame on rank 0 (the e2e read-back)."""
        return self.rgb.cpu(), self.depth.cpu(), self.mask.cpu()


class PeerFramebuffer:
    """A ring of framebuffers owned by rank 0 and mapped into every rank (CUDA IPC), so each
    rank's render kernels write their tiles' pixels directly into rank 0's memory (NVLink peer
    stores).  `ptrs(b)` = (rgb, depth, mask) device pointers of ring slot b in this process.
    `ok` is False (and the caller falls back to TileGather) unless every rank mapped the
    ring and a probe written by every rank reached rank 0."""

    def __init__(self, ctx, width: int, height: int, n_buffers: int, rank: int, world: int):
        import torch
        import torch.distributed as dist

        self.ctx, self.rank, self.world = ctx, rank, world
        n = width * height
        al = lambda b: (b + 255) // 256 * 256  # noqa: E731
        self.off = (0, al(12 * n), al(12 * n) + al(4 * n))
        self.size = self.off[2] + al(n)
        self.n = n
        self.bases, self.local = [], rank == 0
        handles = [None]
        err = ""
        try:
            if rank == 0:
                self.bases = [ctx.alloc(self.size) for _ in range(n_buffers)]
                handles = [[ctx.ipc_export(b) for b in self.bases]]
        except Exception as e:  # reported through the probe verdict
            err = f"rank 0: {e}"
        dist.broadcast_object_list(handles, src=0)
        try:
            if rank != 0 and handles[0] is not None:
                self.bases = [ctx.ipc_open(h) for h in handles[0]]
        except Exception as e:
            err = f"rank {rank}: {e}"
        # probe: every rank writes its rank id into its own 16 bytes of slot 0's mask plane
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
        ok = torch.tensor([0 if err or not self.bases else 1], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        self.ok = bool(ok.item())
        if self.ok:
            marker = (np.full(16, rank + 1, np.uint8))
            self.ctx.memcpy(self.bases[0] + self.off[2] + 16 * rank, marker.ctypes.data, 16)
            dist.barrier()
            good = 1
            if rank == 0:
                got = np.zeros(16 * world, np.uint8)
                self.ctx.memcpy(got.ctypes.data, self.bases[0] + self.off[2], 16 * world)
                good = int(all((got[16 * r:16 * r + 16] == r + 1).all() for r in range(world)))
            ok = torch.tensor([good], dtype=torch.int32, device=ok.device)
            dist.broadcast(ok, src=0)
            self.ok = bool(ok.item())
        self.reason = err or ("" if self.ok else "peer probe failed")

    def ptrs(self, b: int):
        base = self.bases[b % len(self.bases)]
        return base + self.off[0], base + self.off[1], base + self.off[2]

    def to_host(self, b: int, rgb_h: int, depth_h: int, mask_h: int):
        """Rank 0: copy ring slot b into host buffers (raw pointers)."""
        r, d, m = self.ptrs(b)
        self.ctx.memcpy(rgb_h, r, 12 * self.n)
        self.ctx.memcpy(depth_h, d, 4 * self.n)
        self.ctx.memcpy(mask_h, m, self.n)

    def close(self):
        for b in self.bases:
            try:
                (self.ctx.free if self.local else self.ctx.ipc_close)(b)
            except Exception:
                pass
        self.bases = []


class PeerRing:
    """Frames in flight through a PeerFramebuffer ring of R slots (R = 2 x frames in flight).

    Frame i renders into slot i % R.  Completion token: after frame i's kernels (an event on
    its lane stream) a 4-byte all-reduce on ONE token stream, in frame order on every rank, so
    the collectives match across ranks whatever the lanes' progress; `done(i)` is the event
    after that all-reduce — on rank 0 it means every rank's stores of frame i have landed.
    Slot reuse: before frame i writes slot i % R (last used by frame i - R), its lane stream
    waits for the token of frame i - R + 1.  That token completes only after every rank issued
    its all-reduce for frame i - R + 1, and rank 0 issues it only after its host copy of frame
    i - R (the caller reads a finished slot synchronously before starting the next frame), so
    a slot is never overwritten while any rank still writes it or rank 0 still reads it."""

    def __init__(self, peer, n_slots: int):
        import torch

        self.peer = peer
        self.R = n_slots
        self.tok = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.stream = torch.cuda.Stream()
        self.events = [None] * n_slots

    def begin(self, i: int, lane_stream):
        """Slot pointers (rgb, depth, mask) for frame i, once the slot is free (stream order)."""
        prev = self.events[(i + 1) % self.R]
        if prev is not None:
            lane_stream.wait_event(prev)
        return self.peer.ptrs(i % self.R)

    def end(self, i: int, lane_stream):
        """Frame i's kernels are enqueued on lane_stream: enqueue its completion token."""
        import torch
        import torch.distributed as dist

        ev = torch.cuda.Event()
        ev.record(lane_stream)
        self.stream.wait_event(ev)
        with torch.cuda.stream(self.stream):
            dist.all_reduce(self.tok)
            done = torch.cuda.Event()
            done.record(self.stream)
        self.events[i % self.R] = done

    def done(self, i: int):
        return self.events[i % self.R]

