"""Frame/tile scheduler across the GPUs of one node (north_star subsystem 5).

One process per GPU (torchrun), torch.distributed for the plumbing.  The only collectives
are the ones the north star names:
  * broadcast_sequence: rank 0 reads the .nest/.sdfnet files and broadcasts the packed
    weights once (one NCCL broadcast of a float64 buffer + the small metadata);
  * TileGather: every rank renders the image tiles t with t % world == rank
    (nsdf_cuda_render_device) and rank 0 gathers the packed tile pixels (one NCCL gather).
Per-ray work is independent and partition-invariant (trace.hpp:69-70), so the
gathered frame is identical to a single-GPU render.  The host logic here is covered on
the CPU with gloo (tests/test_scheduler.py).
"""
from __future__ import annotations

from typing import Optional

import numpy as np


def owned_pixels(width: int, height: int, tile: int, rank: int, world: int) -> np.ndarray:
    """Row-major pixel indices of the tiles this rank owns (tile index row-major)."""
    tiles_x = (width + tile - 1) // tile
    ys, xs = np.divmod(np.arange(width * height, dtype=np.int64), width)
    t = (ys // tile) * tiles_x + xs // tile
    return np.nonzero(t % world == rank)[0]


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
    """Packs this rank's tile pixels (rgb, depth, mask) and gathers them on rank 0."""

    def __init__(self, width: int, height: int, tile: int, rank: int, world: int, device=None):
        import torch

        self.rank, self.world = rank, world
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
        self.device = device
        self.idx = [torch.from_numpy(owned_pixels(width, height, tile, r, world)).to(device) for r in range(world)]
        self.n_max = max(int(i.numel()) for i in self.idx)
        self.send = torch.zeros((self.n_max, 5), dtype=torch.float32, device=device)
        self.recv = [torch.zeros_like(self.send) for _ in range(world)] if rank == 0 else None
        self.host = None

    def __call__(self, rgb, depth, mask):
        import torch.distributed as dist

        idx = self.idx[self.rank]
        n = idx.numel()
        self.send[:n, 0:3] = rgb.view(-1, 3)[idx]
        self.send[:n, 3] = depth[idx]
        self.send[:n, 4] = mask[idx].float()
        dist.gather(self.send, self.recv if self.rank == 0 else None, dst=0)
        if self.rank == 0:
            self.rgb, self.depth, self.mask = rgb, depth, mask
            for r in range(1, self.world):
                ir = self.idx[r]
                m = ir.numel()
                rgb.view(-1, 3)[ir] = self.recv[r][:m, 0:3]
                depth[ir] = self.recv[r][:m, 3]
                mask[ir] = self.recv[r][:m, 4].to(mask.dtype)

    def to_host(self):
        """D2H of the assembled frame on rank 0 (the e2e read-back)."""
        return self.rgb.cpu(), self.depth.cpu(), self.mask.cpu()
