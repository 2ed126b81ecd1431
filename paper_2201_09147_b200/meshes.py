"""Deterministic meshes for the mesh G-buffer workload (BASELINE config 4): the reference
has no rasterizer (SURVEY.md §7 hard part 9), so the G-buffer is the nearest-hit ray cast
of a fixed triangle mesh (nsdf_cuda_raycast_mesh)."""
import numpy as np


def torus_mesh(R=0.6, r=0.3, nu=96, nv=48):
    """Parametric torus around the y axis (TorusField convention), nu x nv quads."""
    u = np.arange(nu) * 2 * np.pi / nu
    v = np.arange(nv) * 2 * np.pi / nv
    uu, vv = np.meshgrid(u, v, indexing="ij")
    verts = np.stack([(R + r * np.cos(vv)) * np.cos(uu), r * np.sin(vv), (R + r * np.cos(vv)) * np.sin(uu)], -1)
    verts = verts.reshape(-1, 3)
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    a = i * nv + j
    b = ((i + 1) % nu) * nv + j
    c = ((i + 1) % nu) * nv + (j + 1) % nv
    d = i * nv + (j + 1) % nv
    tris = np.concatenate([np.stack([a, b, c], -1).reshape(-1, 3), np.stack([a, c, d], -1).reshape(-1, 3)])
    return verts.astype(np.float64), tris.astype(np.int32)
