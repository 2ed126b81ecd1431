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


def icosphere(subdivisions: int, radius: float):
    """Icosahedron subdivided on the unit sphere, vertices scaled by radius; also returns the
    unit normals.  The construction of the reference's test mesh (test_shading.cpp:74-112):
    the same vertex order (midpoints appended in face order, memoised per edge), so vertex i
    is the same point on both sides."""
    phi = (1.0 + np.sqrt(5.0)) / 2.0
    verts = [(-1, phi, 0), (1, phi, 0), (-1, -phi, 0), (1, -phi, 0), (0, -1, phi), (0, 1, phi), (0, -1, -phi),
             (0, 1, -phi), (phi, 0, -1), (phi, 0, 1), (-phi, 0, -1), (-phi, 0, 1)]

    def normalized(v):
        n = np.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
        return (v[0] / n, v[1] / n, v[2] / n) if n > 0 else (0.0, 0.0, 0.0)

    verts = [normalized(tuple(float(c) for c in v)) for v in verts]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
             (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        mid_of = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in mid_of:
                va, vb = verts[a], verts[b]
                verts.append(normalized(((va[0] + vb[0]) * 0.5, (va[1] + vb[1]) * 0.5, (va[2] + vb[2]) * 0.5)))
                mid_of[key] = len(verts) - 1
            return mid_of[key]

        nxt = []
        for f in faces:
            a, b, c = mid(f[0], f[1]), mid(f[1], f[2]), mid(f[2], f[0])
            nxt += [(f[0], a, c), (f[1], b, a), (f[2], c, b), (a, b, c)]
        faces = nxt
    n = np.array(verts, np.float64)
    return n * radius, np.array(faces, np.int32), n
