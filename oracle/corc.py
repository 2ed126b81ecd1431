"""TEST INFRASTRUCTURE ONLY — ctypes bindings of oracle/_ref/libnsdf_oracle.so, the plain-C
restatement of the reference's float render path (oracle/nsdf_oracle.c)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import REF_DIR
from .pods import Camera, HitRecord, ShadeConfig, TraceConfig

_LIB = None
F = ctypes.POINTER(ctypes.c_float)


class OrcField(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("n_layers", ctypes.c_int), ("rows", ctypes.POINTER(ctypes.c_int32)),
                ("cols", ctypes.POINTER(ctypes.c_int32)), ("packed", ctypes.POINTER(ctypes.c_double)),
                ("activation", ctypes.c_int), ("omega0", ctypes.c_double), ("input_dim", ctypes.c_int),
                ("analytic", ctypes.c_double * 4)]


class OrcLevel(ctypes.Structure):
    _fields_ = [("field", OrcField), ("time", ctypes.c_float), ("delta", ctypes.c_double)]


def path():
    return os.path.join(REF_DIR, "libnsdf_oracle.so")


def load():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(path())
    return _LIB


class _Keep:
    """Keeps numpy buffers alive while ctypes structs point into them."""

    def __init__(self):
        self.bufs = []


def make_field(member, keep: _Keep) -> OrcField:
    from paper_2201_09147_b200.manifest import Analytic

    f = OrcField()
    if isinstance(member, Analytic):
        f.kind = {"sphere": 1, "torus": 2, "box": 3}[member.name]
        vals = member.values()
        for i, v in enumerate(vals):
            f.analytic[i] = v
        f.input_dim = 3
        return f
    rows = np.ascontiguousarray(member.rows, np.int32)
    cols = np.ascontiguousarray(member.cols, np.int32)
    packed = np.ascontiguousarray(member.packed, np.float64)
    keep.bufs += [rows, cols, packed]
    f.kind = 0
    f.n_layers = len(rows)
    f.rows = rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    f.cols = cols.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    f.packed = packed.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    f.activation = member.activation
    f.omega0 = member.omega0
    f.input_dim = member.input_dim
    return f


def make_levels(seq, time=0.0, keep=None):
    keep = keep or _Keep()
    arr = (OrcLevel * len(seq.members))()
    for i, m in enumerate(seq.members):
        arr[i].field = make_field(m, keep)
        arr[i].time = float(np.float32(time))
        arr[i].delta = seq.deltas[i]
    return arr, keep


def _chk(st):
    if st != 0:
        raise RuntimeError(f"oracle error {st}")


def sincos(x):
    lib = load()
    x = np.ascontiguousarray(x, np.float32)
    s = np.zeros_like(x)
    c = np.zeros_like(x)
    so, co = ctypes.c_float(), ctypes.c_float()
    for i, v in enumerate(x.reshape(-1)):
        lib.orc_sincos(ctypes.c_float(v), ctypes.byref(so), ctypes.byref(co))
        s.reshape(-1)[i] = so.value
        c.reshape(-1)[i] = co.value
    return s, c


def sine(x, omega, derivative):
    lib = load()
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros_like(x)
    lib.orc_sine(x.ctypes.data_as(F), out.ctypes.data_as(F), ctypes.c_int64(x.size), ctypes.c_float(omega),
                 int(derivative))
    return out


def mlp(net, points, mode, time=0.0):
    lib = load()
    keep = _Keep()
    f = make_field(net, keep)
    pts = np.ascontiguousarray(points, np.float32)
    rows, k = pts.shape
    d = np.zeros(k, np.float32)
    g = np.zeros((3, k), np.float32)
    _chk(lib.orc_mlp(ctypes.byref(f), mode, pts.ctypes.data_as(F), rows, k, ctypes.c_float(time), d.ctypes.data_as(F),
                     g.ctypes.data_as(F)))
    return d, g


def generate_rays(cam: Camera):
    lib = load()
    rays = np.zeros((cam.width * cam.height, 6), np.float32)
    lib.orc_generate_rays(ctypes.byref(cam), rays.ctypes.data_as(F))
    return rays


def trace_rays(seq, cfg: TraceConfig, rays, time=0.0):
    lib = load()
    lv, keep = make_levels(seq, time)
    r = np.ascontiguousarray(rays, np.float32).reshape(-1, 6)
    out = (HitRecord * max(len(r), 1))()
    _chk(lib.orc_trace_rays(lv, len(seq.members), ctypes.byref(cfg), r.ctypes.data_as(F), ctypes.c_int64(len(r)), out))
    return out


def normal_map(member, points, delta, fallback=None, time=0.0):
    lib = load()
    keep = _Keep()
    f = make_field(member, keep)
    pts = np.ascontiguousarray(points, np.float32)
    k = pts.shape[1]
    nrm = np.zeros((3, k), np.float32)
    fb = None if fallback is None else np.ascontiguousarray(fallback, np.float32)
    o, fc = ctypes.c_uint64(), ctypes.c_uint64()
    _chk(lib.orc_normal_map(ctypes.byref(f), ctypes.c_float(time), pts.ctypes.data_as(F), k, ctypes.c_double(delta),
                            fb.ctypes.data_as(F) if fb is not None else None, nrm.ctypes.data_as(F), ctypes.byref(o),
                            ctypes.byref(fc)))
    return nrm, o.value, fc.value


def shade(points, normals, cfg: ShadeConfig, cam: Camera):
    lib = load()
    pts = np.ascontiguousarray(points, np.float32)
    nrm = np.ascontiguousarray(normals, np.float32)
    k = pts.shape[1]
    rgb = np.zeros((3, k), np.float32)
    _chk(lib.orc_shade(pts.ctypes.data_as(F), nrm.ctypes.data_as(F), k, ctypes.byref(cfg), ctypes.byref(cam),
                       rgb.ctypes.data_as(F)))
    return rgb


def render(seq, cam: Camera, trace: TraceConfig, shade_cfg: ShadeConfig, normal_source=0, fine_index=-1, time=0.0,
           rows=None):
    """shading::render restated; `rows=(lo, hi)` renders only those image rows."""
    lib = load()
    lv, keep = make_levels(seq, time)
    lo, hi = rows if rows else (0, cam.height)
    n = cam.width * (hi - lo)
    rgb = np.zeros(3 * n, np.float32)
    depth = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    _chk(lib.orc_render_rows(lv, len(seq.members), ctypes.byref(cam), ctypes.byref(trace), ctypes.byref(shade_cfg),
                             normal_source, fine_index, lo, hi, rgb.ctypes.data_as(F), depth.ctypes.data_as(F),
                             mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
    return rgb.reshape(hi - lo, cam.width, 3), depth.reshape(hi - lo, cam.width), mask.reshape(hi - lo, cam.width)
