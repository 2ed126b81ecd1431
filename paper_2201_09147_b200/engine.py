"""Python-side mirror of the reference API over the C ABI (include/nsdf_cuda.h).

Names follow the reference (proj/include/nsdf): eval_batch / grad_batch,
forward_and_gradient_batch, generate_rays, multiscale_sphere_trace / trace_image,
neural_normal_map, shade, render.  Everything runs in libnsdf_cuda.so on the GPU; a
missing library or device raises NsdfError (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence as Seq

import numpy as np

from . import abi
from .abi import Camera, FrameStats, HitRecord, Level, NsdfError, ShadeConfig, TraceConfig, check
from .manifest import Analytic, Net, Sequence

_F = ctypes.POINTER(ctypes.c_float)
_I32 = ctypes.POINTER(ctypes.c_int32)
_D = ctypes.POINTER(ctypes.c_double)
_U8 = ctypes.POINTER(ctypes.c_uint8)


def _fp(a):
    return a.ctypes.data_as(_F)


class Context:
    """One nsdf_ctx: a device, a stream and the uploaded fields."""

    def __init__(self, device: int = 0, mode: str = "fp32"):
        self.lib = abi.load_library()
        self._ctx = ctypes.c_void_p()
        check(self.lib.nsdf_cuda_create(device, ctypes.byref(self._ctx)))
        self.device = device
        self.set_mode(mode)

    def close(self):
        if self._ctx:
            self.lib.nsdf_cuda_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_mode(self, mode: str):
        m = {"fp32": abi.MODE_FP32_ORACLE, "oracle": abi.MODE_FP32_ORACLE, "fp16": abi.MODE_FP16_FAST,
             "fast": abi.MODE_FP16_FAST, "fp16low": abi.MODE_FP16_LOW}[mode]
        check(self.lib.nsdf_cuda_set_mode(self._ctx, m))
        self.mode = mode

    def set_stream(self, stream_ptr: int):
        check(self.lib.nsdf_cuda_set_stream(self._ctx, ctypes.c_void_p(stream_ptr)))

    def synchronize(self):
        check(self.lib.nsdf_cuda_synchronize(self._ctx))

    def set_profiling(self, on: bool):
        check(self.lib.nsdf_cuda_set_profiling(self._ctx, int(bool(on))))

    # ---- device memory shared across processes (peer framebuffers) ------------------------
    def alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        check(self.lib.nsdf_cuda_alloc(self._ctx, ctypes.c_size_t(nbytes), ctypes.byref(p)))
        return int(p.value)

    def free(self, ptr: int):
        check(self.lib.nsdf_cuda_free(self._ctx, ctypes.c_void_p(ptr)))

    def ipc_export(self, ptr: int) -> bytes:
        h = (ctypes.c_uint8 * 64)()
        check(self.lib.nsdf_cuda_ipc_export(self._ctx, ctypes.c_void_p(ptr), h))
        return bytes(h)

    def ipc_open(self, handle: bytes) -> int:
        h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
        p = ctypes.c_void_p()
        check(self.lib.nsdf_cuda_ipc_open(self._ctx, h, ctypes.byref(p)))
        return int(p.value)

    def ipc_close(self, ptr: int):
        check(self.lib.nsdf_cuda_ipc_close(self._ctx, ctypes.c_void_p(ptr)))

    def memcpy(self, dst: int, src: int, nbytes: int):
        check(self.lib.nsdf_cuda_memcpy(self._ctx, ctypes.c_void_p(dst), ctypes.c_void_p(src),
                                        ctypes.c_size_t(nbytes)))

    def get_profile(self) -> "abi.Profile":
        p = abi.Profile()
        check(self.lib.nsdf_cuda_get_profile(self._ctx, ctypes.byref(p)))
        return p

    # ---- fields -------------------------------------------------------------------------
    def upload(self, member) -> int:
        h = ctypes.c_int32()
        if isinstance(member, Net):
            rows = np.ascontiguousarray(member.rows, np.int32)
            cols = np.ascontiguousarray(member.cols, np.int32)
            packed = np.ascontiguousarray(member.packed, np.float64)
            check(self.lib.nsdf_cuda_upload_mlp(self._ctx, len(rows), rows.ctypes.data_as(_I32),
                                                cols.ctypes.data_as(_I32), packed.ctypes.data_as(_D),
                                                member.activation, ctypes.c_double(member.omega0),
                                                member.input_dim, ctypes.byref(h)))
        elif isinstance(member, Analytic):
            kind = {"sphere": abi.FIELD_SPHERE, "torus": abi.FIELD_TORUS, "box": abi.FIELD_BOX}.get(member.name)
            if kind is None:
                raise NsdfError(abi.ERR_CONFIG, f"analytic field '{member.name}' is not available on the device")
            vals = np.asarray(member.values(), np.float64)
            check(self.lib.nsdf_cuda_upload_analytic(self._ctx, kind, vals.ctypes.data_as(_D), len(vals),
                                                     ctypes.byref(h)))
        else:
            raise NsdfError(abi.ERR_CONTRACT, f"cannot upload {type(member).__name__}")
        return h.value

    def release(self, handle: int):
        check(self.lib.nsdf_cuda_release(self._ctx, handle))

    def set_tile_owners(self, owners=None):
        """nsdf_cuda_set_tile_owners: explicit tile -> rank map for tile-sharded renders
        (None restores t % world)."""
        if owners is None:
            check(self.lib.nsdf_cuda_set_tile_owners(self._ctx, None, 0))
            return
        o = np.ascontiguousarray(owners, np.int32)
        check(self.lib.nsdf_cuda_set_tile_owners(self._ctx, o.ctypes.data_as(_I32), len(o)))

    def replicate(self, handle: int, dst: "Context") -> int:
        """nsdf_cuda_replicate_field: this context's field, copied device to device into
        `dst` (the multi-GPU weight broadcast); returns the handle in dst."""
        h = ctypes.c_int32()
        check(self.lib.nsdf_cuda_replicate_field(self._ctx, handle, dst._ctx, ctypes.byref(h)))
        return h.value

    def upload_sequence(self, seq: Sequence) -> "DeviceSequence":
        return DeviceSequence(self, seq)

    # ---- batch evaluation -----------------------------------------------------------------
    def eval_grad(self, handle: int, points, time: float = 0.0, want_value=True, want_grad=True):
        pts = np.ascontiguousarray(points, np.float32)
        if pts.ndim != 2:
            raise NsdfError(abi.ERR_CONTRACT, "points must be rows x k")
        rows, k = pts.shape
        out = np.zeros(k, np.float32) if want_value else None
        grad = np.zeros((3, k), np.float32) if want_grad else None
        check(self.lib.nsdf_cuda_eval_grad(self._ctx, handle, _fp(pts), rows, k, ctypes.c_float(time),
                                           _fp(out) if out is not None else None,
                                           _fp(grad) if grad is not None else None))
        return out, grad

    def eval(self, handle, points, time=0.0):
        return self.eval_grad(handle, points, time, True, False)[0]

    def grad(self, handle, points, time=0.0):
        return self.eval_grad(handle, points, time, False, True)[1]

    def eval_f64(self, handle: int, points, time: float = 0.0, want_value=True, want_grad=True):
        """FP64 batch (forward_batch / gradient_batch<double>, the certification path),
        bit-exact with the reference's double kernels."""
        pts = np.ascontiguousarray(points, np.float64)
        if pts.ndim != 2:
            raise NsdfError(abi.ERR_CONTRACT, "points must be rows x k")
        rows, k = pts.shape
        out = np.zeros(k, np.float64) if want_value else None
        grad = np.zeros((3, k), np.float64) if want_grad else None
        dp = ctypes.POINTER(ctypes.c_double)
        check(self.lib.nsdf_cuda_eval_f64(self._ctx, handle, pts.ctypes.data_as(dp), rows, k, ctypes.c_double(time),
                                          out.ctypes.data_as(dp) if out is not None else None,
                                          grad.ctypes.data_as(dp) if grad is not None else None))
        return out, grad

    def eval_grad_device(self, handle, d_points, rows, k, time, d_out, d_grad):
        check(self.lib.nsdf_cuda_eval_grad_device(self._ctx, handle, ctypes.c_void_p(d_points), rows, k,
                                                  ctypes.c_float(time), ctypes.c_void_p(d_out),
                                                  ctypes.c_void_p(d_grad)))

    # ---- the reference's dense kernel table (tensor::gemm / hadamard / activate / scale_rows)
    @staticmethod
    def _dt(x):
        x = np.asarray(x)
        if x.dtype not in (np.float32, np.float64):
            raise NsdfError(abi.ERR_CONTRACT, "tensor ops take float32 or float64 arrays")
        return x.dtype, (1 if x.dtype == np.float64 else 0)

    def tensor_gemm(self, a, b, bias=None):
        """c = a . b (+ bias column), bit-exact with the reference's AVX2 gemm."""
        dt, code = self._dt(a)
        a = np.ascontiguousarray(a, dt)
        b = np.ascontiguousarray(b, dt)
        m, k = a.shape
        n = b.shape[1]
        bias = None if bias is None else np.ascontiguousarray(bias, dt).reshape(-1)
        c = np.zeros((m, n), dt)
        vp = lambda x: None if x is None else x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        check(self.lib.nsdf_cuda_tensor_gemm(self._ctx, code, vp(a), vp(b), vp(bias), vp(c), m, n, k))
        return c

    def tensor_hadamard(self, a, b):
        dt, code = self._dt(a)
        a = np.ascontiguousarray(a, dt)
        b = np.ascontiguousarray(b, dt)
        out = np.zeros_like(a)
        check(self.lib.nsdf_cuda_tensor_hadamard(self._ctx, code, a.ctypes.data_as(ctypes.c_void_p),
                                                 b.ctypes.data_as(ctypes.c_void_p),
                                                 out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(a.size)))
        return out

    def tensor_scale_rows(self, col, m):
        dt, code = self._dt(m)
        col = np.ascontiguousarray(col, dt).reshape(-1)
        m = np.ascontiguousarray(m, dt)
        out = np.zeros_like(m)
        check(self.lib.nsdf_cuda_tensor_scale_rows(self._ctx, code, col.ctypes.data_as(ctypes.c_void_p),
                                                   m.ctypes.data_as(ctypes.c_void_p),
                                                   out.ctypes.data_as(ctypes.c_void_p), m.shape[0], m.shape[1]))
        return out

    def tensor_sine(self, x, omega, derivative=False):
        dt, code = self._dt(x)
        x = np.ascontiguousarray(x, dt)
        out = np.zeros_like(x)
        check(self.lib.nsdf_cuda_tensor_sine(self._ctx, code, x.ctypes.data_as(ctypes.c_void_p),
                                             out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(x.size),
                                             ctypes.c_double(omega), 1 if derivative else 0))
        return out

    # ---- tracing --------------------------------------------------------------------------
    def generate_rays(self, cam: Camera):
        rays = np.zeros((cam.width * cam.height, 6), np.float32)
        check(self.lib.nsdf_cuda_generate_rays(self._ctx, ctypes.byref(cam), _fp(rays)))
        return rays

    def trace_rays(self, levels, cfg: TraceConfig, rays):
        r = np.ascontiguousarray(rays, np.float32).reshape(-1, 6)
        out = (HitRecord * max(len(r), 1))()
        lv, m = _levels(levels)
        check(self.lib.nsdf_cuda_trace_rays(self._ctx, lv, m, ctypes.byref(cfg), _fp(r), len(r), out))
        return out

    def trace_image(self, levels, cam: Camera, cfg: TraceConfig):
        out = (HitRecord * (cam.width * cam.height))()
        st = FrameStats()
        lv, m = _levels(levels)
        check(self.lib.nsdf_cuda_trace_image(self._ctx, lv, m, ctypes.byref(cam), ctypes.byref(cfg), out,
                                             ctypes.byref(st)))
        return out, st

    # ---- normals / shading / render ---------------------------------------------------------
    def normal_map(self, handle, points, delta, fallback=None, time=0.0):
        pts = np.ascontiguousarray(points, np.float32)
        k = pts.shape[1]
        nrm = np.zeros((3, k), np.float32)
        fb = None if fallback is None else np.ascontiguousarray(fallback, np.float32)
        o, f = ctypes.c_uint64(), ctypes.c_uint64()
        check(self.lib.nsdf_cuda_normal_map(self._ctx, handle, ctypes.c_float(time), _fp(pts), k,
                                            ctypes.c_double(delta), _fp(fb) if fb is not None else None,
                                            _fp(nrm), ctypes.byref(o), ctypes.byref(f)))
        return nrm, o.value, f.value

    def map_normals_to_mesh(self, handle, vertices, delta, normals=None, time=0.0):
        """nsdf_cuda_map_normals_to_mesh (shading::map_normals_to_mesh, mesh.cpp:122-156):
        returns (normals k x 3 float64 or None when nothing was mapped and the mesh had none,
        (mapped, violators, fallbacks))."""
        v = np.ascontiguousarray(vertices, np.float64)
        k = v.shape[0]
        out = np.zeros((k, 3), np.float64) if normals is None else np.array(normals, np.float64, order="C")
        counts = (ctypes.c_uint64 * 3)()
        check(self.lib.nsdf_cuda_map_normals_to_mesh(self._ctx, handle, ctypes.c_float(time), v.ctypes.data_as(_D), k,
                                                     ctypes.c_double(delta), out.ctypes.data_as(_D), counts))
        c = tuple(int(x) for x in counts)
        if c[0] == 0:  # the reference replaces the mesh normals only if some vertex was mapped
            out = None if normals is None else np.asarray(normals, np.float64)
        return out, c

    def normal_map_device(self, handle, d_points: int, k: int, delta: float, d_normals: int, d_counts: int,
                          d_fallback: int = 0, time: float = 0.0):
        check(self.lib.nsdf_cuda_normal_map_device(self._ctx, handle, ctypes.c_float(time), ctypes.c_void_p(d_points),
                                                   k, ctypes.c_double(delta), ctypes.c_void_p(d_fallback or None),
                                                   ctypes.c_void_p(d_normals), ctypes.c_void_p(d_counts)))

    def raycast_mesh(self, cam: Camera, vertices, triangles, d_positions: int, d_mask: int):
        v = np.ascontiguousarray(vertices, np.float32)
        t = np.ascontiguousarray(triangles, np.int32)
        check(self.lib.nsdf_cuda_raycast_mesh(self._ctx, ctypes.byref(cam), _fp(v), len(v),
                                              t.ctypes.data_as(_I32), len(t), ctypes.c_void_p(d_positions),
                                              ctypes.c_void_p(d_mask)))

    def shade(self, points, normals, cfg: ShadeConfig, cam: Camera):
        pts = np.ascontiguousarray(points, np.float32)
        nrm = np.ascontiguousarray(normals, np.float32)
        k = pts.shape[1]
        rgb = np.zeros((3, k), np.float32)
        check(self.lib.nsdf_cuda_shade(self._ctx, _fp(pts), _fp(nrm), k, ctypes.byref(cfg), ctypes.byref(cam),
                                       _fp(rgb)))
        return rgb

    def render(self, levels, cam: Camera, trace: TraceConfig, shade: ShadeConfig, normal_source=0, fine_index=-1):
        n = cam.width * cam.height
        rgb = np.zeros(3 * n, np.float32)
        depth = np.zeros(n, np.float32)
        mask = np.zeros(n, np.uint8)
        st = FrameStats()
        lv, m = _levels(levels)
        check(self.lib.nsdf_cuda_render(self._ctx, lv, m, ctypes.byref(cam), ctypes.byref(trace),
                                        ctypes.byref(shade), normal_source, fine_index, _fp(rgb), _fp(depth),
                                        mask.ctypes.data_as(_U8), ctypes.byref(st)))
        return rgb.reshape(cam.height, cam.width, 3), depth.reshape(cam.height, cam.width), \
            mask.reshape(cam.height, cam.width), st

    def render_into(self, levels, cam: Camera, trace: TraceConfig, shade: ShadeConfig, h_rgb: int, h_depth: int,
                    h_mask: int, normal_source=0, fine_index=-1):
        """nsdf_cuda_render into caller-owned HOST buffers (raw pointers, e.g. pinned memory)."""
        lv, m = _levels(levels)
        check(self.lib.nsdf_cuda_render(self._ctx, lv, m, ctypes.byref(cam), ctypes.byref(trace), ctypes.byref(shade),
                                        normal_source, fine_index, ctypes.c_void_p(h_rgb), ctypes.c_void_p(h_depth),
                                        ctypes.c_void_p(h_mask), None))

    def render_device(self, levels, cam, trace, shade, d_rgb: int, d_depth: int, d_mask: int, normal_source=0,
                      fine_index=-1, tile_size=64, tile_rank=0, tile_world=1, stats: bool = False):
        """Device framebuffer (raw device pointers, e.g. torch tensor .data_ptr()); async."""
        lv, m = _levels(levels)
        st = FrameStats() if stats else None
        check(self.lib.nsdf_cuda_render_device(self._ctx, lv, m, ctypes.byref(cam), ctypes.byref(trace),
                                               ctypes.byref(shade), normal_source, fine_index, tile_size, tile_rank,
                                               tile_world, ctypes.c_void_p(d_rgb), ctypes.c_void_p(d_depth),
                                               ctypes.c_void_p(d_mask), ctypes.byref(st) if st else None))
        return st


def render_multi(contexts, level_lists, cam: Camera, trace: TraceConfig, shade: ShadeConfig, normal_source=0,
                 fine_index=-1, tile_size=32, stats: bool = False):
    """nsdf_cuda_render_multi: one frame over N contexts (N GPUs) from one process —
    context i renders the tiles t % N == i with its own field handles (level_lists[i]);
    returns the gathered host framebuffer (rgb, depth, mask[, FrameStats])."""
    n_ctx = len(contexts)
    if n_ctx < 1 or len(level_lists) != n_ctx:
        raise NsdfError(abi.ERR_CONTRACT, "one level list per context is required")
    lib = contexts[0].lib
    n = cam.width * cam.height
    rgb = np.zeros(3 * n, np.float32)
    depth = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    arrays = [_levels(lv) for lv in level_lists]
    m = arrays[0][1]
    ctxs = (ctypes.c_void_p * n_ctx)(*[c._ctx.value for c in contexts])
    lvp = (ctypes.POINTER(Level) * n_ctx)(*[ctypes.cast(a, ctypes.POINTER(Level)) for a, _ in arrays])
    st = FrameStats() if stats else None
    check(lib.nsdf_cuda_render_multi(ctxs, n_ctx, lvp, m, ctypes.byref(cam), ctypes.byref(trace), ctypes.byref(shade),
                                     normal_source, fine_index, tile_size, _fp(rgb), _fp(depth),
                                     mask.ctypes.data_as(_U8), ctypes.byref(st) if st else None))
    out = rgb.reshape(cam.height, cam.width, 3), depth.reshape(cam.height, cam.width), mask.reshape(cam.height, cam.width)
    return (*out, st) if stats else out


def _levels(levels):
    arr = (Level * len(levels))()
    for i, lv in enumerate(levels):
        arr[i] = lv
    return arr, len(levels)


class DeviceSequence:
    """A NestedSequence / AnimatedSequence resident on the device (weights uploaded once)."""

    def __init__(self, ctx: Context, seq: Sequence, handles=None):
        self.ctx = ctx
        self.seq = seq
        self.handles = list(handles) if handles is not None else [ctx.upload(m) for m in seq.members]

    def replicate(self, dst: Context) -> "DeviceSequence":
        """The same sequence on another context (device-to-device weight copies)."""
        return DeviceSequence(dst, self.seq, [self.ctx.replicate(h, dst) for h in self.handles])

    def levels(self, time: float = 0.0, indices: Optional[Seq[int]] = None):
        """nsdf_level array; for animated sequences `time` is the slice (float(t),
        field.cpp:303-305)."""
        idx = range(len(self.handles)) if indices is None else indices
        return [Level(self.handles[i], float(np.float32(time)), float(self.seq.deltas[i])) for i in idx]
