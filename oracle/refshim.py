"""TEST INFRASTRUCTURE ONLY — ctypes bindings of oracle/_ref/libnsdf_ref.so (the reference
library compiled from /root/reference/proj/src plus oracle/ref_shim.cpp)."""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from . import REF_DIR
from .pods import HitRecord, Camera, TraceConfig, ShadeConfig

_LIB = None


def path() -> str:
    return os.path.join(REF_DIR, "libnsdf_ref.so")


def available() -> bool:
    return os.path.exists(path())


def load():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(path())
        lib.nsdf_ref_last_error.restype = ctypes.c_char_p
        lib.nsdf_ref_backend.restype = ctypes.c_char_p
        _LIB = lib
    return _LIB


def _check(lib, st):
    if st != 0:
        raise RuntimeError(f"reference error {st}: {lib.nsdf_ref_last_error().decode()}")


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


F = ctypes.c_float
D = ctypes.c_double
I32 = ctypes.c_int32
U8 = ctypes.c_uint8
U64 = ctypes.c_uint64


def set_backend(name="avx2"):
    lib = load()
    _check(lib, lib.nsdf_ref_set_backend(name.encode()))


def tensor_op(op, a, b=None, bias=None, m=0, n=0, k=0, omega=30.0, derivative=False):
    """tensor::gemm (op 0) / hadamard (1) / activate sine (2) / scale_rows (3) of the reference
    (nsdf_ref_tensor); arrays float32 or float64, row-major; returns the m x n result."""
    lib = load()
    dt = np.asarray(a).dtype
    a = np.ascontiguousarray(a, dt)
    b = None if b is None else np.ascontiguousarray(b, dt)
    bias = None if bias is None else np.ascontiguousarray(bias, dt)
    out = np.zeros((m, n), dt)
    vp = lambda x: None if x is None else x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(lib, lib.nsdf_ref_tensor(op, 1 if dt == np.float64 else 0, vp(a), vp(b), vp(bias), vp(out), m, n, k,
                                    D(omega), 1 if derivative else 0))
    return out


def worker_threads() -> int:
    return load().nsdf_ref_worker_threads()


def random_init(width, hidden, input_dim, omega0, seed):
    """mlp::random_init(Architecture{width, hidden, input_dim}, omega0, Rng(seed))."""
    lib = load()
    n_layers = hidden + 2
    n = width * input_dim + width + hidden * (width * width + width) + width + 1
    packed = np.zeros(n, np.float64)
    rows = np.zeros(n_layers, np.int32)
    cols = np.zeros(n_layers, np.int32)
    _check(lib, lib.nsdf_ref_random_init(width, hidden, input_dim, D(omega0), ctypes.c_uint64(seed),
                                         _p(packed, D), _p(rows, I32), _p(cols, I32)))
    return rows, cols, packed


def mlp(net, points, mode):
    """mode 0 forward_batch, 1 gradient_batch (spatial for 4-input), 2 fused — float path."""
    lib = load()
    pts = np.ascontiguousarray(points, np.float32)
    k = pts.shape[1]
    dist = np.zeros(k, np.float32)
    grad = np.zeros((3, k), np.float32)
    _check(lib, lib.nsdf_ref_mlp(mode, len(net.rows), _p(net.rows, I32), _p(net.cols, I32),
                                 _p(net.packed, D), net.activation, D(net.omega0), net.input_dim,
                                 _p(pts, F), k, _p(dist, F), _p(grad, F)))
    return dist, grad


def mlp_f64(net, points, mode):
    lib = load()
    pts = np.ascontiguousarray(points, np.float64)
    k = pts.shape[1]
    dist = np.zeros(k, np.float64)
    grad = np.zeros((3, k), np.float64)
    _check(lib, lib.nsdf_ref_mlp_f64(mode, len(net.rows), _p(net.rows, I32), _p(net.cols, I32),
                                     _p(net.packed, D), net.activation, D(net.omega0), net.input_dim,
                                     _p(pts, D), k, _p(dist, D), _p(grad, D)))
    return dist, grad


def save_params(lib, rows, cols, packed, activation, omega0, input_dim, path_):
    _check(lib, lib.nsdf_ref_save_params(len(rows), _p(np.ascontiguousarray(rows, np.int32), I32),
                                         _p(np.ascontiguousarray(cols, np.int32), I32),
                                         _p(np.ascontiguousarray(packed, np.float64), D),
                                         activation, D(omega0), input_dim, path_.encode()))


def certify(lib, weight_paths, labels, spec, out_manifest, n_uniform=200000, n_surface=200000,
            margin=1e-3, seed=1, verify=1000000):
    m = len(weight_paths)
    wp = (ctypes.c_char_p * m)(*[p.encode() for p in weight_paths])
    lb = (ctypes.c_char_p * m)(*[s.encode() for s in labels])
    eps = np.zeros(m, np.float64)
    deltas = np.zeros(m, np.float64)
    viol = ctypes.c_uint64(0)
    _check(lib, lib.nsdf_ref_certify(wp, lb, m, spec.encode(), U64(n_uniform), U64(n_surface), D(margin),
                                     U64(seed), U64(verify), out_manifest.encode(), _p(eps, D),
                                     _p(deltas, D), ctypes.byref(viol)))
    return eps, deltas, viol.value


def write_time_manifest(weight_paths, labels, out_manifest, lib=None, margin=1e-3, n=200000, seed=5):
    """Time-dependent .nest (manifest.cpp:72-86 schema): eps_i = sampled max |f_i - blend|
    over (p, t) with the reference's f64 forward, Prop-2 thresholds (nesting.cpp:31-40)."""
    from paper_2201_09147_b200.manifest import load_sdfnet

    rng = np.random.default_rng(seed)
    p = rng.uniform(-1, 1, size=(3, n))
    t = rng.uniform(0, 1, size=(1, n))
    x = np.concatenate([p, t], 0)
    s = np.hypot(p[0], p[2])
    target = (1 - t[0]) * (np.linalg.norm(p, axis=0) - 0.7) + t[0] * (np.hypot(s - 0.6, p[1]) - 0.3)
    eps = []
    for wp in weight_paths:
        net = load_sdfnet(wp)
        d, _ = mlp_f64(net, x, 0)
        eps.append(float(np.max(np.abs(d - target))) + margin)
    m = len(eps)
    deltas = [0.0] * m
    deltas[m - 1] = eps[m - 1] + eps[m - 2]
    for i in range(m - 1, 0, -1):
        deltas[i - 1] = deltas[i] + eps[i] + eps[i - 1]
    man = {
        "time_dependent": True,
        "deltas": deltas,
        "fields": [{"weights": os.path.basename(w), "label": l} for w, l in zip(weight_paths, labels)],
        "provenance": {"proposition": 2, "eps": eps, "margin": margin, "sampler_seed": seed,
                       "n_uniform": n, "n_surface": 0, "verify_samples": 0, "verify_violations": 0,
                       "note": "eps sampled over (p,t) in [-1,1]^3 x [0,1] against the blend oracle"},
    }
    with open(out_manifest, "w") as f:
        json.dump(man, f, indent=1)
    print("blend eps", eps, "deltas", deltas)


def generate_rays(cam: Camera):
    lib = load()
    rays = np.zeros((cam.width * cam.height, 6), np.float32)
    _check(lib, lib.nsdf_ref_generate_rays(ctypes.byref(cam), _p(rays, F)))
    return rays


def field_eval(manifest, index, points, time=0.0, grad=True):
    lib = load()
    pts = np.ascontiguousarray(points, np.float32)
    k = pts.shape[1]
    d = np.zeros(k, np.float32)
    g = np.zeros((3, k), np.float32)
    _check(lib, lib.nsdf_ref_field_eval(manifest.encode(), D(time), index, _p(pts, F), k, _p(d, F),
                                        _p(g, F) if grad else None))
    return d, g


def trace_image(manifest, cam: Camera, cfg: TraceConfig, time=0.0):
    lib = load()
    out = (HitRecord * (cam.width * cam.height))()
    _check(lib, lib.nsdf_ref_trace_image(manifest.encode(), D(time), ctypes.byref(cam), ctypes.byref(cfg), out))
    return out


def trace_rays(manifest, cfg: TraceConfig, rays, time=0.0):
    lib = load()
    r = np.ascontiguousarray(rays, np.float32)
    n = r.shape[0]
    out = (HitRecord * n)()
    _check(lib, lib.nsdf_ref_trace_rays(manifest.encode(), D(time), ctypes.byref(cfg), _p(r, F), n, out))
    return out


def sphere_trace(manifest, index, rays, delta, eps_stop, max_iters, t_max=10.0, time=0.0):
    lib = load()
    r = np.ascontiguousarray(rays, np.float32)
    n = r.shape[0]
    out = (HitRecord * n)()
    _check(lib, lib.nsdf_ref_sphere_trace(manifest.encode(), D(time), index, F(delta), F(eps_stop),
                                          max_iters, F(t_max), _p(r, F), n, out))
    return out


def normal_map(manifest, index, points, delta, fallback=None, time=0.0):
    lib = load()
    pts = np.ascontiguousarray(points, np.float32)
    k = pts.shape[1]
    nrm = np.zeros((3, k), np.float32)
    fb = None if fallback is None else np.ascontiguousarray(fallback, np.float32)
    o, f = U64(0), U64(0)
    _check(lib, lib.nsdf_ref_normal_map(manifest.encode(), D(time), index, _p(pts, F), k, D(delta),
                                        None if fb is None else _p(fb, F), _p(nrm, F), ctypes.byref(o),
                                        ctypes.byref(f)))
    return nrm, o.value, f.value


def map_normals_to_mesh(manifest, index, vertices, delta, normals=None, time=0.0):
    """shading::map_normals_to_mesh; returns (normals k x 3 or None, (mapped, violators,
    fallbacks))."""
    lib = load()
    v = np.ascontiguousarray(vertices, np.float64)
    k = v.shape[0]
    nin = None if normals is None else np.ascontiguousarray(normals, np.float64)
    out = np.zeros((k, 3), np.float64)
    counts = (U64 * 3)()
    has = ctypes.c_int(0)
    _check(lib, lib.nsdf_ref_map_normals_mesh(manifest.encode(), D(time), index, _p(v, D), k,
                                              None if nin is None else _p(nin, D), 0 if nin is None else 1,
                                              D(delta), _p(out, D), counts, ctypes.byref(has)))
    return (out if has.value else None), tuple(int(c) for c in counts)


_WRITE_IMAGE = r'''
import array, ctypes, sys
lib = ctypes.CDLL(sys.argv[1])
w, h = int(sys.argv[4]), int(sys.argv[5])
px = array.array("f")
with open(sys.argv[3], "rb") as f:
    px.frombytes(f.read())
buf = (ctypes.c_float * len(px)).from_buffer(px)
sys.exit(lib.nsdf_ref_write_image(sys.argv[2].encode(), w, h, buf))
'''


def write_image(path_, rgb_hw3):
    """shading::write_ppm / write_png by extension.  Runs in a child interpreter that never
    imports numpy: with numpy's bundled runtime libraries loaded, the reference library's
    std::ofstream crashes in this process (a libstdc++ symbol clash, test-side only)."""
    import subprocess
    import sys
    import tempfile
    rgb = np.ascontiguousarray(rgb_hw3, np.float32)
    with tempfile.NamedTemporaryFile(suffix=".f32", delete=False) as fh:
        fh.write(rgb.tobytes())
    try:
        r = subprocess.run([sys.executable, "-c", _WRITE_IMAGE, path(), str(path_), fh.name,
                            str(rgb.shape[1]), str(rgb.shape[0])], capture_output=True, text=True)
    finally:
        os.unlink(fh.name)
    if r.returncode != 0:
        raise RuntimeError(f"reference write_image failed ({r.returncode}): {r.stderr[-400:]}")


_TRAIN = r'''
import ctypes, sys
lib = ctypes.CDLL(sys.argv[1])
lib.nsdf_ref_last_error.restype = ctypes.c_char_p
a = sys.argv[2:]
D, U = ctypes.c_double, ctypes.c_uint64
st = lib.nsdf_ref_train(a[0].encode(), a[1].encode(), int(a[2]), a[3].encode(), D(float(a[4])), D(float(a[5])),
                        U(int(a[6])), U(int(a[7])), U(int(a[8])), D(float(a[9])), U(int(a[10])), U(int(a[11])),
                        U(int(a[12])), D(float(a[13])), a[14].encode(), a[15].encode())
if st:
    sys.stderr.write(lib.nsdf_ref_last_error().decode())
sys.exit(st)
'''


def train(out_dir, name, shape, archs, epochs, epochs_list, lr, omega0, seed, n_uniform, n_surface, sigma,
          sup_uniform, sup_surface, verify_samples, domain_half=1.0):
    """The reference CLI's train flow (fit_sequence(_4d) -> .sdfnet, .report.txt, .nest) in a
    child interpreter without numpy (see write_image).  Returns (status, message)."""
    import subprocess
    import sys
    args = [shape, archs, epochs, epochs_list, lr, omega0, seed, n_uniform, n_surface, sigma, sup_uniform,
            sup_surface, verify_samples, domain_half, out_dir, name]
    r = subprocess.run([sys.executable, "-c", _TRAIN, path(), *[str(x) for x in args]], capture_output=True,
                       text=True)
    return r.returncode, r.stderr[-2000:]


def shade(points, normals, cfg: ShadeConfig, cam: Camera):
    lib = load()
    pts = np.ascontiguousarray(points, np.float32)
    nrm = np.ascontiguousarray(normals, np.float32)
    k = pts.shape[1]
    rgb = np.zeros((3, k), np.float32)
    _check(lib, lib.nsdf_ref_shade(_p(pts, F), _p(nrm, F), k, ctypes.byref(cfg), ctypes.byref(cam), _p(rgb, F)))
    return rgb


def render(manifest, cam: Camera, trace: TraceConfig, shade_cfg: ShadeConfig, normal_source=0,
           fine_index=-1, time=0.0):
    """shading::render; returns (rgb HxWx3, depth HxW, mask HxW, seconds)."""
    lib = load()
    n = cam.width * cam.height
    rgb = np.zeros(3 * n, np.float32)
    depth = np.zeros(n, np.float32)
    mask = np.zeros(n, np.uint8)
    sec = D(0)
    _check(lib, lib.nsdf_ref_render(manifest.encode(), D(time), ctypes.byref(cam), ctypes.byref(trace),
                                    ctypes.byref(shade_cfg), normal_source, fine_index, _p(rgb, F),
                                    _p(depth, F), _p(mask, U8), ctypes.byref(sec)))
    return (rgb.reshape(cam.height, cam.width, 3), depth.reshape(cam.height, cam.width),
            mask.reshape(cam.height, cam.width), sec.value)


# ---- certification (nesting.cpp:131-361) -------------------------------------------------
def sample_near_surface(field_src, count, gaussian=False, amount=0.1, seed=1):
    lib = load()
    out = np.zeros((count, 3), np.float64)
    _check(lib, lib.nsdf_ref_sample_near_surface(field_src.encode(), U64(count), int(gaussian), D(amount),
                                                 U64(seed), _p(out, D)))
    return out


def sup_diff(f_src, g_src, n_uniform=20000, n_surface=20000, margin=1e-3, noise=0.1, seed=1):
    """{eps, raw_max, argmax (3,), samples} of fields::estimate_sup_diff."""
    lib = load()
    out = np.zeros(6, np.float64)
    _check(lib, lib.nsdf_ref_sup_diff(f_src.encode(), g_src.encode(), U64(n_uniform), U64(n_surface), D(margin),
                                      D(noise), U64(seed), _p(out, D)))
    return {"eps": out[0], "raw_max": out[1], "argmax": out[2:5].copy(), "samples": int(out[5])}


def verify_nesting(manifest, samples=100000, seed=7, max_recorded=1000, time=0.0):
    """{samples_total, checked, violation_count, violations (n, 6)} of fields::verify_nesting."""
    lib = load()
    counts = np.zeros(4, np.uint64)
    rec = np.zeros((max_recorded, 6), np.float64)
    _check(lib, lib.nsdf_ref_verify_nesting(manifest.encode(), D(time), U64(samples), U64(seed), U64(max_recorded),
                                            _p(counts, U64), _p(rec, D)))
    return {"samples_total": int(counts[0]), "checked": int(counts[1]), "violation_count": int(counts[2]),
            "violations": rec[:int(counts[3])].copy()}


# ---- training (trainer::sample_training_set / fit_mlp / backprop_sine_mlp) -------------------
def sample_training_set(oracle, n_uniform=100000, n_surface=100000, sigma=0.01, n_validation=10000, seed=1):
    lib = load()
    n = n_uniform + n_surface
    pts, tg = np.zeros((3, n)), np.zeros(n)
    vp, vt = np.zeros((3, n_validation)), np.zeros(n_validation)
    _check(lib, lib.nsdf_ref_sample_training_set(oracle.encode(), U64(n_uniform), U64(n_surface), D(sigma),
                                                 U64(n_validation), U64(seed), _p(pts, D), _p(tg, D), _p(vp, D),
                                                 _p(vt, D)))
    return pts, tg, vp, vt


def fit_mlp(arch, points, targets, val_points, val_targets, config, omega0=30.0, seed=7):
    from paper_2201_09147_b200.abi import TrainReportC
    from paper_2201_09147_b200.train import arch_params
    lib = load()
    input_dim = points.shape[0]
    params = np.zeros(arch_params(arch, input_dim))
    loss = np.zeros(config.epochs)
    rep = TrainReportC()
    pts, tg = np.ascontiguousarray(points, np.float64), np.ascontiguousarray(targets, np.float64)
    vp, vt = np.ascontiguousarray(val_points, np.float64), np.ascontiguousarray(val_targets, np.float64)
    _check(lib, lib.nsdf_ref_fit_mlp(arch.encode(), input_dim, D(omega0), U64(seed), ctypes.byref(config),
                                     _p(pts, D), _p(tg, D), pts.shape[1], _p(vp, D), _p(vt, D), vp.shape[1],
                                     _p(params, D), _p(loss, D), ctypes.byref(rep)))
    return params, loss[:rep.epochs_recorded].copy(), rep


def backprop(arch, points, targets, omega0=30.0, seed=7):
    from paper_2201_09147_b200.train import arch_params
    lib = load()
    input_dim = points.shape[0]
    params = np.zeros(arch_params(arch, input_dim))
    grads = np.zeros_like(params)
    loss = D(0)
    pts, tg = np.ascontiguousarray(points, np.float64), np.ascontiguousarray(targets, np.float64)
    _check(lib, lib.nsdf_ref_backprop(arch.encode(), input_dim, D(omega0), U64(seed), _p(pts, D), _p(tg, D),
                                      pts.shape[1], _p(params, D), _p(grads, D), ctypes.byref(loss)))
    return params, grads, loss.value
