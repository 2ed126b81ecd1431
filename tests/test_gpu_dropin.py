"""GPU: the drop-in C++ library (include/nsdf/*.hpp re-implemented over the C ABI,
libnsdf_b200.so) against the reference, through the reference-shaped call chain
load_manifest -> shading::render / tracer::trace_image / mlp::forward_and_gradient_batch.
The C++ binary tests/cpp/test_dropin runs reference-suite cases on the device."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from conftest import ASSETS, ROOT, bits, records_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def host():
    os.environ["NSDF_MODE"] = "oracle"  # the library's process-wide context: bit-exact mode
    from paper_2201_09147_b200 import build
    build.build()
    from paper_2201_09147_b200.abi import HOST_LIB_PATH, load_library
    load_library()
    lib = ctypes.CDLL(HOST_LIB_PATH)
    lib.nsdf_host_last_error.restype = ctypes.c_char_p
    return lib


def _check(lib, st):
    assert st == 0, lib.nsdf_host_last_error().decode()


@pytest.mark.parametrize("mode", ["oracle", "fast"])
def test_cpp_dropin_suite(mode):
    from paper_2201_09147_b200 import build
    build.build()
    exe = os.path.join(ROOT, "tests", "cpp", "bin", "test_dropin")
    r = subprocess.run([exe], capture_output=True, text=True, env={**os.environ, "NSDF_MODE": mode}, timeout=300)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout + r.stderr


def test_render_through_cpp_api_bitexact(host, oracle_built):
    from oracle import refshim
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    path = os.path.join(ASSETS, "torus_w30.nest")
    cam = standard_camera(96, 64)
    shade = ShadeConfig(specular=0.3)
    for budgets, src in [((20, 5, 5), 0), ((40, 0, 0), 1)]:
        cfg = TraceConfig(budgets)
        n = cam.width * cam.height
        rgb = np.zeros(3 * n, np.float32)
        depth = np.zeros(n, np.float32)
        mask = np.zeros(n, np.uint8)
        F = ctypes.POINTER(ctypes.c_float)
        _check(host, host.nsdf_host_render_manifest(path.encode(), ctypes.c_double(0), ctypes.byref(cam),
                                                    ctypes.byref(cfg), ctypes.byref(shade), src, -1,
                                                    rgb.ctypes.data_as(F), depth.ctypes.data_as(F),
                                                    mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        rrgb, rdepth, rmask, _ = refshim.render(path, cam, cfg, shade, src)
        assert np.array_equal(mask, rmask.reshape(-1))
        assert np.array_equal(depth.view(np.uint32), rdepth.reshape(-1).view(np.uint32))
        assert np.max(np.abs(rgb - rrgb.reshape(-1))) <= 1e-6


def test_trace_image_through_cpp_api_bitexact(host, oracle_built, tmp_path):
    from oracle import refshim
    from paper_2201_09147_b200.abi import Camera, HitRecord, TraceConfig
    man = tmp_path / "c.nest"
    man.write_text('{"deltas": [0.1, 0.05], "fields": [{"analytic": "sphere", "params": {"r": 1.0}}, '
                   '{"analytic": "box", "params": {"hx": 0.6, "hy": 0.5, "hz": 0.55}}]}')
    cam = Camera((0.3, 0.2, 3), (0, 0, 0), (0, 1, 0), 45.0, 41, 37)
    for budgets in [(40, 40), (50, 0)]:
        cfg = TraceConfig(budgets)
        out = (HitRecord * (cam.width * cam.height))()
        _check(host, host.nsdf_host_trace_image_manifest(str(man).encode(), ctypes.c_double(0), ctypes.byref(cam),
                                                         ctypes.byref(cfg), out))
        want = refshim.trace_image(str(man), cam, cfg)
        a, b = records_np(out), records_np(want)
        for f in ("hit", "level", "iters"):
            assert np.array_equal(a[f], b[f]), f
        for f in ("point", "t", "fd"):
            assert np.array_equal(a[f].view(np.uint32), b[f].view(np.uint32)), f


def test_mlp_through_cpp_api_bitexact(host, oracle_built):
    from oracle import refshim
    from paper_2201_09147_b200.manifest import load_sdfnet
    path = os.path.join(ASSETS, "torus_w30_128x2.sdfnet")
    pts = np.random.default_rng(3).uniform(-1, 1, (3, 999)).astype(np.float32)
    d = np.zeros(999, np.float32)
    g = np.zeros((3, 999), np.float32)
    F = ctypes.POINTER(ctypes.c_float)
    _check(host, host.nsdf_host_forward_and_gradient(path.encode(), pts.ctypes.data_as(F), 999, d.ctypes.data_as(F),
                                                     g.ctypes.data_as(F)))
    rd, rg = refshim.mlp(load_sdfnet(path), pts, 2)
    assert np.array_equal(bits(d), bits(rd)) and np.array_equal(bits(g), bits(rg))
