"""CPU: framebuffer output (row f3).  The drop-in library's shading::write_ppm / write_png
(libnsdf_b200.so) must write the same BYTES as the reference's encoders (image.cpp:32-120)
for the same float framebuffer — including out-of-range values (clamped), exact half-steps
of the 8-bit quantisation (lround: half away from zero) and ragged sizes — and read_ppm
must invert write_ppm to 1/255."""
import ctypes

import numpy as np
import pytest


@pytest.fixture(scope="module")
def libs(oracle_built):
    from oracle import refshim
    from paper_2201_09147_b200 import build
    from paper_2201_09147_b200.certify import _lib
    if not refshim.available():
        pytest.skip("reference library not built")
    build.build_cuda()
    build.build_host()
    return _lib(), refshim


def _frames():
    rng = np.random.default_rng(12)
    yield rng.uniform(-0.2, 1.2, size=(37, 53, 3)).astype(np.float32)
    # exact quantisation boundaries: (k + 0.5) / 255 and their float neighbours
    k = np.arange(255, dtype=np.float32)
    half = (k + np.float32(0.5)) / np.float32(255.0)
    vals = np.concatenate([half, np.nextafter(half, 0), np.nextafter(half, 1), k / 255, [0, 1, -0.0, 2, -3]])
    n = len(vals) // 3 * 3
    yield vals[:n].astype(np.float32).reshape(1, n // 3, 3)
    yield np.zeros((1, 1, 3), np.float32)
    yield rng.uniform(0, 1, size=(270, 480, 3)).astype(np.float32)


@pytest.mark.parametrize("ext", [".ppm", ".png"])
def test_encoders_are_byte_identical(libs, tmp_path, ext):
    lib, ref = libs
    for i, img in enumerate(_frames()):
        ours, theirs = tmp_path / f"o{i}{ext}", tmp_path / f"r{i}{ext}"
        h, w, _ = img.shape
        st = lib.nsdf_host_write_image(str(ours).encode(), w, h, img.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
        assert st == 0, lib.nsdf_host_last_error()
        ref.write_image(theirs, img)
        assert ours.read_bytes() == theirs.read_bytes(), (i, ext)


def test_read_ppm_inverts_write(libs, tmp_path):
    lib, _ = libs
    img = next(_frames())
    p = tmp_path / "a.ppm"
    h, w, _ = img.shape
    assert lib.nsdf_host_write_image(str(p).encode(), w, h, img.ctypes.data_as(ctypes.POINTER(ctypes.c_float))) == 0
    out = np.zeros(img.size, np.float32)
    W, H = ctypes.c_int(), ctypes.c_int()
    assert lib.nsdf_host_read_ppm(str(p).encode(), ctypes.byref(W), ctypes.byref(H),
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), ctypes.c_size_t(out.size)) == 0
    assert (W.value, H.value) == (w, h)
    assert np.max(np.abs(out - np.clip(img.reshape(-1), 0, 1))) <= 0.5 / 255 + 1e-7
