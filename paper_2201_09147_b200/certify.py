"""Certification on the B200 through the drop-in C++ library
(libnsdf_b200.so, include/nsdf_host.h): fields::sample_near_surface / estimate_sup_diff /
verify_nesting (nesting.cpp:131-361).  Neural fields evaluate on the device FP64 path
(mlp_f64.cu), bit-exact with the reference's double arithmetic; sampling and reductions run
on the host in the reference's order, so results equal the reference's for the same seeds.

A field source is "weights:<file.sdfnet>" or an analytic spec such as "torus:R=0.6,r=0.3".
"""
from __future__ import annotations

import ctypes

import numpy as np

from .abi import HOST_LIB_PATH, NsdfError

_LIB = None
D = ctypes.c_double
U64 = ctypes.c_uint64


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(HOST_LIB_PATH)
        lib.nsdf_host_last_error.restype = ctypes.c_char_p
        _LIB = lib
    return _LIB


def _check(st):
    if st != 0:
        raise NsdfError(st, _lib().nsdf_host_last_error().decode())


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def sample_near_surface(field_src: str, count: int, gaussian: bool = False, amount: float = 0.1,
                        seed: int = 1) -> np.ndarray:
    out = np.zeros((count, 3), np.float64)
    _check(_lib().nsdf_host_sample_near_surface(field_src.encode(), U64(count), int(gaussian), D(amount),
                                                U64(seed), _p(out, D)))
    return out


def sup_diff(f_src: str, g_src: str, n_uniform: int = 500000, n_surface: int = 500000, margin: float = 1e-3,
             noise: float = 0.1, seed: int = 1) -> dict:
    """fields::estimate_sup_diff(f, g): {eps, raw_max, argmax (3,), samples}."""
    out = np.zeros(6, np.float64)
    _check(_lib().nsdf_host_sup_diff(f_src.encode(), g_src.encode(), U64(n_uniform), U64(n_surface), D(margin),
                                     D(noise), U64(seed), _p(out, D)))
    return {"eps": out[0], "raw_max": out[1], "argmax": out[2:5].copy(), "samples": int(out[5])}


def verify_nesting(manifest: str, samples: int = 1000000, seed: int = 7, max_recorded: int = 100000,
                   time: float = 0.0) -> dict:
    """fields::verify_nesting(load_manifest(manifest)): {samples_total, checked,
    violation_count, violations (n, 6): x, y, z, pair, f_coarse, f_fine}."""
    counts = np.zeros(4, np.uint64)
    rec = np.zeros((max_recorded, 6), np.float64)
    _check(_lib().nsdf_host_verify_nesting(manifest.encode(), D(time), U64(samples), U64(seed), U64(max_recorded),
                                           _p(counts, U64), _p(rec, D)))
    return {"samples_total": int(counts[0]), "checked": int(counts[1]), "violation_count": int(counts[2]),
            "violations": rec[:int(counts[3])].copy()}
