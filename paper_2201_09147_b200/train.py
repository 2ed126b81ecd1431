"""SIREN training on the B200 through the drop-in C++ library:
trainer::sample_training_set (host, reference RNG order), trainer::fit_mlp and
backprop_sine_mlp (device FP64, bit-identical to the reference trainer)."""
from __future__ import annotations

import ctypes

import numpy as np

from .abi import TrainConfigC, TrainReportC
from .certify import _check, _lib, _p

D = ctypes.c_double
U64 = ctypes.c_uint64


def arch_params(arch: str, input_dim: int = 3) -> int:
    w, k = (int(x) for x in arch.lower().split("x"))
    return w * input_dim + w + k * (w * w + w) + w + 1


def sample_training_set(oracle: str, n_uniform=100000, n_surface=100000, sigma=0.01, n_validation=10000, seed=1):
    n = n_uniform + n_surface
    pts, tg = np.zeros((3, n)), np.zeros(n)
    vp, vt = np.zeros((3, n_validation)), np.zeros(n_validation)
    _check(_lib().nsdf_host_sample_training_set(oracle.encode(), U64(n_uniform), U64(n_surface), D(sigma),
                                                U64(n_validation), U64(seed), _p(pts, D), _p(tg, D), _p(vp, D),
                                                _p(vt, D)))
    return pts, tg, vp, vt


def fit_mlp(arch: str, points, targets, val_points, val_targets, config: TrainConfigC, omega0=30.0, seed=7):
    """trainer::fit_mlp: returns (packed params, epoch_loss, TrainReportC)."""
    input_dim = points.shape[0]
    params = np.zeros(arch_params(arch, input_dim))
    loss = np.zeros(config.epochs)
    rep = TrainReportC()
    pts, tg = np.ascontiguousarray(points, np.float64), np.ascontiguousarray(targets, np.float64)
    vp, vt = np.ascontiguousarray(val_points, np.float64), np.ascontiguousarray(val_targets, np.float64)
    _check(_lib().nsdf_host_fit_mlp(arch.encode(), input_dim, D(omega0), U64(seed), ctypes.byref(config), _p(pts, D),
                                    _p(tg, D), pts.shape[1], _p(vp, D), _p(vt, D), vp.shape[1], _p(params, D),
                                    _p(loss, D), ctypes.byref(rep)))
    return params, loss[:rep.epochs_recorded].copy(), rep


def backprop(arch: str, points, targets, omega0=30.0, seed=7):
    """trainer::backprop_sine_mlp on random_init(arch, omega0, Rng(seed)): (params, grads, loss)."""
    input_dim = points.shape[0]
    params = np.zeros(arch_params(arch, input_dim))
    grads = np.zeros_like(params)
    loss = D(0)
    pts, tg = np.ascontiguousarray(points, np.float64), np.ascontiguousarray(targets, np.float64)
    _check(_lib().nsdf_host_backprop(arch.encode(), input_dim, D(omega0), U64(seed), _p(pts, D), _p(tg, D),
                                     pts.shape[1], _p(params, D), _p(grads, D), ctypes.byref(loss)))
    return params, grads, loss.value
