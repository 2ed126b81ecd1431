"""Certification on the GPU vs the reference, bit for bit.

The device FP64 evaluator (nsdf_cuda_eval_f64, mlp_f64.cu) against the reference's
mlp::forward_batch / gradient_batch<double> (AVX2 double kernels); and the drop-in
library's fields::sample_near_surface / estimate_sup_diff / verify_nesting (which evaluate
neural fields on that device path) against the reference's own functions on the same
fields and seeds (nesting.cpp:131-361): identical sample sets, maxima, argmax, counts and
recorded violations."""
import json
import os
import tempfile

import numpy as np
import pytest

from conftest import ASSETS, random_net

pytestmark = pytest.mark.gpu

TORUS = "torus:R=0.6,r=0.3"


def _asset(name):
    p = os.path.join(ASSETS, name)
    if not os.path.exists(p):
        pytest.skip(f"fixture {name} not generated")
    return p


def _u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def ref(oracle_built):
    from oracle import refshim
    refshim.set_backend("avx2")
    return refshim


@pytest.mark.parametrize("width,hidden,input_dim", [(64, 1, 3), (128, 2, 3), (256, 3, 3), (64, 1, 4), (96, 2, 3)])
def test_f64_eval_bitexact_random(ctx, ref, width, hidden, input_dim):
    net = random_net(width, hidden, input_dim=input_dim, seed=7 + width)
    pts = np.random.default_rng(3).uniform(-1.1, 1.1, (input_dim, 3001))
    h = ctx.upload(net)
    d, g = ctx.eval_f64(h, pts)
    d0, _ = ref.mlp_f64(net, pts, 0)
    _, g0 = ref.mlp_f64(net, pts, 1)
    assert np.array_equal(_u64(d), _u64(d0))
    assert np.array_equal(_u64(g), _u64(g0))
    # forward-only call agrees with the fused one
    d1, _ = ctx.eval_f64(h, pts, want_grad=False)
    assert np.array_equal(_u64(d1), _u64(d))


@pytest.mark.parametrize("name", ["torus_w30_64x1", "torus_w30_128x2", "torus_w30_256x3"])
def test_f64_eval_bitexact_fixtures(ctx, ref, name):
    from paper_2201_09147_b200.manifest import load_sdfnet
    net = load_sdfnet(_asset(f"{name}.sdfnet"))
    pts = np.random.default_rng(5).uniform(-1, 1, (3, 4099))
    d, g = ctx.eval_f64(ctx.upload(net), pts)
    d0, _ = ref.mlp_f64(net, pts, 0)
    _, g0 = ref.mlp_f64(net, pts, 1)
    assert np.array_equal(_u64(d), _u64(d0)) and np.array_equal(_u64(g), _u64(g0))


def test_f64_eval_time_row(ctx, ref):
    """A 3-row batch for a 4-input net gets the constant double time row (field.cpp:213-220)."""
    net = random_net(64, 1, input_dim=4, seed=11)
    p3 = np.random.default_rng(9).uniform(-1, 1, (3, 777))
    t = 0.37
    d, g = ctx.eval_f64(ctx.upload(net), p3, time=t)
    p4 = np.concatenate([p3, np.full((1, 777), t)], 0)
    d0, _ = ref.mlp_f64(net, p4, 0)
    _, g0 = ref.mlp_f64(net, p4, 1)
    assert np.array_equal(_u64(d), _u64(d0)) and np.array_equal(_u64(g), _u64(g0))


@pytest.mark.parametrize("src", ["weights:torus_w30_64x1.sdfnet", TORUS])
@pytest.mark.parametrize("gaussian", [False, True])
def test_sample_near_surface(ref, src, gaussian):
    from paper_2201_09147_b200 import certify
    if src.startswith("weights:"):
        src = "weights:" + _asset(src[8:])
    a = certify.sample_near_surface(src, 6000, gaussian=gaussian, amount=0.05, seed=21)
    b = ref.sample_near_surface(src, 6000, gaussian=gaussian, amount=0.05, seed=21)
    assert np.array_equal(_u64(a), _u64(b))


@pytest.mark.parametrize("net", ["torus_w30_64x1", "torus_w30_256x3"])
def test_sup_diff_vs_analytic(ref, net):
    from paper_2201_09147_b200 import certify
    f = "weights:" + _asset(f"{net}.sdfnet")
    a = certify.sup_diff(f, TORUS, n_uniform=20000, n_surface=20000, seed=3)
    b = ref.sup_diff(f, TORUS, n_uniform=20000, n_surface=20000, seed=3)
    assert a["samples"] == b["samples"] == 40000
    assert np.array_equal(_u64([a["eps"], a["raw_max"]]), _u64([b["eps"], b["raw_max"]]))
    assert np.array_equal(_u64(a["argmax"]), _u64(b["argmax"]))


def test_sup_diff_neural_pair(ref):
    from paper_2201_09147_b200 import certify
    f = "weights:" + _asset("torus_w30_64x1.sdfnet")
    g = "weights:" + _asset("torus_w30_128x2.sdfnet")
    a = certify.sup_diff(f, g, n_uniform=5000, n_surface=5000, seed=9)
    b = ref.sup_diff(f, g, n_uniform=5000, n_surface=5000, seed=9)
    assert np.array_equal(_u64([a["raw_max"], *a["argmax"]]), _u64([b["raw_max"], *b["argmax"]]))


def _shrunk_manifest(path, scale):
    """The same sequence with the coarse deltas scaled (scale < 1 provokes violations: the
    fine neighborhood is no longer nested in the shrunken coarse one)."""
    j = json.load(open(path))
    base = os.path.dirname(path)
    for f in j["fields"]:
        if "weights" in f:
            f["weights"] = os.path.join(base, f["weights"])
    j["deltas"] = [d * scale for d in j["deltas"][:-1]] + j["deltas"][-1:]
    fd, out = tempfile.mkstemp(suffix=".nest")
    os.close(fd)
    json.dump(j, open(out, "w"))
    return out


@pytest.mark.parametrize("scale", [1.0, 0.1])
def test_verify_nesting(ref, scale):
    from paper_2201_09147_b200 import certify
    man = _shrunk_manifest(_asset("torus_w30.nest"), scale)
    try:
        a = certify.verify_nesting(man, samples=100000, seed=7, max_recorded=500)
        b = ref.verify_nesting(man, samples=100000, seed=7, max_recorded=500)
    finally:
        os.unlink(man)
    assert (a["samples_total"], a["checked"], a["violation_count"]) == \
        (b["samples_total"], b["checked"], b["violation_count"])
    assert np.array_equal(_u64(a["violations"]), _u64(b["violations"]))
    if scale == 1.0:
        assert a["violation_count"] == 0  # the fixture was certified with 0 violations
    else:
        assert a["violation_count"] > 0 and len(a["violations"]) > 0


def test_verify_nesting_time_slice(ref):
    from paper_2201_09147_b200 import certify
    man = _asset("blend4d_w30.nest")
    a = certify.verify_nesting(man, samples=100000, seed=3, max_recorded=200, time=0.37)
    b = ref.verify_nesting(man, samples=100000, seed=3, max_recorded=200, time=0.37)
    assert (a["checked"], a["violation_count"]) == (b["checked"], b["violation_count"])
    assert np.array_equal(_u64(a["violations"]), _u64(b["violations"]))


def test_certify_errors_match(ref):
    from paper_2201_09147_b200 import certify
    from paper_2201_09147_b200.abi import NsdfError
    with pytest.raises(NsdfError) as e:
        certify.sup_diff(TORUS, TORUS, n_uniform=100, n_surface=100)
    assert e.value.kind == "config" and "at least 1000 samples" in str(e.value)
    with pytest.raises(NsdfError) as e:
        certify.verify_nesting(_asset("torus_w30.nest"), samples=1000)
    assert e.value.kind == "contract" and "1e5" in str(e.value)
