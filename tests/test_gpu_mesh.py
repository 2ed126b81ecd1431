"""GPU: per-vertex mesh normal mapping, shading::map_normals_to_mesh (mesh.cpp:122-156),
through the C ABI (nsdf_cuda_map_normals_to_mesh) against the compiled reference on the same
meshes and fields: the reference's own cases (test_shading.cpp:215-261: icosphere against the
analytic sphere, a far torus that rejects every vertex, connectivity independence) plus the
fitted torus sequence on a torus mesh — counts exact, normals bitwise in the FP32 oracle mode
and within 0.5 degrees in the fast mode."""
import os

import numpy as np
import pytest

from conftest import ASSETS

pytestmark = pytest.mark.gpu


def _manifest(tmp_path, members, deltas):
    from paper_2201_09147_b200.manifest import Sequence, write_manifest
    seq = Sequence(list(members), list(deltas), [f"m{i}" for i in range(len(members))])
    path = os.path.join(str(tmp_path), "mesh.nest")
    write_manifest(seq, path, [None] * len(members))
    return path, seq


def _angle_deg(a, b):
    c = np.sum(a * b, 1) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1))
    return np.degrees(np.arccos(np.clip(c, -1.0, 1.0)))


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
def test_icosphere_against_analytic_sphere(oracle_built, tmp_path, mode):
    """test_shading.cpp:215-226: every vertex of the subdivided icosphere maps, with the
    sphere's exact normal (|n - v/|v|| < 1e-6), bit for bit with the reference."""
    from oracle import refshim
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import Analytic
    from paper_2201_09147_b200.meshes import icosphere
    path, seq = _manifest(tmp_path, [Analytic("sphere", {"r": 1.0})], [0.05])
    c = Context(0, mode)
    try:
        h = DeviceSequence(c, seq).handles[0]
        for sub, radius, delta, with_normals in [(2, 1.0, 0.05, True), (3, 1.02, 0.1, False), (1, 1.2, 0.1, True)]:
            v, _, n0 = icosphere(sub, radius)
            got, cnt = c.map_normals_to_mesh(h, v, delta, normals=n0 if with_normals else None)
            want, wcnt = refshim.map_normals_to_mesh(path, 0, v, delta, normals=n0 if with_normals else None)
            assert cnt == wcnt
            if radius == 1.2:  # outside the neighborhood: nothing mapped, normals untouched
                assert cnt == (0, len(v), 0) and np.array_equal(got, n0)
                continue
            assert cnt == (len(v), 0, 0)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
            assert np.max(np.linalg.norm(got - v / np.linalg.norm(v, axis=1, keepdims=True), axis=1)) < 1e-6
    finally:
        c.close()


def test_far_torus_rejects_every_vertex_and_connectivity_is_ignored(oracle_built, tmp_path):
    """test_shading.cpp:228-238 and 246-261: a small far torus leaves every normal untouched
    (all violators); reversing the triangle list changes nothing (vertices only)."""
    from oracle import refshim
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import Analytic
    from paper_2201_09147_b200.meshes import icosphere
    path, seq = _manifest(tmp_path, [Analytic("torus", {"R": 0.2, "r": 0.05})], [0.01])
    c = Context(0, "fp32")
    try:
        h = DeviceSequence(c, seq).handles[0]
        v, tris, n0 = icosphere(1, 1.0)
        got, cnt = c.map_normals_to_mesh(h, v, 0.01, normals=n0)
        assert cnt == refshim.map_normals_to_mesh(path, 0, v, 0.01, normals=n0)[1] == (0, len(v), 0)
        assert np.array_equal(got, n0)
        got2, _ = c.map_normals_to_mesh(h, v, 0.01, normals=n0)  # the API has no connectivity at all
        assert np.array_equal(got2, got)
    finally:
        c.close()


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
def test_neural_torus_mesh(oracle_built, mode):
    """The fitted 256x3 torus field on the parametric torus mesh (bench config 4's mesh) and
    on a jittered copy: the delta gate (violators), zero-gradient fallbacks and mapped counts
    equal the reference's; normals bitwise (oracle mode) or within 0.5 degrees (fast mode)."""
    from oracle import refshim
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    from paper_2201_09147_b200.meshes import torus_mesh
    path = os.path.join(ASSETS, "torus_w30.nest")
    if not os.path.exists(path):
        pytest.skip("fixture missing")
    seq = load_manifest(path)
    fine = len(seq.members) - 1
    c = Context(0, mode)
    try:
        h = DeviceSequence(c, seq).handles[fine]
        v, _ = torus_mesh()
        rng = np.random.default_rng(4)
        jit = v + rng.normal(scale=0.05, size=v.shape)  # some vertices leave the delta band
        jit[:7] = 0.0                                      # and a few sit at the origin
        for verts, delta in [(v, float(seq.deltas[fine])), (jit, float(seq.deltas[fine])), (jit, 0.02)]:
            n0 = rng.normal(size=verts.shape)
            got, cnt = c.map_normals_to_mesh(h, verts, delta, normals=n0)
            want, wcnt = refshim.map_normals_to_mesh(path, fine, verts, delta, normals=n0)
            if mode == "fp32":
                assert cnt == wcnt
                assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
            else:
                # the gate compares |f| with delta: a point within the fast mode's |df| ~ 1e-5 of
                # the band edge may flip, nothing else
                assert abs(cnt[0] - wcnt[0]) <= max(2, len(verts) // 10000) and sum(cnt) == sum(wcnt)
                both = ~np.all(got == n0, axis=1) & ~np.all(want == n0, axis=1)
                assert both.sum() >= 0.99 * wcnt[0]
                assert float(np.max(_angle_deg(got[both], want[both]))) <= 0.5
            assert cnt[1] > 0 or delta > 0.05
    finally:
        c.close()


def test_empty_mesh_is_a_contract_error():
    from paper_2201_09147_b200.abi import ERR_CONTRACT, NsdfError
    from paper_2201_09147_b200.engine import Context
    from paper_2201_09147_b200.manifest import Analytic
    c = Context(0, "fp32")
    try:
        h = c.upload(Analytic("sphere", {"r": 1.0}))
        with pytest.raises(NsdfError) as e:
            c.map_normals_to_mesh(h, np.zeros((0, 3)), 0.1)
        assert e.value.status == ERR_CONTRACT
    finally:
        c.close()


@pytest.mark.parametrize("seed", range(int(os.environ.get("NSDF_FUZZ_N", "6"))))
def test_random_vertex_sets_bitexact(oracle_built, seed):
    """Random vertex clouds (1 to 3000 vertices on, near and off the fitted torus: typically
    60-90% mapped, the rest δ-gate violators) with and without input normals against the
    reference in the FP32 oracle mode: counts exact, normals bit for bit."""
    from oracle import refshim
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    from paper_2201_09147_b200.meshes import torus_mesh
    path = os.path.join(ASSETS, "torus3.nest")
    if not os.path.exists(path):
        pytest.skip("fixture missing")
    seq = load_manifest(path)
    rng = np.random.default_rng(4000 + seed)
    v0, _ = torus_mesh()
    k = 1 if seed == 0 else int(rng.integers(1, 3000))
    v = v0[rng.integers(0, len(v0), k)] * rng.uniform(0.9, 1.1, (k, 1)) + rng.normal(0, 0.05, (k, 3))
    v = np.ascontiguousarray(v, np.float64)
    normals = None if seed % 2 else rng.normal(size=(k, 3))
    delta = float(seq.deltas[2]) * float(rng.uniform(0.5, 2.0))
    c = Context(0, "fp32")
    try:
        h = DeviceSequence(c, seq).handles[2]
        got, cnt = c.map_normals_to_mesh(h, v, delta, normals=normals)
        want, wcnt = refshim.map_normals_to_mesh(path, 2, v, delta, normals=normals)
        assert cnt == wcnt
        if want is None:
            assert got is None or not cnt[0]
        else:
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    finally:
        c.close()
