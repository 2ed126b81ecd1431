"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle on identical
weights, points and rays.  FP32 oracle mode must be bit-exact (100% mask,
dt = 0); the tolerance tests for the fast mode live in test_gpu_fast.py."""
import os

import numpy as np
import pytest

from conftest import ASSETS, bits, random_net, records_np

pytestmark = pytest.mark.gpu

ARCHS = [(64, 1), (128, 2), (256, 3), (16, 1), (12, 2), (5, 0)]


def _pts(k, rows=3, seed=0, half=1.2):
    return np.random.default_rng(seed).uniform(-half, half, size=(rows, k)).astype(np.float32)


@pytest.mark.parametrize("width,hidden", ARCHS)
def test_mlp_forward_gradient_bitexact(ctx, oracle_built, width, hidden):
    from oracle import corc, refshim
    net = random_net(width, hidden, seed=100 + width + hidden)
    h = ctx.upload(net)
    pts = _pts(1000 + width, seed=width)
    d_gpu, g_gpu = ctx.eval_grad(h, pts)
    d_ref, g_ref = refshim.mlp(net, pts, 2)
    d_orc, g_orc = corc.mlp(net, pts, 2)
    assert np.array_equal(bits(d_orc), bits(d_ref)) and np.array_equal(bits(g_orc), bits(g_ref))
    assert np.array_equal(bits(d_gpu), bits(d_ref)), np.max(np.abs(d_gpu - d_ref))
    assert np.array_equal(bits(g_gpu), bits(g_ref)), np.max(np.abs(g_gpu - g_ref))
    # separate calls are bitwise equal to the fused one (mlp.hpp:87-91)
    assert np.array_equal(bits(ctx.eval(h, pts)), bits(d_gpu))
    assert np.array_equal(bits(ctx.grad(h, pts)), bits(g_gpu))
    ctx.release(h)


def test_mlp_4d_spatial_gradient_bitexact(ctx, oracle_built):
    from oracle import refshim
    net = random_net(64, 1, input_dim=4, seed=7)
    h = ctx.upload(net)
    pts = _pts(777, rows=4, seed=3)
    d_gpu, g_gpu = ctx.eval_grad(h, pts)
    d_ref = refshim.mlp(net, pts, 0)[0]
    g_ref = refshim.mlp(net, pts, 1)[1]
    assert np.array_equal(bits(d_gpu), bits(d_ref))
    assert np.array_equal(bits(g_gpu), bits(g_ref))
    # 3-row batch + slice time == 4-row batch with a constant time row (field.cpp:213-220)
    t = np.float32(0.37)
    p4 = np.concatenate([pts[:3], np.full((1, pts.shape[1]), t, np.float32)])
    d3, g3 = ctx.eval_grad(h, pts[:3], time=float(t))
    d4, g4 = ctx.eval_grad(h, p4)
    assert np.array_equal(bits(d3), bits(d4)) and np.array_equal(bits(g3), bits(g4))


def test_batch_width_invariance(ctx):
    """Any split of a batch reproduces the same bits (test_tensor.cpp:283-309)."""
    net = random_net(128, 2, seed=9)
    h = ctx.upload(net)
    pts = _pts(4099, seed=11)
    d_all, g_all = ctx.eval_grad(h, pts)
    for lo, hi in [(0, 1), (1, 65), (65, 1000), (1000, 4099)]:
        d, g = ctx.eval_grad(h, pts[:, lo:hi])
        assert np.array_equal(bits(d), bits(d_all[lo:hi]))
        assert np.array_equal(bits(g), bits(g_all[:, lo:hi]))


def test_generate_rays_bitexact(ctx, oracle_built):
    from oracle import refshim
    from paper_2201_09147_b200.abi import Camera, standard_camera
    for cam in [standard_camera(64, 48), Camera((0, 0, 3), (0, 0, 0), (0, 1, 0), 40.0, 101, 101),
                Camera((1, 2, 3), (0.1, -0.2, 0.3), (0, 0, 1), 70.0, 33, 17)]:
        assert np.array_equal(bits(ctx.generate_rays(cam)), bits(refshim.generate_rays(cam)))


def _manifest(tmp_path, members, deltas, name="seq.nest"):
    from paper_2201_09147_b200.manifest import Sequence, save_sdfnet, write_manifest, Analytic
    names = []
    for i, m in enumerate(members):
        if isinstance(m, Analytic):
            names.append(None)
        else:
            nm = f"net{i}.sdfnet"
            save_sdfnet(m, os.path.join(tmp_path, nm))
            names.append(nm)
    seq = Sequence(list(members), list(deltas), [f"m{i}" for i in range(len(members))])
    path = os.path.join(tmp_path, name)
    write_manifest(seq, path, names)
    return path, seq


def _compare_records(a, b):
    ra, rb = records_np(a), records_np(b)
    for f in ["hit", "level", "iters"]:
        assert np.array_equal(ra[f], rb[f]), f
    for f in ["point", "t", "fd"]:
        assert np.array_equal(ra[f].view(np.uint32), rb[f].view(np.uint32)), f


def test_trace_analytic_sequences_match_reference(ctx, oracle_built, tmp_path):
    from oracle import refshim
    from paper_2201_09147_b200.abi import Camera, TraceConfig
    from paper_2201_09147_b200.manifest import Analytic
    from paper_2201_09147_b200.engine import DeviceSequence
    path, seq = _manifest(str(tmp_path), [Analytic("sphere", {"r": 1.0}), Analytic("sphere", {"r": 0.95})],
                          [0.1, 0.05])
    ds = DeviceSequence(ctx, seq)
    cam = Camera((0, 0, 3), (0, 0, 0), (0, 1, 0), 45.0, 65, 65)
    for budgets in [(40, 40), (50, 0), (1, 3), (0, 7)]:
        cfg = TraceConfig(budgets)
        got, _ = ctx.trace_image(ds.levels(), cam, cfg)
        want = refshim.trace_image(path, cam, cfg)
        _compare_records(got, want)


def test_analytic_fields_bitexact(ctx, oracle_built, tmp_path):
    """Analytic torus / box / sphere values and gradients (field.cpp:57-124, double then
    float cast) bit for bit against the compiled reference: the torus needs glibc's hypot,
    restated on the device (common.cuh hypot_ref) because CUDA's hypot differs in the last
    bit; then whole traces of an analytic torus pair, bitwise."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import TraceConfig, standard_camera
    from paper_2201_09147_b200.manifest import Analytic
    from paper_2201_09147_b200.engine import DeviceSequence
    members = [Analytic("torus", {"R": 0.6, "r": 0.3}), Analytic("box", {"hx": 0.6, "hy": 0.45, "hz": 0.5}),
               Analytic("sphere", {"cx": 0.1, "r": 0.7})]
    path, seq = _manifest(str(tmp_path), members, [0.2, 0.1, 0.05])
    ds = DeviceSequence(ctx, seq)
    rng = np.random.default_rng(17)
    pts = rng.uniform(-1.3, 1.3, size=(3, 200000)).astype(np.float32)
    pts[:, :1000] *= np.float32(1e-3)  # near the torus axis / the origin
    pts[1, 1000:2000] = 0.0            # on the torus' plane of symmetry
    for i, h in enumerate(ds.handles):
        d_gpu, g_gpu = ctx.eval_grad(h, pts)
        d_ref, g_ref = refshim.field_eval(path, i, pts)
        assert np.array_equal(bits(d_gpu), bits(d_ref)), (members[i].name, int(np.sum(bits(d_gpu) != bits(d_ref))))
        assert np.array_equal(bits(g_gpu), bits(g_ref)), (members[i].name, int(np.sum(bits(g_gpu) != bits(g_ref))))
    path2, seq2 = _manifest(str(tmp_path), [Analytic("torus", {"R": 0.6, "r": 0.4}),
                                            Analytic("torus", {"R": 0.6, "r": 0.3})], [0.15, 0.05], name="t2.nest")
    ds2 = DeviceSequence(ctx, seq2)
    cam = standard_camera(96, 64)
    for budgets in [(40, 40), (30, 0), (0, 60)]:
        cfg = TraceConfig(budgets)
        got, _ = ctx.trace_image(ds2.levels(), cam, cfg)
        _compare_records(got, refshim.trace_image(path2, cam, cfg))


def test_trace_kats(ctx):
    """Reference tracer KATs (test_tracer.cpp:74-87, 104-121, 185-192, 281-307)."""
    from paper_2201_09147_b200.abi import TraceConfig
    from paper_2201_09147_b200.manifest import Analytic, Sequence
    from paper_2201_09147_b200.engine import DeviceSequence
    ray = np.array([[3, 0, 0, -1, 0, 0]], np.float32)
    one = DeviceSequence(ctx, Sequence([Analytic("sphere", {"r": 1.0})], [0.05], ["s"]))
    r = records_np(ctx.trace_rays(one.levels(), TraceConfig((100,)), ray))[0]
    assert r["hit"] == 1 and abs(r["point"][0] - 1.0) < 2e-3 and abs(r["t"] - 2.0) < 4e-3 and r["fd"] <= 1e-3
    con = DeviceSequence(ctx, Sequence([Analytic("sphere", {"r": 1.0}), Analytic("sphere", {"r": 0.95})],
                                       [0.1, 0.05], ["a", "b"]))
    r = records_np(ctx.trace_rays(con.levels(), TraceConfig((50, 50)), ray))[0]
    assert r["hit"] == 1 and r["level"] == 1 and abs(r["point"][0] - 0.95) < 2e-3
    assert r["iters"][0] > 0 and r["iters"][1] > 0
    r = records_np(ctx.trace_rays(con.levels(), TraceConfig((50, 0)), ray))[0]
    assert r["hit"] == 1 and abs(r["point"][0] - 1.0) < 2e-3 and r["iters"][1] == 0
    inside = np.array([[1.05, 0, 0, -1, 0, 0]], np.float32)
    r = records_np(ctx.trace_rays(con.levels(), TraceConfig((30, 30)), inside))[0]
    assert r["hit"] == 1 and r["iters"][0] == 1 and abs(r["point"][0] - 0.95) < 2e-3
    miss = np.array([[4, 0.3, 0, -1, 0, 0]], np.float32)
    r = records_np(ctx.trace_rays(one.levels(), TraceConfig((1,)), miss))[0]
    assert r["hit"] == 0 and r["iters"][0] == 1 and r["t"] > 0


def test_trace_neural_sequence_bitexact(ctx, oracle_built, tmp_path):
    from oracle import refshim
    from paper_2201_09147_b200.abi import TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    nets = [random_net(64, 1, seed=5, omega0=10.0), random_net(128, 2, seed=6, omega0=10.0)]
    path, seq = _manifest(str(tmp_path), nets, [0.3, 0.1])
    ds = DeviceSequence(ctx, seq)
    cam = standard_camera(48, 40)
    for budgets in [(20, 10), (0, 15), (12, 0)]:
        cfg = TraceConfig(budgets)
        got, st = ctx.trace_image(ds.levels(), cam, cfg)
        want = refshim.trace_image(path, cam, cfg)
        _compare_records(got, want)
        rec = records_np(want)
        assert st.evals[0] + st.evals[1] == int(rec["iters"].astype(np.int64).sum())


def _fixture(name):
    p = os.path.join(ASSETS, name)
    if not os.path.exists(p):
        pytest.skip(f"fixture {name} not generated")
    return p


def test_render_fixture_bitexact_small(ctx, oracle_built):
    """Whole render of the committed torus sequence vs the reference, bitwise."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    path = _fixture("torus_w30.nest")
    seq = load_manifest(path)
    ds = DeviceSequence(ctx, seq)
    cam = standard_camera(64, 64)
    shade = ShadeConfig(specular=0.3)
    for budgets, src in [((20, 5, 5), 0), ((40, 0, 0), 1), ((0, 0, 30), 0)]:
        cfg = TraceConfig(budgets)
        rgb, depth, mask, st = ctx.render(ds.levels(), cam, cfg, shade, src)
        rrgb, rdepth, rmask, _ = refshim.render(path, cam, cfg, shade, src)
        assert np.array_equal(mask, rmask)
        assert np.array_equal(depth.view(np.uint32), rdepth.view(np.uint32))
        assert np.max(np.abs(rgb - rrgb)) <= 1e-6


def test_normal_map_and_shade_bitexact(ctx, oracle_built):
    from oracle import corc
    from paper_2201_09147_b200.abi import ShadeConfig, standard_camera
    net = random_net(64, 2, seed=12, omega0=10.0)
    h = ctx.upload(net)
    pts = _pts(513, seed=4, half=0.8)
    fb = _pts(513, seed=5)
    n_gpu, o_gpu, f_gpu = ctx.normal_map(h, pts, 0.05, fb)
    n_orc, o_orc, f_orc = corc.normal_map(net, pts, 0.05, fb)
    assert np.array_equal(bits(n_gpu), bits(n_orc)) and (o_gpu, f_gpu) == (o_orc, f_orc)
    cam = standard_camera()
    for sc in [ShadeConfig(), ShadeConfig(specular=0.3)]:
        rgb = ctx.shade(pts, n_gpu, sc, cam)
        want = corc.shade(pts, n_orc, sc, cam)
        assert np.max(np.abs(rgb - want)) <= 1e-6


@pytest.mark.parametrize("seed", range(int(os.environ.get("NSDF_FUZZ_N", "8"))))
def test_render_randomized_bitexact(ctx, oracle_built, seed):
    """Randomised scenes in the FP32 oracle mode against the reference renderer on the same
    manifest: image size (1 x 1 up to 80 x 80), camera position and field of view, per-level
    budgets (zeros included), specular, normal source.  Mask and depth bit for bit, colour
    within the shading tolerance the fixed cases use (1e-6).  NSDF_FUZZ_N sets the count."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import Camera, ShadeConfig, TraceConfig
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    path = os.path.join(ASSETS, "torus3.nest")
    if not os.path.exists(path):
        pytest.skip("fixture missing")
    rng = np.random.default_rng(2000 + seed)
    w, h = (1, 1) if seed == 0 else (int(rng.integers(1, 81)), int(rng.integers(1, 81)))
    d = rng.normal(size=3)
    pos = d / np.linalg.norm(d) * rng.uniform(1.6, 4.0)
    cam = Camera(tuple(pos), tuple(rng.uniform(-0.2, 0.2, 3)), (0, 1, 0), float(rng.uniform(20, 90)), w, h)
    budgets = [int(b) for b in rng.integers(0, 31, 3)]
    if not any(budgets):
        budgets[0] = 20
    cfg = TraceConfig(tuple(budgets))
    shade = ShadeConfig(specular=float(rng.uniform(0, 1)))
    src = int(rng.integers(0, 2))
    rgb, depth, mask, _ = ctx.render(DeviceSequence(ctx, load_manifest(path)).levels(), cam, cfg, shade, src)
    rrgb, rdepth, rmask, _ = refshim.render(path, cam, cfg, shade, src)
    assert np.array_equal(mask.reshape(-1), rmask.reshape(-1)), (w, h, budgets)
    assert np.array_equal(depth.reshape(-1).view(np.uint32), rdepth.reshape(-1).view(np.uint32))
    assert np.max(np.abs(rgb.reshape(-1) - rrgb.reshape(-1))) <= 1e-6


@pytest.mark.parametrize("seed", range(int(os.environ.get("NSDF_FUZZ_N", "8"))))
def test_trace_rays_and_normal_map_randomized_bitexact(ctx, oracle_built, seed):
    """Randomised ray batches through trace_rays (batch sizes from 1, origins outside, near
    and inside the surface, directions aimed or random, per-level budgets with zeros) and
    random point sets through the normal map (on, near and far off the surface: the δ gate,
    with and without fallback normals) in the FP32 oracle mode against the reference: every
    HitRecord field and every normal bit for bit, the outside/fallback counts equal."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import TraceConfig
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    path = _fixture("torus3.nest")
    seq = load_manifest(path)
    ds = DeviceSequence(ctx, seq)
    rng = np.random.default_rng(3000 + seed)
    n = 1 if seed == 0 else int(rng.integers(1, 3000))
    d = rng.normal(size=(n, 3))
    o = d / np.linalg.norm(d, axis=1, keepdims=True) * rng.uniform(0.0, 4.0, (n, 1))
    aim = rng.uniform(-0.3, 0.3, (n, 3)) - o
    rnd = rng.normal(size=(n, 3))
    dirs = np.where(rng.uniform(size=(n, 1)) < 0.7, aim, rnd)
    dirs /= np.maximum(np.linalg.norm(dirs, axis=1, keepdims=True), 1e-12)
    rays = np.concatenate([o, dirs], axis=1).astype(np.float32)
    budgets = [int(b) for b in rng.integers(0, 31, 3)]
    if not any(budgets):
        budgets[1] = 15
    cfg = TraceConfig(tuple(budgets))
    _compare_records(ctx.trace_rays(ds.levels(), cfg, rays), refshim.trace_rays(path, cfg, rays))
    # normal map of the finest member on the traced hits plus random points
    rec = records_np(refshim.trace_rays(path, cfg, rays))
    pts = np.concatenate([rec["point"][rec["hit"] == 1], rng.uniform(-1.5, 1.5, (int(rng.integers(1, 500)), 3))])
    pts = np.ascontiguousarray(pts.T, np.float32)
    delta = float(seq.deltas[2])
    fb = None if seed % 2 else rng.normal(size=pts.shape).astype(np.float32)
    n_gpu, o_gpu, f_gpu = ctx.normal_map(ds.handles[2], pts, delta, fb)
    n_ref, o_ref, f_ref = refshim.normal_map(path, 2, pts, delta, fb)
    assert (o_gpu, f_gpu) == (o_ref, f_ref)
    assert np.array_equal(bits(n_gpu), bits(n_ref))
