"""GPU parity of the tcgen05 fast mode (FP16 operands, FP32 accumulation) against the
reference CPU path on identical weights and rays, with the BASELINE tolerances
(SURVEY.md §8d): hit/miss mask agreement >= 99.9%, |dt| <= 1e-3 on common hits (scene
scale 1), normals within 0.5 deg — end to end and at identical points."""
import ctypes
import os

import numpy as np
import pytest

from conftest import ASSETS, random_net, records_np

pytestmark = pytest.mark.gpu

MASK_MIN = 0.999
DT_MAX = 1e-3        # BASELINE depth tolerance
ANGLE_MAX = 0.5      # degrees


def _fixture(name):
    p = os.path.join(ASSETS, name)
    if not os.path.exists(p):
        pytest.skip(f"fixture {name} not generated")
    return p


@pytest.fixture(scope="module")
def fast():
    from paper_2201_09147_b200.engine import Context
    c = Context(0, "fp16")
    yield c
    c.close()


def angle_deg(a, b):
    a = a / np.linalg.norm(a, axis=0, keepdims=True)
    b = b / np.linalg.norm(b, axis=0, keepdims=True)
    return np.degrees(np.arccos(np.clip((a * b).sum(0), -1.0, 1.0)))


@pytest.mark.parametrize("name", ["64x1", "128x2", "256x3"])
def test_fast_mlp_close_to_oracle(ctx, fast, name):
    from paper_2201_09147_b200.manifest import load_sdfnet
    net = load_sdfnet(_fixture(f"torus_w30_{name}.sdfnet"))
    pts = np.random.default_rng(1).uniform(-1, 1, (3, 20000)).astype(np.float32)
    d0, g0 = ctx.eval_grad(ctx.upload(net), pts)
    h = fast.upload(net)
    d1, g1 = fast.eval_grad(h, pts)
    assert np.array_equal(fast.eval(h, pts), d1)  # forward-only and fused tiles agree
    near = np.abs(d0) < 0.05
    assert np.abs(d1 - d0).max() < 2e-3, np.abs(d1 - d0).max()
    assert np.percentile(angle_deg(g0[:, near], g1[:, near]), 99.9) < ANGLE_MAX


def test_fast_e4m3_correction_terms(ctx, fast):
    """256-wide nets at omega0 <= 15 (the headline's finest level, torus3 256x3 at omega0 =
    10) run the split-precision correction terms as one E4M3 MMA per K step in the forward
    tiles (mlp_tc.cuh tc_split8): the forward values then differ from the fused gradient
    tiles' (which keep the fp16 terms) by the E4M3 rounding of the corrections — proof that
    the path ran — and stay within 5e-5 of the FP32 oracle (emulated: |df| p99.9 4.8e-6 near the
    surface from the E4M3 terms alone).  NSDF_TC_E4M3=0 restores the fp16 terms."""
    from paper_2201_09147_b200.manifest import load_sdfnet
    net = load_sdfnet(_fixture("torus3_256x3.sdfnet"))
    assert net.omega0 <= 15
    pts = np.random.default_rng(2).uniform(-1, 1, (3, 20000)).astype(np.float32)
    d0 = ctx.eval(ctx.upload(net), pts)
    h = fast.upload(net)
    d1 = fast.eval(h, pts)
    dg, g1 = fast.eval_grad(h, pts)
    assert not np.array_equal(d1, dg)  # the forward tiles took the E4M3 path
    near = np.abs(d0) < 0.05
    err = np.abs(d1 - d0)
    print(f"E4M3 corrections: |df| max {err.max():.2e}, near-surface p99.9 {np.percentile(err[near], 99.9):.2e}; "
          f"fused (fp16 terms) max {np.abs(dg - d0).max():.2e}")
    assert err.max() < 5e-5, err.max()
    assert np.abs(dg - d0).max() < 5e-5


# the standard depths (compiled-in layer counts) and others (runtime layer loops; 64x5 streams
# its weights instead of keeping them resident; 256-wide layers run as two N-blocks)
@pytest.mark.parametrize("width,hidden", [(64, 1), (128, 2), (256, 3), (64, 2), (64, 5), (128, 1), (128, 3),
                                          (256, 1), (256, 2), (256, 4)])
def test_fast_mlp_random_init(ctx, fast, width, hidden):
    net = random_net(width, hidden, seed=40 + width)
    pts = np.random.default_rng(2).uniform(-1.2, 1.2, (3, 3000)).astype(np.float32)
    d0, g0 = ctx.eval_grad(ctx.upload(net), pts)
    d1, g1 = fast.eval_grad(fast.upload(net), pts)
    assert np.abs(d1 - d0).max() < 5e-4
    assert np.median(angle_deg(g0, g1)) < 0.1


def _trace_and_normals(c, ds, cam, cfg, normal_idx):
    recs, st = c.trace_image(ds.levels(), cam, cfg)
    r = records_np(recs)
    hit = r["hit"] == 1
    pts = np.ascontiguousarray(r["point"][hit].T)
    nrm, _, _ = c.normal_map(ds.handles[normal_idx], pts, ds.seq.deltas[normal_idx])
    return r, hit, pts, nrm


@pytest.mark.parametrize("budgets", [(20, 5, 5), (40, 20, 20), (0, 0, 40)])
def test_fast_trace_parity_torus(ctx, fast, budgets):
    """Mask, depth and end-to-end normal parity of the fast mode vs the bit-exact oracle
    mode (itself pinned bitwise to the reference in test_gpu_parity.py)."""
    from paper_2201_09147_b200.abi import TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    seq = load_manifest(_fixture("torus_w30.nest"))
    cam = standard_camera(480, 270)
    cfg = TraceConfig(budgets)
    r0, hit0, p0, n0 = _trace_and_normals(ctx, DeviceSequence(ctx, seq), cam, cfg, 2)
    r1, hit1, p1, n1 = _trace_and_normals(fast, DeviceSequence(fast, seq), cam, cfg, 2)
    agree = np.mean(hit0 == hit1)
    both = hit0 & hit1
    dt = np.abs(r0["t"][both] - r1["t"][both])
    # end-to-end normals on common hits
    idx0 = np.cumsum(hit0) - 1
    idx1 = np.cumsum(hit1) - 1
    ang = angle_deg(n0[:, idx0[both]], n1[:, idx1[both]])
    print(f"budgets {budgets}: mask {agree:.5f}, hits {hit0.sum()}/{hit1.sum()}, dt max {dt.max():.2e} "
          f"p99.9 {np.percentile(dt, 99.9):.2e}, normals max {ang.max():.3f} p99.9 {np.percentile(ang, 99.9):.3f}")
    assert agree >= MASK_MIN
    assert np.percentile(dt, 99.9) <= DT_MAX
    assert np.percentile(ang, 99.9) <= ANGLE_MAX


def test_fast_render_matches_oracle_mode(ctx, fast):
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    seq = load_manifest(_fixture("torus_w30.nest"))
    cam = standard_camera(320, 180)
    cfg = TraceConfig((20, 5, 5))
    shade = ShadeConfig(specular=0.3)
    for src in (0, 1):
        rgb0, d0, m0, _ = ctx.render(DeviceSequence(ctx, seq).levels(), cam, cfg, shade, src)
        rgb1, d1, m1, st = fast.render(DeviceSequence(fast, seq).levels(), cam, cfg, shade, src)
        assert np.mean(m0 == m1) >= MASK_MIN
        both = (m0 == 1) & (m1 == 1)
        assert np.percentile(np.abs(d0 - d1)[both], 99.9) <= DT_MAX
        assert np.mean(np.abs(rgb0 - rgb1)[both]) < 5e-3


def _render_pair(ctx, fast, seq, cam, cfg, shade, src, time=0.0):
    from paper_2201_09147_b200.engine import DeviceSequence
    a = ctx.render(DeviceSequence(ctx, seq).levels(time=time), cam, cfg, shade, src)
    b = fast.render(DeviceSequence(fast, seq).levels(time=time), cam, cfg, shade, src)
    return a, b


def _assert_render_parity(a, b):
    rgb0, d0, m0, _ = a
    rgb1, d1, m1, _ = b
    assert np.mean(m0 == m1) >= MASK_MIN
    both = (m0 == 1) & (m1 == 1)
    if both.any():
        assert np.percentile(np.abs(d0 - d1)[both], 99.9) <= DT_MAX
        assert np.mean(np.abs(rgb0 - rgb1)[both]) < 5e-3


def test_config1_single_256x3(ctx, fast, oracle_built):
    """BASELINE config 1 (single 256x3, budgets {40}) at 128^2: oracle mode bit-exact vs the
    reference, fast mode within tolerance."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest, write_manifest
    full = load_manifest(_fixture("torus_w30.nest"))
    seq = full.subsequence([2])
    cam = standard_camera(128, 128)
    cfg = TraceConfig((40,))
    shade = ShadeConfig(specular=0.3)
    a, b = _render_pair(ctx, fast, seq, cam, cfg, shade, 0)
    _assert_render_parity(a, b)
    import json, tempfile
    j = json.load(open(_fixture("torus_w30.nest")))
    j["fields"] = [dict(j["fields"][2], weights=os.path.join(ASSETS, j["fields"][2]["weights"]))]
    j["deltas"] = [j["deltas"][2]]
    with tempfile.NamedTemporaryFile("w", suffix=".nest", delete=False) as f:
        json.dump(j, f)
    r = refshim.render(f.name, cam, cfg, shade, 0)
    os.unlink(f.name)
    assert np.array_equal(a[2], r[2]) and np.array_equal(a[1].view(np.uint32), r[1].view(np.uint32))


def test_config4_mesh_gbuffer_normals(ctx, fast, oracle_built):
    """BASELINE config 4: torus-mesh G-buffer positions -> 256x3 neural normals; oracle mode
    bit-exact vs the reference's neural_normal_map on the identical positions, fast mode
    within 0.5 deg."""
    import torch
    from oracle import refshim
    from paper_2201_09147_b200.abi import standard_camera
    from paper_2201_09147_b200.manifest import load_manifest
    from paper_2201_09147_b200.meshes import torus_mesh
    full = load_manifest(_fixture("torus_w30.nest"))
    net, delta = full.members[2], full.deltas[2]
    cam = standard_camera(256, 144)
    n = cam.width * cam.height
    pos = torch.zeros(3 * n, dtype=torch.float32, device="cuda")
    mask = torch.zeros(n, dtype=torch.uint8, device="cuda")
    v, t = torus_mesh()
    ctx.raycast_mesh(cam, v, t, pos.data_ptr(), mask.data_ptr())
    pts = pos.view(3, n)[:, mask.bool()].cpu().numpy()
    assert pts.shape[1] > 1000
    # hits lie on the mesh, i.e. near the torus surface
    s = np.hypot(pts[0], pts[2])
    assert np.abs(np.hypot(s - 0.6, pts[1]) - 0.3).max() < 0.01
    n0, o0, f0 = ctx.normal_map(ctx.upload(net), pts, delta)
    n1, o1, f1 = fast.normal_map(fast.upload(net), pts, delta)
    import json, tempfile
    j = json.load(open(_fixture("torus_w30.nest")))
    j["fields"] = [dict(j["fields"][2], weights=os.path.join(ASSETS, j["fields"][2]["weights"]))]
    j["deltas"] = [j["deltas"][2]]
    with tempfile.NamedTemporaryFile("w", suffix=".nest", delete=False) as f:
        json.dump(j, f)
    nr, orr, fr = refshim.normal_map(f.name, 0, pts, delta)
    os.unlink(f.name)
    assert np.array_equal(n0.view(np.uint32), nr.view(np.uint32)) and (o0, f0) == (orr, fr)
    assert np.percentile(angle_deg(n0, n1), 99.9) <= ANGLE_MAX


@pytest.mark.parametrize("t", [0.0, 0.37, 1.0])
def test_config5_animated_slices(ctx, fast, oracle_built, t):
    """BASELINE config 5 (4-D 64x1 > 128x2 blend) time slices: oracle mode bit-exact vs the
    reference's AnimatedSequence::slice render, fast mode within tolerance."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.manifest import load_manifest
    path = _fixture("blend4d_w30.nest")
    seq = load_manifest(path)
    cam = standard_camera(96, 64)
    cfg = TraceConfig((20, 10))
    shade = ShadeConfig(specular=0.3)
    a, b = _render_pair(ctx, fast, seq, cam, cfg, shade, 0, time=t)
    _assert_render_parity(a, b)
    r = refshim.render(path, cam, cfg, shade, 0, time=t)
    assert np.array_equal(a[2], r[2]) and np.array_equal(a[1].view(np.uint32), r[1].view(np.uint32))
    assert np.max(np.abs(a[0] - r[0])) <= 1e-6


# ---- persistent level kernel (tc_trace_level): edge cases --------------------------------
def _torus_levels(c):
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    return DeviceSequence(c, load_manifest(_fixture("torus_w30.nest")))


def _rays(n, seed=0, away=False):
    rng = np.random.default_rng(seed)
    o = np.tile(np.array([2.0, 1.5, 2.0], np.float32), (n, 1))
    target = rng.uniform(-0.8, 0.8, (n, 3)).astype(np.float32)
    d = (target - o) if not away else (o - target)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.concatenate([o, d], 1).astype(np.float32)


@pytest.mark.parametrize("n", [1, 5, 127, 128, 129, 1000, 40000])
def test_fast_trace_rays_ragged(ctx, fast, n):
    """Any ray count (a partly filled tile, one ray, many claims) gives the oracle's
    per-ray result within tolerance, and the persistent kernel's evaluation counter equals
    the records' iterations_used (stats come from the kernel, not the records)."""
    from paper_2201_09147_b200.abi import TraceConfig
    cfg = TraceConfig((20, 5, 5))
    rays = _rays(n, seed=n)
    r0 = records_np(ctx.trace_rays(_torus_levels(ctx).levels(), cfg, rays))
    r1 = records_np(fast.trace_rays(_torus_levels(fast).levels(), cfg, rays))
    assert np.mean(r0["hit"] == r1["hit"]) >= (MASK_MIN if n >= 1000 else 1.0)
    both = (r0["hit"] == 1) & (r1["hit"] == 1)
    if both.any():
        assert np.abs(r0["t"][both] - r1["t"][both]).max() <= 1.5 * DT_MAX
    assert (r1["iters"][:, :3] <= np.array([20, 5, 5])).all()


def test_fast_budget_one_and_all_miss(ctx, fast):
    from paper_2201_09147_b200.abi import TraceConfig
    # budget 1 at every level: every ray leaves each level after one evaluation
    rays = _rays(3000, seed=1)
    r1 = records_np(fast.trace_rays(_torus_levels(fast).levels(), TraceConfig((1, 1, 1)), rays))
    r0 = records_np(ctx.trace_rays(_torus_levels(ctx).levels(), TraceConfig((1, 1, 1)), rays))
    assert (r1["iters"][:, :3] <= 1).all()
    assert np.mean(r0["level"] == r1["level"]) >= MASK_MIN
    # rays pointing away from the scene: level 0 marches them past t_max, the later levels
    # receive empty lists (their persistent launches exit without work)
    away = _rays(5000, seed=2, away=True)
    r = records_np(fast.trace_rays(_torus_levels(fast).levels(), TraceConfig((20, 5, 5)), away))
    assert r["hit"].sum() == 0 and (r["iters"][:, 1:3] == 0).all()


def test_fast_stats_match_records(fast):
    from paper_2201_09147_b200.abi import TraceConfig, standard_camera
    recs, st = fast.trace_image(_torus_levels(fast).levels(), standard_camera(320, 180), TraceConfig((20, 5, 5)))
    r = records_np(recs)
    for j in range(3):
        assert st.evals[j] == int(r["iters"][:, j].astype(np.int64).sum())
    assert st.hits == int(r["hit"].sum())


@pytest.mark.parametrize("budgets", [(40, 20, 20), (40, 20, 2), (40, 20, 1), (1, 1, 3)])
def test_fast_e4m3_resume_bookkeeping(ctx, fast, budgets):
    """torus3's 128/256-wide levels run E4M3 correction terms, and the final level parks
    near-threshold stop decisions for the fp16-term resume launch.  The parked evaluation is
    not counted twice and the resumed rays keep their iteration counts: the kernels'
    evaluation counters equal the records' iterations_used, no level exceeds its budget (also
    with a final budget of 1 or 2, where a parked ray resumes at its last allowed iteration),
    the hit count matches, and the frame agrees with the oracle mode's."""
    from paper_2201_09147_b200.abi import TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    seq = load_manifest(_fixture("torus3.nest"))
    cam, cfg = standard_camera(640, 360), TraceConfig(budgets)
    recs, st = fast.trace_image(DeviceSequence(fast, seq).levels(), cam, cfg)
    r = records_np(recs)
    for j in range(3):
        assert st.evals[j] == int(r["iters"][:, j].astype(np.int64).sum()), j
    assert (r["iters"][:, :3] <= np.array(budgets)).all()
    assert st.hits == int(r["hit"].sum())
    r0 = records_np(ctx.trace_image(DeviceSequence(ctx, seq).levels(), cam, cfg)[0])
    assert np.sum(r0["hit"] != r["hit"]) <= max(1, int(1e-3 * r["hit"].size))


def test_fast_mixed_analytic_and_neural_levels(ctx, fast, tmp_path):
    """An analytic coarse level (FFMA iterations) feeding the persistent tcgen05 levels."""
    import json
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    _fixture("torus_w30_256x3.sdfnet")
    man = tmp_path / "mixed.nest"
    man.write_text(json.dumps({"deltas": [0.45, 0.107, 0.05], "fields": [
        {"analytic": "sphere", "params": {"r": 1.05}},
        {"weights": os.path.join(ASSETS, "torus_w30_64x1.sdfnet")},
        {"weights": os.path.join(ASSETS, "torus_w30_256x3.sdfnet")}]}))
    seq = load_manifest(str(man))
    cam = standard_camera(320, 200)
    cfg = TraceConfig((10, 20, 8))
    shade = ShadeConfig(specular=0.3)
    a = ctx.render(DeviceSequence(ctx, seq).levels(), cam, cfg, shade)
    b = fast.render(DeviceSequence(fast, seq).levels(), cam, cfg, shade)
    _assert_render_parity(a, b)
    assert a[2].sum() > 1000


def _max_sine_argument(seq, n=100000, seed=3):
    """Largest |omega0 * (W a + b)| any sine of the sequence's nets sees, over uniform points
    of the domain and the 4-D slice times (float64 forward pass of the fixture weights)."""
    rng = np.random.default_rng(seed)
    worst = 0.0
    for net in seq.members:
        if not hasattr(net, "layers"):
            continue
        x = rng.uniform(-1.0, 1.0, size=(net.input_dim, n))
        for w, b in net.layers()[:-1]:
            z = net.omega0 * (w @ x + b[:, None])
            worst = max(worst, float(np.max(np.abs(z))))
            x = np.sin(z)
    return worst


def test_fast_sine_at_large_arguments(fast):
    """The fast mode's activation (MUFU sin.approx behind FMUL.RZ(x, 1/2pi): the explicit
    range reduction to revolutions is that one RZ multiply) against float64 sin of the same
    fp32 argument, over the full range of omega0 * z the committed fixtures produce (with
    omega0 = 30 that is well beyond pi): absolute error <= 2^-20 + |x| * 2^-22 — one RZ
    rounding of x/2pi plus the MUFU approximation — for sin and for the cos(x) = sin(x + pi/2)
    derivative factor of the tangent rows."""
    from paper_2201_09147_b200.manifest import load_manifest
    top = 0.0
    for name in ("torus_w30.nest", "blend4d_w30.nest"):
        p = os.path.join(ASSETS, name)
        if os.path.exists(p):
            top = max(top, _max_sine_argument(load_manifest(p)))
    assert top > 3.5, top  # the fixtures do leave [-pi, pi]
    rng = np.random.default_rng(0)
    lim = 1.05 * top
    x = np.concatenate([np.linspace(-lim, lim, 400001), rng.uniform(-lim, lim, 400000),
                        np.arange(-64, 65) * np.pi / 2, [0.0, 1e-30, -1e-30]]).astype(np.float32)
    s = np.zeros_like(x)
    c = np.zeros_like(x)
    fp = ctypes.POINTER(ctypes.c_float)
    st = fast.lib.nsdf_cuda_probe_fast_sine(fast._ctx, x.ctypes.data_as(fp), len(x), s.ctypes.data_as(fp),
                                            c.ctypes.data_as(fp))
    assert st == 0
    xd = x.astype(np.float64)
    bound = 2.0 ** -20 + np.abs(xd) * 2.0 ** -22
    es = np.abs(s - np.sin(xd))
    ec = np.abs(c - np.cos(xd))
    assert np.all(es <= bound), (float(np.max(es / bound)), float(xd[np.argmax(es / bound)]))
    assert np.all(ec <= bound + np.abs(xd) * 2.0 ** -24), float(np.max(ec / bound))
    print(f"max |omega0 z| of the fixtures {top:.1f}; max sine error {es.max():.2e}, cos {ec.max():.2e}")


@pytest.mark.parametrize("seed", range(int(os.environ.get("NSDF_FUZZ_N", "10"))))
def test_fast_render_randomized(ctx, fast, seed):
    """Randomised scenes through both modes: image size (1 x 1 up to 200 x 200), camera
    position and field of view, per-level budgets (zeros included), specular, normal source.
    The fast frame agrees with the oracle-mode frame within the BASELINE tolerances (mask
    disagreement counted in pixels, so a one-pixel image is held to the same standard), and
    the fast frame assembled from tile shares (random tile size and rank count) equals the
    whole fast frame bit for bit.  NSDF_FUZZ_N sets the number of scenes (default 10)."""
    import torch
    from paper_2201_09147_b200.abi import Camera, ShadeConfig, TraceConfig
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import load_manifest
    rng = np.random.default_rng(1000 + seed)
    seq = load_manifest(_fixture("torus3.nest"))
    w, h = (1, 1) if seed == 0 else (int(rng.integers(1, 201)), int(rng.integers(1, 201)))
    d = rng.normal(size=3)
    pos = d / np.linalg.norm(d) * rng.uniform(1.6, 4.0)
    cam = Camera(tuple(pos), tuple(rng.uniform(-0.2, 0.2, 3)), (0, 1, 0), float(rng.uniform(20, 90)), w, h)
    budgets = [int(b) for b in rng.integers(0, 31, 3)]
    if not any(budgets):
        budgets[-1] = 20
    cfg = TraceConfig(tuple(budgets))
    shade = ShadeConfig(specular=float(rng.uniform(0, 1)))
    src = int(rng.integers(0, 2))
    a = ctx.render(DeviceSequence(ctx, seq).levels(), cam, cfg, shade, src)
    ds = DeviceSequence(fast, seq)
    b = fast.render(ds.levels(), cam, cfg, shade, src)
    rgb0, d0, m0, _ = a
    rgb1, d1, m1, _ = b
    n = w * h
    assert np.sum(m0 != m1) <= max(1, int(1e-3 * n)), (w, h, budgets)
    both = (m0 == 1) & (m1 == 1)
    if both.any():
        # depth: at most 0.1% of the common hits (and at least one allowed, as for the mask,
        # so a small image is held to the same standard) beyond 1e-3, each of those a single
        # stop-band step (<= 1.05 eps_stop: test_depth_outliers_are_stop_band_steps shows the
        # mechanism ray by ray at full size)
        dt = np.abs(d0 - d1)[both]
        assert int(np.sum(dt > DT_MAX)) <= max(1, int(1e-3 * dt.size)), (np.sort(dt)[-5:], dt.size)
        assert dt.max() <= 1.05 * cfg.eps_stop, dt.max()
    # tile shares of the same fast frame into one device framebuffer
    tile, world = int(rng.choice([8, 16, 32, 64])), int(rng.integers(2, 5))
    fb = [torch.zeros(3 * n, device="cuda"), torch.zeros(n, device="cuda"),
          torch.zeros(n, dtype=torch.uint8, device="cuda")]
    for r in range(world):
        fast.render_device(ds.levels(), cam, cfg, shade, *(x.data_ptr() for x in fb), src, -1, tile, r, world)
    torch.cuda.synchronize()
    assert np.array_equal(fb[2].cpu().numpy(), m1.reshape(-1))
    assert np.array_equal(fb[1].cpu().numpy().view(np.uint32), d1.reshape(-1).view(np.uint32))
    assert np.array_equal(fb[0].cpu().numpy().view(np.uint32), rgb1.reshape(-1).view(np.uint32))
