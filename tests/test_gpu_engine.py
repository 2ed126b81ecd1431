"""GPU: engine behaviour beyond arithmetic parity — the frame/tile scheduler's per-rank path
(tile-sharded renders reassemble the single-GPU frame bit for bit), determinism, stats
accounting, and the reference's error conventions through the C ABI."""
import os

import numpy as np
import pytest

from conftest import ASSETS, random_net

pytestmark = pytest.mark.gpu


def _seq():
    from paper_2201_09147_b200.manifest import load_manifest
    p = os.path.join(ASSETS, "torus_w30.nest")
    if not os.path.exists(p):
        pytest.skip("fixture missing")
    return load_manifest(p)


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
@pytest.mark.parametrize("world,tile,balanced", [(2, 64, False), (3, 32, False), (8, 16, False), (3, 16, True),
                                                 (8, 32, True)])
def test_tile_sharded_ranks_reassemble_the_frame(mode, world, tile, balanced):
    """Each simulated rank renders only its tiles (t % world == rank, or the cost-balanced
    owner map of scheduler.balanced_tile_owners set with nsdf_cuda_set_tile_owners) into its
    own device framebuffer, exactly as bench.py's ranks do; the packed-tile gather
    (scheduler.py) is emulated by the same index sets.  The union must equal the single-GPU
    frame bitwise."""
    import torch
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.scheduler import balanced_tile_owners, owned_pixels, tile_costs
    from conftest import records_np
    ctx = Context(0, mode)
    ds = DeviceSequence(ctx, _seq())
    W, H = 200, 120
    owners = None
    if balanced:
        rec = records_np(ctx.trace_image(ds.levels(), standard_camera(W, H), TraceConfig((20, 5, 5)))[0])
        costs = tile_costs(rec["iters"], rec["hit"], W, H, tile, [64, 128, 256], 256)
        owners = balanced_tile_owners(costs, world)
        ctx.set_tile_owners(owners)
    cam = standard_camera(W, H)
    cfg = TraceConfig((20, 5, 5))
    shade = ShadeConfig(specular=0.3)
    n = W * H

    def bufs():
        return (torch.full((3 * n,), -1.0, device="cuda"), torch.full((n,), -1.0, device="cuda"),
                torch.full((n,), 7, dtype=torch.uint8, device="cuda"))

    full = bufs()
    ctx.render_device(ds.levels(), cam, cfg, shade, *(b.data_ptr() for b in full))
    torch.cuda.synchronize()
    out = bufs()
    for rank in range(world):
        mine = bufs()
        ctx.render_device(ds.levels(), cam, cfg, shade, *(b.data_ptr() for b in mine), tile_size=tile,
                          tile_rank=rank, tile_world=world)
        torch.cuda.synchronize()
        idx = torch.from_numpy(owned_pixels(W, H, tile, rank, world, owners)).cuda()
        # untouched pixels keep the sentinel, owned pixels are written
        others = torch.ones(n, dtype=torch.bool, device="cuda")
        others[idx] = False
        assert bool((mine[2][others] == 7).all())
        out[0].view(-1, 3)[idx] = mine[0].view(-1, 3)[idx]
        out[1][idx] = mine[1][idx]
        out[2][idx] = mine[2][idx]
    for a, b in zip(out, full):
        assert torch.equal(a.view(torch.uint8) if a.dtype != torch.uint8 else a,
                           b.view(torch.uint8) if b.dtype != torch.uint8 else b)
    if balanced:  # a map for another tiling is a config error, not a silent mis-render
        from paper_2201_09147_b200.abi import NsdfError
        with pytest.raises(NsdfError):
            ctx.render_device(ds.levels(), cam, cfg, shade, *(b.data_ptr() for b in bufs()), tile_size=tile * 2,
                              tile_rank=0, tile_world=world)
        ctx.set_tile_owners(None)
    ctx.close()


def test_fast_mode_is_deterministic():
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    ctx = Context(0, "fp16")
    ds = DeviceSequence(ctx, _seq())
    cam = standard_camera(256, 160)
    a = ctx.render(ds.levels(), cam, TraceConfig((20, 5, 5)), ShadeConfig(specular=0.3))
    b = ctx.render(ds.levels(), cam, TraceConfig((20, 5, 5)), ShadeConfig(specular=0.3))
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    ctx.close()


def test_stats_match_records(ctx):
    """Per-level evaluation counts (the FLOP source) equal the HitRecords' iterations_used."""
    from conftest import records_np
    from paper_2201_09147_b200.abi import TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    ds = DeviceSequence(ctx, _seq())
    recs, st = ctx.trace_image(ds.levels(), standard_camera(160, 90), TraceConfig((20, 5, 5)))
    r = records_np(recs)
    for j in range(3):
        assert st.evals[j] == int(r["iters"][:, j].astype(np.int64).sum())
    assert st.hits == int(r["hit"].sum())


def test_error_conventions(ctx):
    """ErrorKinds and messages of the reference's validation (trace.cpp:10-23,
    camera.cpp:7-18, mlp.cpp:13-39, nesting.cpp:56-69, shade.cpp:47-65)."""
    from paper_2201_09147_b200.abi import Camera, Level, NsdfError, ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import DeviceSequence
    from paper_2201_09147_b200.manifest import Analytic, Net, Sequence
    ds = DeviceSequence(ctx, Sequence([Analytic("sphere", {"r": 1.0}), Analytic("sphere", {"r": 0.9})],
                                      [0.1, 0.05], ["a", "b"]))
    cam = standard_camera(16, 16)
    cases = [
        (lambda: ctx.trace_image(ds.levels(), cam, TraceConfig((0, 0))), "config", "all iteration budgets are zero"),
        (lambda: ctx.trace_image(ds.levels(), cam, TraceConfig((5,))), "config", "got 1 budgets for 2 levels"),
        (lambda: ctx.trace_image(ds.levels(), cam, TraceConfig((5, -1))), "config", "non-negative"),
        (lambda: ctx.trace_image(ds.levels(), cam, TraceConfig((5, 5), eps_stop=0.0)), "config", "eps_stop"),
        (lambda: ctx.trace_image(ds.levels(), Camera(width=0), TraceConfig((5, 5))), "config", "image size"),
        (lambda: ctx.trace_image(ds.levels(), Camera((0, 0, 3), (0, 0, 3)), TraceConfig((5, 5))), "config",
         "coincide"),
        (lambda: ctx.trace_image(ds.levels(), Camera((0, 3, 0), (0, 0, 0)), TraceConfig((5, 5))), "config",
         "parallel"),
        (lambda: ctx.trace_image([Level(ds.handles[0], 0.0, 0.1), Level(ds.handles[1], 0.0, -1.0)], cam,
                                 TraceConfig((5, 5))), "validation", "not positive"),
        (lambda: ctx.render(ds.levels(), cam, TraceConfig((5, 5)), ShadeConfig(lights=())), "contract",
         "at least one directional light"),
        (lambda: ctx.render(ds.levels(), cam, TraceConfig((5, 5)), ShadeConfig(), 1, 7), "config", "out of range"),
        (lambda: ctx.upload(Net.from_layers([(np.zeros((4, 3)), np.zeros(4)), (np.zeros((2, 4)), np.zeros(2))])),
         "validation", "single output"),
        (lambda: ctx.eval(ds.handles[0], np.zeros((2, 5), np.float32)), "contract", "rows are required"),
    ]
    for fn, kind, text in cases:
        with pytest.raises(NsdfError) as e:
            fn()
        assert e.value.kind == kind and text in str(e.value), (kind, text, str(e.value))


def test_empty_and_ragged_batches(ctx):
    net = random_net(64, 1, seed=4)
    h = ctx.upload(net)
    d, g = ctx.eval_grad(h, np.zeros((3, 0), np.float32))
    assert d.shape == (0,) and g.shape == (3, 0)
    for k in (1, 127, 128, 129, 4097):
        pts = np.random.default_rng(k).uniform(-1, 1, (3, k)).astype(np.float32)
        d1, g1 = ctx.eval_grad(h, pts)
        assert d1.shape == (k,) and np.isfinite(d1).all() and np.isfinite(g1).all()


def _device_count():
    import torch
    return torch.cuda.device_count()


def _assert_paths(st, n_levels, mode, normals=True):
    from paper_2201_09147_b200.abi import PATH_SIMT, PATH_TCGEN05
    want = PATH_TCGEN05 if mode == "fp16" else PATH_SIMT
    assert list(st.level_path)[:n_levels] == [want] * n_levels, list(st.level_path)
    if normals:
        assert st.normals_path == want


def _render_multi_case(mode, devices, tile, replicate):
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence, render_multi
    seq = _seq()
    ctxs = [Context(d, mode) for d in devices]
    try:
        d0 = DeviceSequence(ctxs[0], seq)
        dss = [d0] + [d0.replicate(c) if replicate else DeviceSequence(c, seq) for c in ctxs[1:]]
        cam = standard_camera(200, 120)
        cfg, shade = TraceConfig((20, 5, 5)), ShadeConfig(specular=0.3)
        ref = ctxs[0].render(d0.levels(), cam, cfg, shade)
        _assert_paths(ref[3], 3, mode)
        for rep in range(2):  # the second frame reuses the peer framebuffer / events
            rgb, depth, mask, st = render_multi(ctxs, [d.levels() for d in dss], cam, cfg, shade, tile_size=tile,
                                                stats=True)
            assert np.array_equal(mask, ref[2])
            assert np.array_equal(depth.view(np.uint32), ref[1].view(np.uint32))
            assert np.array_equal(rgb.view(np.uint32), ref[0].view(np.uint32))
            assert st.hits == ref[3].hits and list(st.evals)[:3] == list(ref[3].evals)[:3]
            _assert_paths(st, 3, mode)
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
@pytest.mark.parametrize("n_ctx,tile,replicate", [(1, 32, False), (2, 32, True), (3, 17, False), (4, 8, True)])
def test_render_multi_equals_single(mode, n_ctx, tile, replicate):
    """nsdf_cuda_render_multi (N contexts, interleaved tiles, every context storing its
    pixels into ctxs[0]'s framebuffer) reproduces the single-context frame bit for bit, with
    weights uploaded per context or replicated device to device; every level reports the
    tcgen05 path in the fast mode.  Here the contexts share device 0 (the one GPU of this
    box); test_render_multi_distinct_devices runs them on distinct GPUs."""
    _render_multi_case(mode, [0] * n_ctx, tile, replicate)


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
def test_render_multi_distinct_devices(mode):
    """The same frame with one context per GPU (peer stores over NVLink into device 0's
    framebuffer, weights broadcast device to device, per-device kernel attributes): bitwise
    equal to the single-device frame, tcgen05 on every level of every device."""
    n = _device_count()
    if n < 2:
        pytest.skip("needs more than one GPU")
    _render_multi_case(mode, list(range(min(n, 8))), 32, True)


def test_replicated_field_is_independent_and_bitwise_equal():
    """nsdf_cuda_replicate_field copies the packed device image (one allocation); the
    replica evaluates bit for bit like the source and survives the source's release."""
    from paper_2201_09147_b200.engine import Context
    a, b = Context(0, "fp16"), Context(0, "fp16")
    try:
        for width, hidden in [(64, 1), (128, 2), (256, 3), (12, 2)]:
            net = random_net(width, hidden, seed=width)
            h = a.upload(net)
            pts = np.random.default_rng(width).uniform(-1, 1, (3, 5000)).astype(np.float32)
            d0, g0 = a.eval_grad(h, pts)
            r = a.replicate(h, b)
            a.release(h)
            d1, g1 = b.eval_grad(r, pts)
            assert np.array_equal(d0.view(np.uint32), d1.view(np.uint32))
            assert np.array_equal(g0.view(np.uint32), g1.view(np.uint32))
            b.release(r)
    finally:
        a.close()
        b.close()


def test_kernel_path_stats():
    """nsdf_frame_stats reports the kernel family of every traced level and of the normal
    tiles: tcgen05 in the fast mode, FFMA tiles in the oracle mode, NONE for skipped levels;
    analytic members always take the FFMA tiles."""
    from paper_2201_09147_b200.abi import PATH_NONE, PATH_SIMT, PATH_TCGEN05, ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200.manifest import Analytic, Sequence
    seq = _seq()
    cam = standard_camera(64, 48)
    for mode, want in (("fp16", PATH_TCGEN05), ("fp32", PATH_SIMT)):
        c = Context(0, mode)
        try:
            ds = DeviceSequence(c, seq)
            st = c.render(ds.levels(), cam, TraceConfig((20, 0, 5)), ShadeConfig())[3]
            assert list(st.level_path)[:3] == [want, PATH_NONE, want]
            assert st.normals_path == want and st.fallback_path == PATH_NONE
            st = c.render(ds.levels(), cam, TraceConfig((20, 5, 0)), ShadeConfig(), normal_source=1)[3]
            assert list(st.level_path)[:3] == [want, want, PATH_NONE] and st.normals_path == want
            an = DeviceSequence(c, Sequence([Analytic("sphere", {"r": 0.7})], [0.05], ["s"]))
            st = c.render(an.levels(), cam, TraceConfig((30,)), ShadeConfig())[3]
            assert st.level_path[0] == PATH_SIMT and st.normals_path == PATH_SIMT
        finally:
            c.close()


def test_every_new_context_takes_the_configuration_path():
    """The kernel launch configuration (dynamic-SMEM opt-in > 48 KB for the 128/256-wide
    tiles, occupancy) is per device: with the cache cleared before each new context, every
    context configures the kernels itself — first a small launch then a large one of the same
    kernel (f64 evaluator: 64- then 256-wide), then the reverse order in the next context, whose
    smaller request must not lower the opt-in under the cached larger one — and its frame runs
    tcgen05 on every level."""
    from paper_2201_09147_b200 import abi
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    seq = _seq()
    lib = abi.load_library()
    ref = None
    for order in ((64, 256), (256, 64), (128, 64)):
        assert lib.nsdf_cuda_reset_kernel_config() == 0
        c = Context(0, "fp16")
        try:
            for w in order:
                net = random_net(w, 1 if w == 64 else 2, seed=w)
                h = c.upload(net)
                d, g = c.eval_f64(h, np.random.default_rng(w).uniform(-1, 1, (3, 777)))
                assert np.isfinite(d).all() and np.isfinite(g).all()
            out = c.render(DeviceSequence(c, seq).levels(), standard_camera(96, 64), TraceConfig((20, 5, 5)),
                           ShadeConfig(specular=0.3))
            _assert_paths(out[3], 3, "fp16")
            if ref is None:
                ref = out
            assert np.array_equal(out[1].view(np.uint32), ref[1].view(np.uint32))
        finally:
            c.close()


def test_contexts_on_many_threads_all_run_tcgen05():
    """Contexts created and used from concurrent host threads (the launch-attribute cache is
    per device and locked): every thread's first frame runs the tcgen05 kernels (the 128- and
    256-wide ones need the > 48 KB SMEM opt-in) and all frames are identical."""
    import threading
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    seq = _seq()
    cam = standard_camera(160, 96)
    out, errs = [None] * 6, []

    def work(i):
        try:
            c = Context(0, "fp16")
            ds = DeviceSequence(c, seq)
            out[i] = c.render(ds.levels(), cam, TraceConfig((20, 5, 5)), ShadeConfig(specular=0.3))
            c.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(out))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for o in out:
        _assert_paths(o[3], 3, "fp16")
        assert np.array_equal(o[2], out[0][2])


def test_empty_light_list_matches_reference(oracle_built, tmp_path):
    """The reference checks the lights inside shade(), which render() only calls for frames
    with hits: a hit-free frame with no light is the background image; with hits it raises
    ErrorKind::contract (render.cpp:41, shade.cpp:47-49)."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import Camera, NsdfError, ShadeConfig, TraceConfig, ERR_CONTRACT
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    p = os.path.join(ASSETS, "torus_w30.nest")
    seq = _seq()
    c = Context(0, "fp32")
    try:
        ds = DeviceSequence(c, seq)
        shade = ShadeConfig(lights=(), background=(0.2, 0.3, 0.4))
        away = Camera((0, 0, 3), (0, 0, 6), (0, 1, 0), 30.0, 40, 30)   # looks away from the torus
        rgb, depth, mask, st = c.render(ds.levels(), away, TraceConfig((20, 5, 5)), shade)
        want = refshim.render(p, away, TraceConfig((20, 5, 5)), shade)
        assert st.hits == 0 and not mask.any()
        assert np.array_equal(rgb, want[0]) and np.array_equal(depth, want[1])
        toward = Camera((0, 1.5, 2), (0, 0, 0), (0, 1, 0), 50.0, 40, 30)
        with pytest.raises(NsdfError) as e:
            c.render(ds.levels(), toward, TraceConfig((20, 5, 5)), shade)
        assert e.value.status == ERR_CONTRACT and "light" in str(e.value)
        with pytest.raises(Exception):
            refshim.render(p, toward, TraceConfig((20, 5, 5)), shade)
        # the same over two contexts (render_multi) and through the split render
        from paper_2201_09147_b200.engine import render_multi
        c2 = Context(0, "fp32")
        try:
            lv = [ds.levels(), ds.replicate(c2).levels()]
            rgb2, depth2, mask2 = render_multi([c, c2], lv, away, TraceConfig((20, 5, 5)), shade, tile_size=8)
            assert np.array_equal(rgb2, want[0]) and not mask2.any()
            with pytest.raises(NsdfError) as e:
                render_multi([c, c2], lv, toward, TraceConfig((20, 5, 5)), shade, tile_size=8)
            assert e.value.status == ERR_CONTRACT
        finally:
            c2.close()
    finally:
        c.close()


def test_split_render_begin_end():
    """nsdf_cuda_render_begin / _end equal nsdf_cuda_render; one frame in flight per context
    (a second begin, or a plain render in between, is a contract error)."""
    import ctypes
    from paper_2201_09147_b200.abi import ERR_CONTRACT, FrameStats, ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence, _levels
    c = Context(0, "fp16")
    try:
        ds = DeviceSequence(c, _seq())
        cam, cfg, shade = standard_camera(120, 80), TraceConfig((40, 20, 20)), ShadeConfig(specular=0.3)
        ref = c.render(ds.levels(), cam, cfg, shade)
        lv, m = _levels(ds.levels())
        assert c.lib.nsdf_cuda_render_begin(c._ctx, lv, m, ctypes.byref(cam), ctypes.byref(cfg), ctypes.byref(shade),
                                            0, -1) == 0
        assert c.lib.nsdf_cuda_render_begin(c._ctx, lv, m, ctypes.byref(cam), ctypes.byref(cfg), ctypes.byref(shade),
                                            0, -1) == ERR_CONTRACT
        n = cam.width * cam.height
        rgb, depth, mask = np.zeros(3 * n, np.float32), np.zeros(n, np.float32), np.zeros(n, np.uint8)
        fp = ctypes.POINTER(ctypes.c_float)
        st = FrameStats()
        assert c.lib.nsdf_cuda_render_end(c._ctx, rgb.ctypes.data_as(fp), depth.ctypes.data_as(fp),
                                          mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), ctypes.byref(st)) == 0
        assert np.array_equal(rgb.reshape(ref[0].shape), ref[0]) and np.array_equal(mask.reshape(ref[2].shape), ref[2])
        assert c.lib.nsdf_cuda_render_end(c._ctx, rgb.ctypes.data_as(fp), depth.ctypes.data_as(fp),
                                          mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), None) == ERR_CONTRACT
    finally:
        c.close()


@pytest.mark.parametrize("mode", ["fp32", "fp16"])
def test_chunked_host_batches_equal_small_batches(mode):
    """The host-buffer batch API pipelines large batches in 65536-column chunks (H2D / tiles /
    D2H on separate streams, double-buffered): results equal per-point evaluation in small
    batches bit for bit (per-point work is batch-independent), for eval/grad with 3- and 4-row
    points and for the normal map with fallback normals and its counters."""
    from paper_2201_09147_b200.engine import Context
    c = Context(0, mode)
    try:
        for net, rows in ((random_net(128, 2, seed=8), 3), (random_net(64, 1, seed=9, input_dim=4), 4)):
            h = c.upload(net)
            k = 3 * 65536 + 777  # four chunks, the last one ragged
            pts = np.random.default_rng(rows).uniform(-1, 1, (rows, k)).astype(np.float32)
            d, g = c.eval_grad(h, pts, time=0.25)
            v_only = c.eval(h, pts, time=0.25)
            for lo in range(0, k, 50000):
                hi = min(k, lo + 50000)
                d1, g1 = c.eval_grad(h, np.ascontiguousarray(pts[:, lo:hi]), time=0.25)
                assert np.array_equal(d[lo:hi], d1) and np.array_equal(g[:, lo:hi], g1)
            assert np.array_equal(v_only, d)
        h = c.upload(random_net(64, 1, seed=10))
        k = 2 * 65536 + 4099
        pts = np.random.default_rng(3).uniform(-1, 1, (3, k)).astype(np.float32)
        fb = np.random.default_rng(4).normal(size=(3, k)).astype(np.float32)
        n_all, o_all, f_all = c.normal_map(h, pts, 0.05, fallback=fb)
        o_sum = f_sum = 0
        for lo in range(0, k, 40000):
            hi = min(k, lo + 40000)
            n1, o1, f1 = c.normal_map(h, np.ascontiguousarray(pts[:, lo:hi]), 0.05,
                                      fallback=np.ascontiguousarray(fb[:, lo:hi]))
            assert np.array_equal(n_all[:, lo:hi], n1)
            o_sum, f_sum = o_sum + o1, f_sum + f1
        assert (o_all, f_all) == (o_sum, f_sum) and o_all > 0
    finally:
        c.close()
