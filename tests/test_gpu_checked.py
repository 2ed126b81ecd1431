"""GPU memory-safety evidence without compute-sanitizer (closed on this GPU pool): the
bounds-checked build of the engine (paper_2201_09147_b200/_checked/libnsdf_cuda.so,
-DNSDF_CHECKED=1) checks on the device every list index, ray slot, CTA-staged compaction
append, list write and framebuffer pixel the kernels compute — the persistent trace's claimed
list items and staged appends included — counting (and skipping) any out-of-bounds access.
A workload covering the engine's index paths runs on it in a fresh process: full and tile-
sharded renders (static and cost-balanced owners), renders of random views at ragged image
sizes, render_multi, ragged trace_rays batches,
batch evaluation, the normal map and the mesh normal map, in the fast (tcgen05) and the
FP32 oracle modes.  Every frame must equal the normal build's bit for bit and the violation
count must be zero."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ASSETS, ROOT

pytestmark = pytest.mark.gpu

CHECKED = os.path.join(ROOT, "paper_2201_09147_b200", "_checked", "libnsdf_cuda.so")

WORKLOAD = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, os.path.join(sys.argv[1], "tools"))
from paper_2201_09147_b200 import abi
from paper_2201_09147_b200.abi import Camera, ShadeConfig, TraceConfig, standard_camera
from paper_2201_09147_b200.engine import Context, DeviceSequence, render_multi
from paper_2201_09147_b200.manifest import load_manifest
from paper_2201_09147_b200.meshes import torus_mesh
from paper_2201_09147_b200.scheduler import balanced_tile_owners, tile_costs
from conftest_free_records import records_np
import ctypes, torch
out = {"lib": abi.LIB_PATH, "digests": {}}
def digest(a):
    a = np.ascontiguousarray(a)
    return float(a.astype(np.float64).sum()), int(a.reshape(-1).view(np.uint8).astype(np.int64).sum() % 1000003)
seq = load_manifest(os.path.join(sys.argv[1], "assets", "torus3.nest"))
for mode in ("fp16", "fp32"):
    c = Context(0, mode)
    ds = DeviceSequence(c, seq)
    cam = standard_camera(480, 270) if mode == "fp16" else standard_camera(160, 96)
    for b in ((40, 20, 20), (20, 5, 5), (0, 0, 40), (30, 0, 0)):
        rgb, depth, mask, st = c.render(ds.levels(), cam, TraceConfig(b), ShadeConfig(specular=0.3))
        out["digests"][f"{mode} render {b}"] = digest(rgb) + digest(depth) + digest(mask)
        rgb, depth, mask, st = c.render(ds.levels(), cam, TraceConfig(b), ShadeConfig(), normal_source=1)
        out["digests"][f"{mode} mapped {b}"] = digest(rgb) + digest(depth)
    rng = np.random.default_rng(5)
    for k in range(6):  # ragged image sizes, random views and budgets
        w, h = int(rng.integers(1, 151)), int(rng.integers(1, 151))
        d = rng.normal(size=3)
        rc = Camera(tuple(d / np.linalg.norm(d) * rng.uniform(1.6, 4.0)), (0, 0, 0), (0, 1, 0), float(rng.uniform(20, 90)), w, h)
        b = tuple(int(x) for x in rng.integers(0, 31, 3))
        b = b if any(b) else (0, 0, 20)
        rgb, depth, mask, st = c.render(ds.levels(), rc, TraceConfig(b), ShadeConfig(specular=0.5), normal_source=k % 2)
        out["digests"][f"{mode} random {k}"] = digest(rgb) + digest(depth) + digest(mask)
    n = cam.width * cam.height
    rec = records_np(c.trace_image(ds.levels(), cam, TraceConfig((40, 20, 20)))[0])
    for world, tile, bal in ((3, 16, False), (8, 32, True)):
        owners = balanced_tile_owners(tile_costs(rec["iters"], rec["hit"], cam.width, cam.height, tile, [64, 128, 256],
                                                 256), world) if bal else None
        c.set_tile_owners(owners)
        fbs = [torch.zeros(3 * n, device="cuda"), torch.zeros(n, device="cuda"), torch.zeros(n, dtype=torch.uint8, device="cuda")]
        for r in range(world):
            c.render_device(ds.levels(), cam, TraceConfig((40, 20, 20)), ShadeConfig(), *(x.data_ptr() for x in fbs),
                            tile_size=tile, tile_rank=r, tile_world=world)
        torch.cuda.synchronize()
        out["digests"][f"{mode} tiles {world}"] = digest(fbs[0].cpu().numpy()) + digest(fbs[2].cpu().numpy())
        c.set_tile_owners(None)
    ctxs = [c] + [Context(0, mode) for _ in range(2)]
    dss = [ds] + [ds.replicate(x) for x in ctxs[1:]]
    m = render_multi(ctxs, [d.levels() for d in dss], cam, TraceConfig((40, 20, 20)), ShadeConfig(), tile_size=16)
    out["digests"][f"{mode} multi"] = digest(m[0]) + digest(m[2])
    for x in ctxs[1:]:
        x.close()
    for k in (1, 127, 129, 4097, 70000):
        rays = np.random.default_rng(k).uniform(-1, 1, (k, 6)).astype(np.float32)
        rays[:, :3] *= 3.0
        rays[:, 3:] /= np.linalg.norm(rays[:, 3:], axis=1, keepdims=True)
        r2 = records_np(c.trace_rays(ds.levels(), TraceConfig((20, 10, 10)), rays))
        out["digests"][f"{mode} rays {k}"] = digest(r2["t"])
    pts = np.random.default_rng(1).uniform(-1, 1, (3, 100003)).astype(np.float32)
    d, g = c.eval_grad(ds.handles[2], pts)
    out["digests"][f"{mode} eval"] = digest(d) + digest(g)
    nrm, o, f = c.normal_map(ds.handles[2], pts, 0.05)
    out["digests"][f"{mode} normal_map"] = digest(nrm) + (o, f)
    v, _ = torus_mesh()
    mn, cnt = c.map_normals_to_mesh(ds.handles[2], v, 0.05)
    out["digests"][f"{mode} mesh"] = digest(mn) + tuple(cnt)
    cnt_ = ctypes.c_uint64(); site = ctypes.c_int32(); val = ctypes.c_int32(); bnd = ctypes.c_int32(); chk = ctypes.c_int32()
    abi.check(c.lib.nsdf_cuda_check_report(c._ctx, 1, ctypes.byref(cnt_), ctypes.byref(site), ctypes.byref(val),
                                           ctypes.byref(bnd), ctypes.byref(chk)))
    out[f"{mode} violations"] = [cnt_.value, site.value, val.value, bnd.value]
    out["checked_build"] = chk.value
    # positive control: one deliberate violation must be seen (checked build only)
    abi.check(c.lib.nsdf_cuda_check_selftest(c._ctx))
    abi.check(c.lib.nsdf_cuda_check_report(c._ctx, 1, ctypes.byref(cnt_), ctypes.byref(site), ctypes.byref(val),
                                           ctypes.byref(bnd), ctypes.byref(chk)))
    out[f"{mode} selftest"] = [cnt_.value, site.value, val.value, bnd.value]
    c.close()
print(json.dumps(out))
'''


def _run(lib):
    env = dict(os.environ)
    if lib:
        env["NSDF_CUDA_LIB"] = lib
    else:
        env.pop("NSDF_CUDA_LIB", None)
    r = subprocess.run([sys.executable, "-c", WORKLOAD, ROOT], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_checked_build_runs_clean_and_matches():
    if not os.path.exists(CHECKED):
        pytest.skip("checked build missing (build.build_cuda(checked=True))")
    if not os.path.exists(os.path.join(ASSETS, "torus3.nest")):
        pytest.skip("fixture missing")
    checked = _run(CHECKED)
    normal = _run(None)
    assert checked["lib"].endswith("_checked/libnsdf_cuda.so") and checked["checked_build"] == 1
    assert normal["checked_build"] == 0
    for mode in ("fp16", "fp32"):
        assert checked[f"{mode} violations"][0] == 0, checked[f"{mode} violations"]
        assert checked[f"{mode} selftest"] == [1, 2, -1, 1] and normal[f"{mode} selftest"][0] == 0
    assert checked["digests"] == normal["digests"]
