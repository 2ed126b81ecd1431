"""Full-size parity report of the fast mode (split-fp16 tcgen05) against the reference
renderer (oracle/_ref, AVX2, all host cores) on BASELINE.json's configurations, with every
tolerance the north star names (SURVEY.md §8d "Parity metrics"):

  (i)   hit/miss mask agreement (>= 99.9%)
  (ii)  |t_gpu - t_cpu| on common hits (<= 1e-3: max, p99.9, p99)
  (iii) normal angle on common hits (<= 0.5 deg): end to end (each side's normal at its own
        hit point) and at identical points (the reference's hit points) to isolate the
        normal kernel
plus the oracle mode's bitwise agreement (mask, depth bits) for the same frame.

    python tools/parity_report.py [--out profiles/r2_parity.json]
Test/measurement infrastructure: reads the reference through oracle/refshim only.
"""
import argparse
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import refshim  # noqa: E402
from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera  # noqa: E402
from paper_2201_09147_b200.engine import Context, DeviceSequence  # noqa: E402
from paper_2201_09147_b200.manifest import load_manifest  # noqa: E402

TORUS = os.path.join(ROOT, "assets", "torus_w30.nest")
TORUS3 = os.path.join(ROOT, "assets", "torus3.nest")
BLEND = os.path.join(ROOT, "assets", "blend4d_w30.nest")
# (name, manifest, members, resolution, budgets, time, normal source: 0 own / 1 mapped)
CASES = [
    ("config2 1080p torus3 (40,20,20) [headline]", TORUS3, None, (1920, 1080), (40, 20, 20), 0.0, 0),
    ("config2 1080p torus3 (20,5,5) [speed setting]", TORUS3, None, (1920, 1080), (20, 5, 5), 0.0, 0),
    ("config2 1080p torus_w30 omega0=30 (40,20,20)", TORUS, None, (1920, 1080), (40, 20, 20), 0.0, 0),
    ("config1 512x512 256x3 omega0=30 (40)", TORUS, [2], (512, 512), (40,), 0.0, 0),
    ("config3 1080p torus3 64x1 (40,0), normals mapped from 256x3", TORUS3, [0, 2], (1920, 1080), (40, 0), 0.0, 1),
    ("config5 4K slice t=0.5 omega0=30 (20,10)", BLEND, None, (3840, 2160), (20, 10), 0.5, 0),
]


def sub_manifest(path, members):
    """A .nest listing only `members` of `path` (absolute weight paths) for the reference."""
    if members is None:
        return path, None
    with open(path) as f:
        j = json.load(f)
    base = os.path.dirname(path)
    j["fields"] = [dict(j["fields"][i], weights=os.path.join(base, j["fields"][i]["weights"])) for i in members]
    j["deltas"] = [j["deltas"][i] for i in members]
    fd, tmp = tempfile.mkstemp(suffix=".nest")
    with os.fdopen(fd, "w") as f:
        json.dump(j, f)
    return tmp, tmp


def records(recs):
    n = len(recs)
    hit = np.fromiter((r.hit for r in recs), np.int32, n)
    t = np.fromiter((r.t for r in recs), np.float32, n)
    p = np.array([tuple(r.point) for r in recs], np.float32).reshape(n, 3)
    return hit, t, p


def angle_deg(g0, g1):
    # float64 (an f32 dot of unit vectors quantizes angles near 0 to ~0.03 deg); atan2 form
    g0, g1 = g0.astype(np.float64), g1.astype(np.float64)
    cr = np.cross(g0.T, g1.T).T
    return np.degrees(np.arctan2(np.linalg.norm(cr, axis=0), (g0 * g1).sum(0)))


def stats(x):
    if x.size == 0:
        return {"max": 0.0, "p99.9": 0.0, "p99": 0.0}
    return {"max": float(x.max()), "p99.9": float(np.percentile(x, 99.9)), "p99": float(np.percentile(x, 99))}


def gbuffer_case():
    """Config 4: the torus-mesh G-buffer at 2560x1440 -> 256x3 neural normal map
    (neural_normal_map semantics, shade.cpp:8-42) on identical points."""
    import torch
    from paper_2201_09147_b200.meshes import torus_mesh
    man, tmp = sub_manifest(TORUS, [2])
    try:
        seq = load_manifest(TORUS).subsequence([2])
        ctx = Context(0, "fp16")
        cam = standard_camera(2560, 1440)
        n = cam.width * cam.height
        pos = torch.zeros(3 * n, dtype=torch.float32, device="cuda")
        mask = torch.zeros(n, dtype=torch.uint8, device="cuda")
        v, t = torus_mesh()
        ctx.raycast_mesh(cam, v, t, pos.data_ptr(), mask.data_ptr())
        pts = pos.view(3, n)[:, mask.bool()].contiguous().cpu().numpy()
        delta = float(seq.deltas[0])
        ds = DeviceSequence(ctx, seq)
        g_nrm, g_out, g_fb = ctx.normal_map(ds.handles[0], pts, delta)
        r_nrm, r_out, r_fb = refshim.normal_map(man, 0, pts, delta)
        ctx.close()
        ang = angle_deg(g_nrm, r_nrm)
        return {"case": "config4 2560x1440 mesh G-buffer -> 256x3 normal map (identical points)",
                "points": int(pts.shape[1]), "outside_count": [int(g_out), int(r_out)],
                "fallback_count": [int(g_fb), int(r_fb)], "normal_deg_same_points": stats(ang),
                "pass": bool(stats(ang)["p99.9"] <= 0.5 and g_fb == r_fb)}
    finally:
        os.unlink(tmp)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    refshim.set_backend("avx2")
    report = []
    for name, path, members, (w, h), budgets, tm, src in CASES:
        man, tmp = sub_manifest(path, members)
        try:
            seq = load_manifest(path)
            if members is not None:
                seq = seq.subsequence(members)
            normal_idx = len(budgets) - 1 if src == 1 else max(j for j, b in enumerate(budgets) if b > 0)
            cam, cfg, shade = standard_camera(w, h), TraceConfig(budgets), ShadeConfig(specular=0.3)
            rr, rd, rm, _ = refshim.render(man, cam, cfg, shade, src, -1, time=tm)
            rh, rt, rp = records(refshim.trace_image(man, cam, cfg, time=tm))
            row = {"case": name, "pixels": w * h, "ref_hits": int(rm.sum())}
            for mode in ("fp32", "fp16"):
                ctx = Context(0, mode)
                ds = DeviceSequence(ctx, seq)
                lv = ds.levels(time=tm)
                gr, gd, gm, _ = ctx.render(lv, cam, cfg, shade, src, -1)
                if mode == "fp32":
                    row["oracle_mode_bitwise"] = bool(np.array_equal(gm, rm) and
                                                      np.array_equal(gd.view(np.uint32), rd.view(np.uint32)))
                    ctx.close()
                    continue
                both = (gm == 1) & (rm == 1)
                row["mask_agreement"] = float(np.mean(gm == rm))
                row["dt"] = stats(np.abs(gd - rd)[both])
                recs, _ = ctx.trace_image(lv, cam, cfg)
                gh, gt, gp = records(recs)
                common = (gh == 1) & (rh == 1)
                hnd = ds.handles[normal_idx]
                # end to end: each side's gradient at its own hit point
                _, g_gpu = ctx.eval_grad(hnd, gp[common].T.copy(), time=tm)
                _, g_ref = refshim.field_eval(man, normal_idx, rp[common].T.copy(), time=tm)
                row["normal_deg_end_to_end"] = stats(angle_deg(g_gpu, g_ref))
                # identical points: the normal kernel alone
                _, g_gpu_same = ctx.eval_grad(hnd, rp[common].T.copy(), time=tm)
                row["normal_deg_same_points"] = stats(angle_deg(g_gpu_same, g_ref))
                row["pass"] = bool(row["mask_agreement"] >= 0.999 and row["dt"]["p99.9"] <= 1e-3 and
                                   row["normal_deg_end_to_end"]["p99.9"] <= 0.5)
                ctx.close()
            report.append(row)
            print(json.dumps(row), flush=True)
        finally:
            if tmp:
                os.unlink(tmp)
    report.append(gbuffer_case())
    print(json.dumps(report[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
