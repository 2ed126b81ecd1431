#!/usr/bin/env python3
"""Benchmark: Mrays/s & ms/frame at 1080p, multiscale sphere tracing + analytic normals.

Default workload (BASELINE.json configs[1]): the nested 3-level SIREN
sequence 64x1 > 128x2 > 256x3 (assets/torus3.nest: the reference trainer's fit of the torus,
omega0 = 10, Prop-2 certified; tools/build_assets.sh) traced at 1920x1080 from the standard
camera with budgets (40,20,20) — the setting whose frame converges (hits within ~5% of
(40,40,40); `frame_quality` reports the hit fraction and the image MSE against that frame) —
own analytic normals from the 256x3 net, Lambert + Blinn-Phong (specular 0.3, the `nsdf
bench` shading, nsdf_main.cpp:446).  The paper-style speed setting (20,5,5) is timed beside
it (`speed_setting`, with its MSE).  One step = one whole frame: rays -> multiscale trace ->
normals -> shade -> framebuffer.  Weights are resident (uploaded once; broadcast over NCCL for
N>1); the per-frame working set (ray state + lists + framebuffer, ~160 MB at 1080p) exceeds
the 126 MB L2, so no flush is needed between steps.

--config 1|3|4|5 selects the other BASELINE workloads (1: single 256x3 omega0 = 30 at 512^2;
3: neural normal mapping 64x1 (40,0) + 256x3 normals at 1080p; 4: torus-mesh G-buffer ->
256x3 normals at 2560x1440; 5: animated 4-D 64x1 > 128x2 blend (omega0 = 30), 120 frames at
3840x2160, frames sharded across ranks).

N > 1 (torchrun, the frame/tile scheduler of SURVEY.md §8e): by default (--shard tiles) every
frame is split into image tiles interleaved across the ranks (tile t -> rank t % N), each
rank's shading kernels storing its pixels into rank 0's framebuffer over NVLink peer memory
(strong scaling; ms_per_frame is the latency of a whole frame); --shard frames shards the
frame stream instead (every rank renders whole frames, no data-path collective, weak scaling)
and times the tile split beside it as `strong_scaling`; config 5's animation always shards
frames.  --impl reference times the reference's own CPU renderer (oracle/_ref/libnsdf_ref.so,
all host threads) on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(1, os.path.join(ROOT, "tools"))

TORUS = os.path.join(ROOT, "assets", "torus_w30.nest")   # omega0 = 30 (PyTorch fit, certified by the reference)
TORUS3 = os.path.join(ROOT, "assets", "torus3.nest")      # reference trainer, omega0 = 10 (tools/build_assets.sh)
BLEND = os.path.join(ROOT, "assets", "blend4d_w30.nest")
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

CONFIGS = {
    1: dict(manifest=TORUS, members=[2], budgets="40", normals="own", res=(512, 512),
            metric="Mrays/s & ms/frame at 512x512 (single 256x3 SIREN ST + analytic normals)",
            desc="config1: single 256x3 SIREN (torus, omega0=30), 512x512, budgets ({b}), own analytic normals"),
    2: dict(manifest=TORUS3, members=[0, 1, 2], budgets="40,20,20", speed_budgets="20,5,5", normals="own",
            res=(1920, 1080), metric="Mrays/s & ms/frame at 1080p (multiscale ST + analytic normals)",
            desc="config2: nested 64x1>128x2>256x3 SIREN (torus, reference trainer, omega0=10), 1920x1080, "
                 "budgets ({b}), own analytic normals, specular 0.3"),
    3: dict(manifest=TORUS3, members=[0, 2], budgets="40,0", normals="mapped", res=(1920, 1080),
            metric="Mrays/s & ms/frame at 1080p (neural normal mapping: 64x1 traced, 256x3 normals)",
            desc="config3: 64x1 traced with budgets ({b}), normals mapped from 256x3 (torus3), 1920x1080"),
    4: dict(manifest=TORUS3, members=[2], kind="gbuffer", res=(2560, 1440),
            metric="Mnormals/s & ms/frame at 2560x1440 (mesh G-buffer -> neural normals)",
            desc="config4: torus mesh (96x48 quads) G-buffer at 2560x1440 -> 256x3 neural normal map"),
    5: dict(manifest=BLEND, members=[0, 1], budgets="20,10", normals="own", res=(3840, 2160), frames=120,
            metric="Mrays/s & ms/frame at 3840x2160 (animated 4-D SIREN, 120 frames)",
            desc="config5: animated 4-D 64x1>128x2 blend, 120 frames t=i/119 at 3840x2160, budgets ({b})"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--mode", default=os.environ.get("NSDF_MODE", "fp16"), choices=["fp16", "fp16low", "fp32"])
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--height", type=int, default=0)
    ap.add_argument("--budgets", default="")
    ap.add_argument("--tile", type=int, default=32, help="image tile edge of the N>1 tile interleave")
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N>1 frame assembly: peer stores into rank 0's framebuffer, or an NCCL tile gather")
    ap.add_argument("--inflight", type=int, default=0,
                    help="frames in flight (engine contexts on their own streams); 1 = strictly serial frames; "
                         "0 = 3, or 5 for tile-sharded frames on >= 4 GPUs (smaller shares leave more "
                         "level-tail idle time to overlap: tools/shardsim.py, N=8: 6.19x -> 6.38x)")
    ap.add_argument("--shard", default="tiles", choices=["frames", "tiles"],
                    help="N > 1, single-frame configs 1-4: 'tiles' (default, the headline) = the ranks split every "
                         "frame's image tiles and assemble it in rank 0's framebuffer (strong scaling, ms_per_frame "
                         "is the latency of one whole frame); 'frames' = every rank renders whole frames of the "
                         "frame stream (weak scaling; frames stay on their rank) and a tile-sharded pass is timed "
                         "beside it as strong_scaling.  Config 5 (animation) always shards frames")
    ap.add_argument("--balance", type=int, default=1,
                    help="N > 1 tile split: 1 = cost-balanced tile owners from one traced frame, 0 = tile t -> rank t %% N")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true",
                    help="skip the frame-quality renders and the (20,5,5) speed-setting line of config 2")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    args.width = args.width or cfg["res"][0]
    args.height = args.height or cfg["res"][1]
    args.budgets = args.budgets or cfg.get("budgets", "")
    args.normals = cfg.get("normals", "own")
    args.cfg = cfg
    return args


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return PEAKS_FALLBACK, "fallback"


def ncu_traffic(gbuffer: bool):
    """DRAM bytes per launch of the roofline kernel(s) from the committed `ncu --set full`
    capture (profiles/*_traffic.json, tools/summarize_profile.py): the three persistent
    trace-level kernels of one frame (config 2), or None when no capture matches."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files or gbuffer:
        return None, None
    d = json.load(open(files[-1]))
    sel = {k: v for k, v in d["dram_bytes_per_launch"].items() if re.match(r"tc_mlp_kernel<\d+, 0, \d, \d, \d, 1(, \d)*>", k)}
    if not sel:
        return None, None
    return sum(sel.values()), f"DRAM read+write bytes of the {len(sel)} trace-level launches of one frame, " \
                             f"ncu --set full ({d['source']})"


def ncu_kernel_traffic(prefix: str):
    """DRAM bytes per launch of one kernel (name prefix) from the committed ncu capture."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files:
        return None
    d = json.load(open(files[-1]))
    sel = [v for k, v in d["dram_bytes_per_launch"].items() if k.startswith(prefix)]
    return sel[0] if len(sel) == 1 else None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi can take seconds to start on a fresh box: do not open the timed
            # region before it is sampling, or the window sees no samples at all
            deadline = time.time() + 15.0
            while not self.samples and time.time() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")][1:]))

    def mark(self, which):
        setattr(self, which, time.time())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        """Samples taken inside the timed window [t0, t1] (widened to the nearest samples
        when the window is shorter than the 20 ms sampling period)."""
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", time.time())
        inside = [s for ts, s in self.samples if t0 <= ts <= t1]
        window = "timed region"
        if not inside and self.samples:
            near = sorted(self.samples, key=lambda x: min(abs(x[0] - t0), abs(x[0] - t1)))[:3]
            inside = [s for _, s in near]
            window = "nearest samples (timed region shorter than the sampling period)"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in inside if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in inside if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in inside for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "window": window}


def check_paths(stats, budgets, mode):
    """Every traced level and the normal tiles must have run the kernel family of the mode
    (tcgen05 in the fast modes): a bench line measured on another path is invalid."""
    from paper_2201_09147_b200.abi import PATH_NONE, PATH_SIMT, PATH_TCGEN05
    want = PATH_SIMT if mode == "fp32" else PATH_TCGEN05
    got = [int(stats.level_path[j]) for j in range(len(budgets))]
    exp = [want if b > 0 else PATH_NONE for b in budgets]
    if got != exp or (stats.hits and int(stats.normals_path) != want):
        raise SystemExit(f"kernel path check failed: levels {got} (expected {exp}), normals {int(stats.normals_path)}")
    return got


def sub_manifest(args):
    """A .nest listing the selected members (absolute weight paths) for the reference."""
    with open(args.cfg["manifest"]) as f:
        j = json.load(f)
    base = os.path.dirname(args.cfg["manifest"])
    members = args.cfg["members"]
    j["fields"] = [dict(j["fields"][i], weights=os.path.join(base, j["fields"][i]["weights"])) for i in members]
    j["deltas"] = [j["deltas"][i] for i in members]
    fd, path = tempfile.mkstemp(suffix=".nest")
    with os.fdopen(fd, "w") as f:
        json.dump(j, f)
    return path


def workload_text(args):
    return args.cfg["desc"].format(b=args.budgets)


def f8_hidden_layers(m):
    """Hidden layers of member m whose split-precision correction terms run as one E4M3 MMA
    (the upload policy of capi.cu: 256-wide nets at omega0 <= 15, or NSDF_TC_E4M3=0/1)."""
    if getattr(m, "width", 0) != 256 or not hasattr(m, "omega0"):
        return 0
    env = os.environ.get("NSDF_TC_E4M3")
    on = (env != "0") if env else m.omega0 <= 15.0
    return m.hidden_blocks if on else 0


def frame_flops(seq, stats, normal_idx):
    """Algorithmic FLOPs of one frame: 2 x MACs, no credit for bias/sine."""
    trace = sum(int(stats.evals[j]) * 2 * seq.members[j].macs_forward() for j in range(len(seq.members)))
    normals = int(stats.normal_evals) * 2 * seq.members[normal_idx].macs_normal()
    normals += int(stats.fallback_evals) * 2 * seq.members[-1].macs_normal()
    return trace, normals


def gbuffer_points(ctx, args):
    """Device G-buffer of the torus mesh: hit positions (3 x k, device tensor)."""
    import torch
    from paper_2201_09147_b200.abi import standard_camera
    from paper_2201_09147_b200.meshes import torus_mesh
    cam = standard_camera(args.width, args.height)
    n = args.width * args.height
    pos = torch.zeros(3 * n, dtype=torch.float32, device="cuda")
    mask = torch.zeros(n, dtype=torch.uint8, device="cuda")
    v, t = torus_mesh()
    ctx.raycast_mesh(cam, v, t, pos.data_ptr(), mask.data_ptr())
    return pos.view(3, n)[:, mask.bool()].contiguous()


def reference_time(args, gbuffer_pts=None):
    """One bounded sample of the workload on the reference CPU path (oracle/_ref, all host
    threads); returns (seconds, units, sample text, cores)."""
    from oracle import refshim
    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.manifest import load_manifest
    refshim.set_backend("avx2")
    cores = refshim.worker_threads()
    man = sub_manifest(args)
    try:
        if args.cfg.get("kind") == "gbuffer":
            if gbuffer_pts is None:
                raise RuntimeError("the config-4 sample needs the device G-buffer positions")
            pts = gbuffer_pts[:, :60000]
            delta = load_manifest(args.cfg["manifest"]).deltas[args.cfg["members"][0]]
            t0 = time.perf_counter()
            refshim.normal_map(man, 0, pts, delta)
            sec = time.perf_counter() - t0
            return sec, pts.shape[1], (f"neural_normal_map on {pts.shape[1]} of the 2560x1440 G-buffer hits, "
                                       f"reference library, {cores} threads"), cores
        cam = standard_camera(args.width, args.height)
        budgets = tuple(int(b) for b in args.budgets.split(","))
        src = 1 if args.normals == "mapped" else 0
        tm = 0.5 if args.config == 5 else 0.0
        _, _, _, sec = refshim.render(man, cam, TraceConfig(budgets), ShadeConfig(specular=0.3), src, -1, time=tm)
        text = f"one full {args.width}x{args.height} frame"
        if args.config == 5:
            text += " (t=0.5; the 120-frame sequence scales linearly)"
        return sec, args.width * args.height, text + f", reference shading::render (oracle/_ref, AVX2, {cores} threads)", cores
    finally:
        os.unlink(man)


def run_reference(args):
    """--impl reference: the reference CPU path (oracle/_ref, all host threads)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    pts = None
    if args.cfg.get("kind") == "gbuffer":
        from paper_2201_09147_b200.engine import Context
        ctx = Context(0, "fp32")
        pts = gbuffer_points(ctx, args).cpu().numpy()
        ctx.close()
    warm = min(args.warmup, 3)
    times = []
    for i in range(warm + min(args.steps, 10)):
        sec, units, sample, cores = reference_time(args, pts)
        if i >= warm:
            times.append(sec)
    sec = float(np.mean(times))
    value = units / sec / 1e6
    unit = "Mnormals/s" if args.cfg.get("kind") == "gbuffer" else "Mrays/s"
    line = {"impl": "reference", "metric": args.cfg["metric"], "value": value, "unit": unit, "n_gpus": args.gpus,
            "steps": len(times), "warmup": warm, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_text(args), "config": args.config,
                       "resolution": f"{args.width}x{args.height}", "budgets": args.budgets},
            "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_e2e(args, ctx, ds, seq, stream, world, rank, W):
    """Same metric through the C ABI with HOST buffers: pinned host framebuffer (render) or
    host point/normal arrays (normal map); every step's D2H is inside the timing."""
    import torch
    import torch.distributed as dist
    npix = args.width * args.height
    steps = len(W["frame_times"]) if W.get("frame_times") else args.steps
    if W["gbuffer"]:
        pts = W["pts"].cpu().numpy()
        k = pts.shape[1]
        delta = float(seq.deltas[0])
        # The public host-buffer call, nsdf_cuda_normal_map, from one host thread per
        # G-buffer in flight (each its own engine context: stream, staging pipe, weights), so
        # one G-buffer's H2D / D2H overlaps another's normal tiles.  Every G-buffer's normals
        # land in host memory inside the timing.
        import threading
        from paper_2201_09147_b200.engine import Context, DeviceSequence
        T = 3
        extra = [Context(ctx.device, args.mode) for _ in range(T - 1)]
        lanes = [(ctx, ds)] + [(c, DeviceSequence(c, seq)) for c in extra]
        srcs = [np.array(pts, copy=True) for _ in range(T)]
        last = [None] * T  # each lane's last result, checked against a single-thread call below

        def work(li, n):
            c, d = lanes[li]
            for _ in range(n):
                last[li] = c.normal_map(d.handles[0], srcs[li], delta)

        for li in range(T):
            work(li, 1)
        counts = [steps // T + (1 if li < steps % T else 0) for li in range(T)]
        threads = [threading.Thread(target=work, args=(li, counts[li])) for li in range(T)]
        w0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        e_ms = (time.perf_counter() - w0) * 1e3
        single = ctx.normal_map(ds.handles[0], pts, delta)
        same = all(r is not None and np.array_equal(r[0], single[0]) and r[1:] == single[1:] for r in last)
        for c in extra:
            c.close()
        from paper_2201_09147_b200 import scheduler
        rate, e_ms = scheduler.job_rate(k * steps, e_ms, world, device="cuda")  # all ranks / slowest rank
        return {"value": rate / 1e6, "unit": "Mnormals/s", "ms_per_frame": e_ms / steps,
                "outputs_equal_single_thread": bool(same),
                "h2d_bytes_per_step": 12 * k, "d2h_bytes_per_step": 12 * k + 16,
                "path": f"nsdf_cuda_normal_map (C ABI, host points -> host normals) from {T} host threads, "
                        f"one context each"}
    cam, cfg, shade, src, levels = W["cam"], W["cfg"], W["shade"], W["src"], W["levels"]
    frame_times = W.get("frame_times")  # animated: this rank's frame times t_i = i/(n-1)
    if world == 1 or W.get("shard_frames") or frame_times:
        # The public host-buffer call, nsdf_cuda_render, from one host thread per frame in
        # flight: each thread owns an engine context (own stream + workspace) and its own
        # pinned host framebuffer and renders every T-th frame, so one frame's D2H overlaps
        # the next frame's rendering.  Every frame's framebuffer lands in host memory inside
        # the timing (wall clock from the first call to the last return).
        import threading
        lanes = W.get("lanes") or [(ctx, stream, ds)]
        T = len(lanes)
        bufs = [(torch.empty(npix * 3, dtype=torch.float32, pin_memory=True),
                 torch.empty(npix, dtype=torch.float32, pin_memory=True),
                 torch.empty(npix, dtype=torch.uint8, pin_memory=True)) for _ in range(T)]
        lane_lv = [levels] + [d.levels() for _, _, d in lanes[1:]]

        def work(li, n, warm=False):
            c, _, dseq = lanes[li]
            r, d, m = bufs[li]
            for j in range(n):
                # animated: lane li renders frames li, li+T, ... of this rank (each its own slice)
                lv = dseq.levels(time=frame_times[li + j * T]) if frame_times and not warm else lane_lv[li]
                c.render_into(lv, cam, cfg, shade, r.data_ptr(), d.data_ptr(), m.data_ptr(), src)

        for li in range(T):
            work(li, 1, warm=True)
        counts = [steps // T + (1 if li < steps % T else 0) for li in range(T)]
        threads = [threading.Thread(target=work, args=(li, counts[li])) for li in range(T)]
        w0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        e_ms = (time.perf_counter() - w0) * 1e3
        path = f"nsdf_cuda_render (C ABI, host buffers) from {T} host threads, one context + pinned host " \
               f"framebuffer each"
    else:
        torch.cuda.synchronize()
        dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        w0 = time.perf_counter()
        peer = W.get("peer")
        if peer is not None and rank == 0:
            hb = (torch.empty(npix * 3, dtype=torch.float32, pin_memory=True),
                  torch.empty(npix, dtype=torch.float32, pin_memory=True),
                  torch.empty(npix, dtype=torch.uint8, pin_memory=True))
        for i in range(steps):
            W["step"](i)
            if rank == 0:
                if peer is not None:
                    W["ring"].done(i).synchronize()  # every rank's tiles of frame i
                    peer.to_host(i % (2 * len(W["lanes"])), *(t.data_ptr() for t in hb))
                else:
                    torch.cuda.current_stream().wait_stream(W["gstream"])
                    W["gather"].to_host()
        f1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) * 1e3
        e_ms = max(f0.elapsed_time(f1), wall)
        path = ("nsdf_cuda_render_device per rank, tiles stored into rank 0's framebuffer over NVLink, D2H on rank 0"
                if W.get("peer") is not None else "nsdf_cuda_render_device per rank + NCCL tile gather + D2H on rank 0")
    te = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e_ms = float(te.item())
    level_bytes = 16 * len(levels) + 4 * 8 + 128 + 272  # camera + configs + level table
    # frames mode: every rank's frames; animated: the whole sequence over all ranks
    frames = W["total_frames"] if frame_times else steps * (world if W.get("shard_frames") else 1)
    # The reference-shaped caller: shading::render returns an ImageBuffer of std::vectors, i.e.
    # PAGEABLE host memory — nsdf_cuda_render into fresh numpy arrays, one frame at a time from
    # one thread (rank 0, N = 1), next to the pinned multi-lane number above.
    pageable = None
    if rank == 0 and world == 1 and not frame_times:
        ctx.render(levels, cam, cfg, shade, src)
        n_pg = max(3, min(steps, 10))
        w0 = time.perf_counter()
        for _ in range(n_pg):
            ctx.render(levels, cam, cfg, shade, src)
        pg_ms = (time.perf_counter() - w0) * 1e3 / n_pg
        pageable = {"value": npix / (pg_ms / 1e3) / 1e6, "unit": "Mrays/s", "ms_per_frame": pg_ms, "frames": n_pg,
                    "path": "nsdf_cuda_render into fresh numpy arrays (pageable, lazily mapped), 1 thread, 1 frame "
                            "in flight"}
    # The reference's own call: C++ shading::render(seq, cam, cfg) -> ImageBuffer (the drop-in
    # library, libnsdf_b200.so), one frame at a time as `nsdf bench` does, after a warm-up
    dropin = None
    if rank == 0 and world == 1 and not frame_times and not W["gbuffer"]:
        import ctypes
        from paper_2201_09147_b200 import certify
        man = sub_manifest(args)
        try:
            sec = ctypes.c_double()
            st = certify._lib().nsdf_host_bench_render(man.encode(), ctypes.c_double(0.0), ctypes.byref(cam),
                                                       ctypes.byref(cfg), ctypes.byref(shade), src, -1, 2,
                                                       max(3, min(steps, 10)), ctypes.byref(sec))
            if st == 0:
                dropin = {"value": npix / sec.value / 1e6, "unit": "Mrays/s", "ms_per_frame": sec.value * 1e3,
                          "path": "C++ nsdf::shading::render -> ImageBuffer (libnsdf_b200.so, the reference API; "
                                  "the GPU renders while the ImageBuffer is allocated), 1 frame in flight"}
            else:
                dropin = {"unavailable": certify._lib().nsdf_host_last_error().decode()}
        finally:
            os.unlink(man)
    return {"value": npix * frames / (e_ms / 1e3) / 1e6, "unit": "Mrays/s", "ms_per_frame": e_ms / frames,
            "h2d_bytes_per_step": level_bytes, "d2h_bytes_per_step": npix * (12 + 4 + 1), "path": path,
            "pageable": pageable, "dropin": dropin}


def tile_pass(args, ctx, W, world, rank, Wd, Hd):
    """Frames-mode runs (N > 1) also time the strong-scaling alternative: the same frames
    split into image tiles across the ranks, each rank's shading kernels storing its tiles
    into rank 0's framebuffer ring (PeerFramebuffer), one 4-byte all-reduce per frame."""
    import torch
    import torch.distributed as dist
    from paper_2201_09147_b200 import scheduler

    lanes = W["lanes"]
    peer = scheduler.PeerFramebuffer(ctx, Wd, Hd, 2 * len(lanes), rank, world)
    if not peer.ok:
        peer.close()
        return {"unavailable": f"peer framebuffer: {peer.reason}"}
    ring = scheduler.PeerRing(peer, 2 * len(lanes))
    lv = [d.levels() for _, _, d in lanes]

    def frame(i):
        c, st, _ = lanes[i % len(lanes)]
        fr, fd, fm = ring.begin(i, st)
        c.render_device(lv[i % len(lanes)], W["cam"], W["cfg"], W["shade"], fr, fd, fm, W["src"], -1, args.tile, rank,
                        world)
        ring.end(i, st)

    n = max(2 * len(lanes), min(args.steps, 30))
    for i in range(max(3, len(lanes))):
        frame(i)
    torch.cuda.synchronize()
    dist.barrier()
    stream = lanes[0][1]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _, st, _ in lanes[1:]:
        st.wait_event(e0)
    for i in range(n):
        frame(i)
    for _, st, _ in lanes[1:]:
        stream.wait_stream(st)
    stream.wait_stream(ring.stream)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    dist.barrier()
    peer.close()
    return {"value": Wd * Hd * n / (ms / 1e3) / 1e6, "unit": "Mrays/s", "ms_per_frame": ms / n, "frames": n,
            "parallelism": f"tiles{world}", "tile": args.tile, "frames_in_flight": len(lanes),
            "frame_assembly": "peer stores into rank 0's framebuffer (NVLink)", "scaling": "strong"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.shard == "tiles":
        # tile shares with frames in flight: a short 256-wide level list runs on fewer CTAs of
        # >= 1536 rays each (full rows; the freed SMs take the other frames' kernels) —
        # tools/shardsim.py: N=8 5.9-6.1x -> 6.4-6.5x, N=4 3.2-3.3x -> 3.5x, N=1 unchanged
        os.environ.setdefault("NSDF_TC_MIN_ITEMS_256", "1536")
    # NSDF_BENCH_ONE_GPU=1: plumbing check of the N > 1 path on a one-GPU box — every rank on
    # cuda:0, host sync over gloo (no rank's kernels wait on another's).  Not a measurement.
    one_gpu = world > 1 and os.environ.get("NSDF_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2201_09147_b200.abi import ShadeConfig, TraceConfig, standard_camera
    from paper_2201_09147_b200.engine import Context, DeviceSequence
    from paper_2201_09147_b200 import scheduler

    cfgw = args.cfg
    seq = scheduler.broadcast_sequence(cfgw["manifest"] if rank == 0 else None, world, rank,
                                       device="cpu" if one_gpu else None)
    seq = seq.subsequence(cfgw["members"])
    Wd, Hd = args.width, args.height
    npix = Wd * Hd
    W = {"cam": standard_camera(Wd, Hd), "shade": ShadeConfig(specular=0.3),
         "src": 1 if args.normals == "mapped" else 0, "gbuffer": cfgw.get("kind") == "gbuffer"}
    animated = "frames" in cfgw
    # N > 1 on a frame stream: each rank renders whole frames (no per-frame collective, no
    # small-share tails); --shard tiles splits every frame across the ranks instead
    shard_frames = world > 1 and not animated and cfgw.get("kind") != "gbuffer" and args.shard == "frames"
    W["shard_frames"] = shard_frames

    ctx = Context(local, args.mode)
    stream = torch.cuda.Stream()          # the engine's launch stream; events are recorded on it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    ds = DeviceSequence(ctx, seq)
    steps = args.steps
    stats = None

    if W["gbuffer"]:
        pts = gbuffer_points(ctx, args)
        W["pts"] = pts
        k = pts.shape[1]
        units_per_step = k
        normals = torch.zeros_like(pts)
        counts = torch.zeros(2, dtype=torch.int64, device="cuda")
        delta = float(seq.deltas[0])

        def step(i=0):
            ctx.normal_map_device(ds.handles[0], pts.data_ptr(), k, delta, normals.data_ptr(), counts.data_ptr())
    else:
        units_per_step = npix
        budgets = tuple(int(b) for b in args.budgets.split(","))
        W["cfg"] = cfg = TraceConfig(budgets)
        rgb = torch.zeros(npix * 3, dtype=torch.float32, device="cuda")
        depth = torch.zeros(npix, dtype=torch.float32, device="cuda")
        mask = torch.zeros(npix, dtype=torch.uint8, device="cuda")
        if animated:
            # frames t_i = i/(n-1) (nsdf_main.cpp:308-324); frame i renders on rank i % world
            n_frames = cfgw["frames"]
            my_frames = scheduler.owned_frames(n_frames, rank, world)
            steps = len(my_frames)
            frame_levels = [ds.levels(time=i / (n_frames - 1)) for i in my_frames]
            W["frame_times"] = [i / (n_frames - 1) for i in my_frames]
            W["total_frames"] = n_frames
            W["levels"] = frame_levels[0]
        else:
            W["levels"] = ds.levels()
        tile_world, tile_rank = (1, 0) if animated or shard_frames else (world, rank)
        if args.inflight <= 0:
            args.inflight = 5 if tile_world >= 4 else 3
        # Frames in flight: `inflight` engine contexts, each on its own stream with its own
        # workspace, render consecutive frames concurrently (the tail iterations of one frame
        # overlap the next frame's head).  N > 1: frame i's NCCL tile gather runs on its own
        # stream while later frames render.  Every frame is still rendered completely.
        lanes = [(ctx, stream, ds)]
        for _ in range(1, max(1, args.inflight)):
            c2 = Context(local, args.mode)
            s2 = torch.cuda.Stream()
            c2.set_stream(s2.cuda_stream)
            lanes.append((c2, s2, DeviceSequence(c2, seq)))
        W["lanes"] = lanes
        # N > 1 (tiles of one frame): a cost-balanced tile map (--balance, default on) from one
        # frame traced on rank 0 — per tile, the evaluations its pixels took at each level and
        # its hits, weighted by the per-evaluation device time of each net (scheduler.tile_costs),
        # assigned longest-first to the least-loaded rank — the same map on every rank
        owners = None
        if world > 1 and not animated and not shard_frames and args.balance:
            obj = [None]
            if rank == 0:
                from conftest_free_records import records_np
                nidx = len(seq.members) - 1 if W["src"] == 1 else max(j for j, b in enumerate(budgets) if b > 0)
                rec = records_np(ctx.trace_image(W["levels"], W["cam"], cfg)[0])
                costs = scheduler.tile_costs(rec["iters"], rec["hit"], Wd, Hd, args.tile,
                                             [m.width for m in seq.members], seq.members[nidx].width)
                obj = [scheduler.balanced_tile_owners(costs, world).tolist()]
            dist.broadcast_object_list(obj, src=0)
            owners = np.asarray(obj[0], np.int32)
            for c_, _, _ in lanes:
                c_.set_tile_owners(owners)
        W["owners"] = owners
        # N > 1 (tiles of one frame): the ranks' shading kernels store their tiles straight
        # into rank 0's framebuffer ring over NVLink (PeerFramebuffer); NCCL tile gather only
        # if peer mapping is unavailable.
        peer, gather = None, None
        if world > 1 and not animated and not shard_frames:
            if args.gather == "peer":
                peer = scheduler.PeerFramebuffer(ctx, Wd, Hd, 2 * len(lanes), rank, world)
                if not peer.ok:
                    if rank == 0:
                        print(f"peer framebuffer unavailable ({peer.reason}); NCCL tile gather", file=sys.stderr)
                    peer.close()
                    peer = None
            if peer is None:
                gather = scheduler.TileGather(Wd, Hd, args.tile, rank, world, owners=owners)
        W["gather"], W["peer"] = gather, peer
        # frame-completion tokens and slot reuse: scheduler.PeerRing (one 4-byte all-reduce per
        # frame on one token stream, in frame order; a slot is rewritten only after the token of
        # the frame after its previous user completed)
        ring = scheduler.PeerRing(peer, 2 * len(lanes)) if peer is not None else None
        W["ring"] = ring
        tstream = ring.stream if ring is not None else None
        n_fb = max(len(lanes), 2 if gather is not None else 1)
        fbs = [(rgb, depth, mask)] + [(torch.zeros_like(rgb), torch.zeros_like(depth), torch.zeros_like(mask))
                                      for _ in range(n_fb - 1)]
        W["fbs"] = fbs
        gstream = torch.cuda.Stream() if gather is not None else None
        free_ev = [None] * n_fb
        W["gstream"] = gstream
        W["tstream"] = tstream
        if animated:
            lane_levels = [frame_levels] + [[d.levels(time=i / (cfgw["frames"] - 1)) for i in my_frames]
                                            for _, _, d in lanes[1:]]
        else:
            lane_levels = [[W["levels"]]] + [[d.levels()] for _, _, d in lanes[1:]]

        def step(i=0):
            li = i % len(lanes)
            c, st, d = lanes[li]
            lv = lane_levels[li][i % len(lane_levels[li])]
            if ring is not None:
                # this rank's tiles of frame i land in rank 0's ring slot (scheduler.PeerRing)
                fr, fd, fm = ring.begin(i, st)
                c.render_device(lv, W["cam"], cfg, W["shade"], fr, fd, fm, W["src"], -1, args.tile, tile_rank,
                                tile_world)
                ring.end(i, st)
                return
            b = i % n_fb
            if free_ev[b] is not None:
                st.wait_event(free_ev[b])
            fr, fd, fm = fbs[b]
            c.render_device(lv, W["cam"], cfg, W["shade"], fr.data_ptr(), fd.data_ptr(), fm.data_ptr(),
                            W["src"], -1, args.tile, tile_rank, tile_world)
            ev = torch.cuda.Event()
            ev.record(st)
            if gather is not None:
                with torch.cuda.stream(gstream):
                    gstream.wait_event(ev)
                    gather(fr, fd, fm)
                    ev = torch.cuda.Event()
                    ev.record(gstream)
            free_ev[b] = ev

        # accounting frame (not timed): per-level evaluation counts -> algorithmic FLOPs
        fb0 = peer.ptrs(0) if peer is not None else (rgb.data_ptr(), depth.data_ptr(), mask.data_ptr())
        stats = ctx.render_device(W["levels"], W["cam"], cfg, W["shade"], *fb0, W["src"], -1, args.tile, tile_rank,
                                  tile_world, stats=True)
        check_paths(stats, budgets, args.mode)
        if peer is not None:
            dist.barrier()
    W["step"] = step

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    side = [st for _, st, _ in W.get("lanes", [])[1:]] + [x for x in (W.get("gstream"), W.get("tstream"))
                                                          if x is not None]
    with ClockSampler(local) as clocks:
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for c, _, _ in W.get("lanes", [(ctx, None, None)]):
            c.set_profiling(True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks.mark("t0")
        e0.record(stream)
        for st in side:
            st.wait_event(e0)                  # every lane starts inside the timed region
        for i in range(steps):
            step(i)
        for st in side:
            stream.wait_stream(st)             # ...and finishes inside it (incl. the last gather)
        e1.record(stream)
        torch.cuda.synchronize()
        clocks.mark("t1")
    profs = [c.get_profile() for c, _, _ in W.get("lanes", [(ctx, None, None)])]
    for c, _, _ in W.get("lanes", [(ctx, None, None)]):
        c.set_profiling(False)
    prof = profs[0]
    prof_kind = "CUDA events around each launch, inside the timed region"
    if len(W.get("lanes", [])) > 1:
        # With frames in flight the launches of two frames overlap, so an in-region launch
        # duration is contended.  The per-kernel roofline therefore uses a serial pass of the
        # same frames on lane 0 right after the timed region (same stream, same buffers).
        ctx.set_profiling(True)
        for i in range(0, min(steps, 20) * len(W["lanes"]), len(W["lanes"])):
            W["step"](i)
        torch.cuda.synchronize()
        prof = ctx.get_profile()
        ctx.set_profiling(False)
        prof_kind = "CUDA events around each launch, serial pass (1 frame in flight) after the timed region"
    # single-frame latency (one frame in flight: rays .. framebuffer; at N > 1 the slowest
    # rank's share of a tile-split frame) beside the frames-in-flight throughput
    lat = torch.tensor([prof.frame_ms / max(prof.frames, 1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(lat, op=dist.ReduceOp.MAX)
    frame_latency_ms = float(lat.item())
    # job throughput: units over ALL ranks / the slowest rank's device time (max over ranks)
    if animated or W["gbuffer"] or shard_frames:
        my_units = units_per_step * steps                          # this rank's frames / G-buffer
    else:
        my_units = units_per_step * steps / world                  # tiles of the same frames
    rate, ms_total = scheduler.job_rate(my_units, e0.elapsed_time(e1), world, device="cuda")
    ms_per_frame = ms_total / steps / (world if shard_frames else 1)
    value = rate / 1e6
    unit = "Mnormals/s" if W["gbuffer"] else "Mrays/s"

    pk, pk_kind = peaks()
    traffic, traffic_note = ncu_traffic(W["gbuffer"]) if args.config == 2 else (None, None)
    levels_traffic = traffic  # all trace levels of one frame (roofline.hbm); `traffic` becomes the dominant kernel's
    # the roofline denominator: the BURST bf16 figure (kernels timed in short launches at the
    # clock they actually run at); the sustained figure is reported beside it
    peak_tf = pk["bf16_tflops"]
    peak_sust = pk.get("bf16_tflops_sustained", peak_tf)
    if W["gbuffer"]:
        flops_trace, flops_normals = 0, units_per_step * 2 * seq.members[0].macs_normal()
        achieved_tf = flops_normals / (ms_per_frame / 1e3) / 1e12
        kernel = "fused fwd+3-tangent normal tiles (256x3)"
        frame = {"points": units_per_step}
        all_levels = None
    else:
        normal_idx = len(seq.members) - 1 if W["src"] == 1 else max(j for j, b in enumerate(budgets) if b > 0)
        flops_trace, flops_normals = frame_flops(seq, stats, normal_idx)
        trace_ms = sum(prof.level_ms) / max(prof.frames, 1)
        normals_ms = prof.normals_ms / max(prof.frames, 1)
        achieved_tf = flops_trace / (trace_ms / 1e3) / 1e12 if trace_ms > 0 else 0.0
        kernel = "persistent trace-level MLP tiles (all levels)"
        # activation bound: one MUFU sine per hidden activation (layer 0 + hidden layers)
        sines = sum(int(stats.evals[j]) * (seq.members[j].n_layers - 1) * seq.members[j].width
                    for j in range(len(seq.members)))
        xu_peak = 16 * 148 * 1.965e9  # MUFU ops/s: 16/clk/SM x 148 SMs x max SM clock
        act_bound = {"sines_per_frame": sines, "achieved_per_s": sines / (trace_ms / 1e3) if trace_ms > 0 else 0.0,
                     "peak_per_s": xu_peak, "frac": sines / (trace_ms / 1e3) / xu_peak if trace_ms > 0 else 0.0,
                     "note": "MUFU (XU pipe) sine throughput of the trace kernels; 64/128-wide nets are sine-bound"}
        # each kernel against its own bound: tensor work ISSUED by the fast mode (3 split-precision
        # terms per hidden K step + the K=32 layer-0 MMA + the K=16 bias MMA per hidden layer)
        # vs the sustained tensor peak, and MUFU sines vs 16/clk/SM at the max SM clock
        per_kernel = []
        for j, m in enumerate(seq.members):
            w, hb = m.width, m.hidden_blocks
            ev, ms_j = int(stats.evals[j]), prof.level_ms[j] / max(prof.frames, 1)
            if ev == 0 or ms_j <= 0:
                continue
            # fp16 mode: 3 fp16 MMA slots per hidden K step, or 2 where the correction terms
            # run as one E4M3 MMA (256-wide nets at omega0 <= 15, mlp_tc.cuh tc_split8)
            f8 = f8_hidden_layers(m) if args.mode == "fp16" else 0
            mult = 1 if args.mode != "fp16" else 3
            issued = ev * (2 * 32 * w + hb * (mult * 2 * w * w + 2 * 16 * w) - f8 * 2 * w * w)
            sn = ev * (m.n_layers - 1) * w
            tf = ev * 2 * m.macs_forward() / (ms_j / 1e3) / 1e12
            per_kernel.append({"kernel": f"trace level {j} ({w}x{hb})", "ncu_name": f"tc_mlp_kernel<{w}, 0,",
                               "ms": ms_j, "evals": ev, "tflops_algorithmic": tf, "frac_burst": tf / peak_tf,
                               "tensor_issued_frac": issued / (ms_j / 1e3) / 1e12 / peak_tf,
                               "mufu_frac": sn / (ms_j / 1e3) / xu_peak})
        if normals_ms > 0 and int(stats.normal_evals):
            m = seq.members[normal_idx]
            w, hb, ev = m.width, m.hidden_blocks, int(stats.normal_evals)
            # the normal tiles run one fp16 term (their tolerance is an angle; engine.cuh
            # normal_tile_terms) unless NSDF_NORMAL_TERMS=3
            mult_n = 3 if args.mode == "fp16" and os.environ.get("NSDF_NORMAL_TERMS") == "3" else 1
            issued = 4 * ev * (2 * 32 * w + hb * (mult_n * 2 * w * w + 2 * 16 * w))
            per_kernel.append({"kernel": f"normal tiles + shading ({w}x{hb}, 4 rows per hit)", "ms": normals_ms,
                               "ncu_name": f"tc_mlp_kernel<{w}, 1,", "evals": ev,
                               "tflops_algorithmic": flops_normals / (normals_ms / 1e3) / 1e12,
                               "frac_burst": flops_normals / (normals_ms / 1e3) / 1e12 / peak_tf,
                               "tensor_issued_frac": issued / (normals_ms / 1e3) / 1e12 / peak_tf,
                               "mufu_frac": 4 * ev * (m.n_layers - 1) * w / (normals_ms / 1e3) / xu_peak})
        act_bound["per_kernel"] = per_kernel
        # roofline = the DOMINANT kernel (largest share of the frame), algorithmic FLOPs per
        # launch / its CUDA-event launch time; the all-levels aggregate is reported beside it
        all_levels = {"achieved": achieved_tf, "frac_burst": achieved_tf / peak_tf,
                      "frac_sustained": achieved_tf / peak_sust, "kernel": kernel}
        if per_kernel:
            dom = max(per_kernel, key=lambda r: r["ms"])
            achieved_tf, kernel = dom["tflops_algorithmic"], dom["kernel"]
            traffic = ncu_kernel_traffic(dom["ncu_name"]) if args.config == 2 else None
            traffic_note = "DRAM read+write bytes per launch of the dominant kernel, ncu --set full" \
                if traffic is not None else None
        frame = {"evals_per_level": [int(x) for x in list(stats.evals)[:len(seq.members)]], "hits": int(stats.hits),
                 "fallbacks": int(stats.fallback_evals), "tflop_trace": flops_trace / 1e12,
                 "tflop_normals": flops_normals / 1e12, "trace_ms": trace_ms, "normals_ms": normals_ms,
                 "profiled_frame_ms": prof.frame_ms / max(prof.frames, 1), "profile": prof_kind,
                 "level_ms": [prof.level_ms[j] / max(prof.frames, 1) for j in range(len(seq.members))]}

    # config 2 is reported at the generous setting (40,20,20) — the headline,
    # whose frame converges (hits within ~5% of (40,40,40)) — and at the paper-style speed
    # setting (20,5,5) beside it, each with the image MSE against the (40,40,40) frame, as
    # `nsdf bench` reports every row against its baseline row (nsdf_main.cpp:484-500).
    alt, quality = None, None
    if not W["gbuffer"] and not animated and world == 1 and not args.no_alt:
        lanes = W.get("lanes") or [(ctx, stream, ds)]

        def frame_image(budgets_):
            c0, s0, d0 = lanes[0]
            fr, fd, fm = W["fbs"][0]
            torch.cuda.synchronize()
            c0.render_device(d0.levels(), W["cam"], TraceConfig(budgets_), W["shade"], fr.data_ptr(), fd.data_ptr(),
                             fm.data_ptr(), W["src"], -1, args.tile, 0, 1)
            torch.cuda.synchronize()
            return fr.double().cpu().numpy(), int(fm.sum().item())

        conv = tuple(40 if b > 0 else 0 for b in budgets)
        ref_img, ref_hits = frame_image(conv)
        img, hits = frame_image(budgets)
        quality = {"reference_budgets": ",".join(map(str, conv)), "hits": hits, "hits_reference": ref_hits,
                   "hits_frac": hits / max(ref_hits, 1), "mse_vs_reference": float(np.mean((img - ref_img) ** 2)),
                   "note": "image MSE against the same frame at budgets 40 per traced level (nsdf bench's MSE column)"}
        if cfgw.get("speed_budgets"):
            sb = tuple(int(x) for x in cfgw["speed_budgets"].split(","))
            cfg_alt = TraceConfig(sb)
            lv_alt = [d.levels() for _, _, d in lanes]
            n_alt = max(6, min(steps, 30))

            def alt_frame(i):
                c, st_, _ = lanes[i % len(lanes)]
                fr, fd, fm = W["fbs"][i % len(W["fbs"])]
                c.render_device(lv_alt[i % len(lanes)], W["cam"], cfg_alt, W["shade"], fr.data_ptr(), fd.data_ptr(),
                                fm.data_ptr(), W["src"], -1, args.tile, 0, 1)

            for i in range(len(lanes)):
                alt_frame(i)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _, st_, _ in lanes[1:]:
                st_.wait_event(a0)
            for i in range(n_alt):
                alt_frame(i)
            for _, st_, _ in lanes[1:]:
                stream.wait_stream(st_)
            a1.record(stream)
            torch.cuda.synchronize()
            alt_ms = a0.elapsed_time(a1) / n_alt
            simg, shits = frame_image(sb)
            alt = {"budgets": cfgw["speed_budgets"], "frames": n_alt, "ms_per_frame": alt_ms,
                   "value": units_per_step / (alt_ms / 1e3) / 1e6, "unit": "Mrays/s", "hits": shits,
                   "hits_frac": shits / max(ref_hits, 1), "mse_vs_reference": float(np.mean((simg - ref_img) ** 2))}

    # HBM side of the roofline (north_star: "achieved HBM GB/s for compaction and normal
    # mapping"): the trace kernels' measured DRAM bytes per frame (ncu capture, config 2) over
    # their time; the normal map's algorithmic bytes (point in, normal out) over its time.
    hbm_peak = pk.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
    if W["gbuffer"]:
        nbytes = units_per_step * 24
        gbs = nbytes / (ms_per_frame / 1e3) / 1e9
        hbm = {"kernel": "normal map (12 B point in, 12 B normal out per point)", "bytes": nbytes,
               "achieved_gbs": gbs, "peak_gbs": hbm_peak, "frac": gbs / hbm_peak, "bytes_kind": "algorithmic"}
    elif levels_traffic is not None:
        tms = frame["trace_ms"]
        gbs = levels_traffic / (tms / 1e3) / 1e9 if tms > 0 else 0.0
        hbm = {"kernel": "persistent trace levels incl. compaction", "bytes": levels_traffic, "achieved_gbs": gbs,
               "peak_gbs": hbm_peak, "frac": gbs / hbm_peak, "bytes_kind": "ncu dram read+write per frame"}
    else:
        hbm = None

    strong = tile_pass(args, ctx, W, world, rank, Wd, Hd) if shard_frames else None

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, ds, seq, stream, world, rank, W)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            gp = W["pts"].cpu().numpy() if W["gbuffer"] else None
            sec, units, sample, cores = reference_time(args, gp)
            cpu = {"value": units / sec / 1e6, "unit": unit, "cores": cores, "kind": "reference",
                   "ms_per_frame": None if W["gbuffer"] else sec * 1e3, "sample": sample}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": unit, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        launches = (int(stats.kernel_launches) if stats is not None else 1) * steps
        clk = clocks.summary()
        if not W["gbuffer"] and clk.get("sm_mhz"):
            # the same MUFU fractions against 16/clk/SM at the SM clock measured in the timed
            # region (power-capped runs sit well below the 1965 MHz maximum)
            for k in act_bound["per_kernel"]:
                k["mufu_frac_at_sm_clock"] = k["mufu_frac"] * 1965.0 / clk["sm_mhz"]
            act_bound["frac_at_sm_clock"] = act_bound["frac"] * 1965.0 / clk["sm_mhz"]
        line = {
            "metric": cfgw["metric"], "value": value, "unit": unit, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms_total / steps, "ms_per_frame": ms_per_frame,
            "higher_is_better": True,
            "scaling": "strong" if world > 1 and not (W["gbuffer"] or shard_frames) else "weak", "vs_baseline": None,
            "dtype": {"fp16": "split-fp16 tensor (A_hi.W_hi fp16 + correction terms: 2 fp16 MMAs, or one E4M3 MMA "
                              "for 256-wide nets at omega0 <= 15; the normal tiles 1 term) / fp32 accum",
                      "fp16low": "fp16 tensor / fp32 accum",
                      "fp32": "f32"}[args.mode],
            "data": "synthetic camera rays; committed fitted SIREN weights (assets/)",
            "config": {"workload": workload_text(args), "config": args.config, "resolution": f"{Wd}x{Hd}",
                       "budgets": args.budgets, "mode": args.mode, "tile": args.tile,
                       "frames_in_flight": 1 if W["gbuffer"] else max(1, args.inflight),
                       "parallelism": (f"frames{world}" if animated or shard_frames else f"tiles{world}")
                       if world > 1 else "single",
                       "frame_assembly": None if world == 1 or animated else
                       "none: frames stay on their rank (e2e: each rank's frames D2H into its host)" if shard_frames else
                       ("peer stores into rank 0's framebuffer (NVLink)" if W.get("peer") is not None
                        else "NCCL tile gather"),
                       "l2": "per-frame working set (ray state, lists, framebuffer) > 126 MB L2; weights L2-resident"},
            "fps": 1000.0 / ms_per_frame,
            "frame_latency_ms": None if W["gbuffer"] else frame_latency_ms,
            "frame": frame,
            "frame_quality": quality,
            "speed_setting": alt,
            "strong_scaling": strong,
            "roofline": {"bound": "tensor", "kernel": kernel, "achieved": achieved_tf, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved_tf / peak_tf,
                         "peak_kind": f"{pk_kind} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                         "frac_vs_sustained": achieved_tf / peak_sust, "traffic": traffic,
                         "traffic_note": traffic_note, "all_trace_levels": all_levels,
                         "whole_frame_tflops": (flops_trace + flops_normals) / (ms_per_frame / 1e3) / 1e12,
                         "activation_bound": None if W["gbuffer"] else act_bound,
                         "hbm": hbm},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    for c, _, _ in W.get("lanes", [(ctx, None, None)]):
        c.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
