"""A/B timing of engine builds on one GPU: alternates `bench.py` runs over the libraries
given (NSDF_CUDA_LIB), so clock/power drift hits every variant alike.

    python tools/ab.py [--rounds 3] [--steps 50] lib_a.so lib_b.so ...
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--mode", default="fp16")
ap.add_argument("libs", nargs="+")
args = ap.parse_args()
res = {lib: [] for lib in args.libs}
for r in range(args.rounds):
    for lib in args.libs:
        env = dict(os.environ, NSDF_CUDA_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "bench.py", "--steps", str(args.steps), "--config", str(args.config),
                              "--no-cpu-baseline", "--no-e2e", "--no-alt", "--mode", args.mode], cwd=ROOT, env=env,
                             capture_output=True, text=True)
        line = json.loads(out.stdout.strip().splitlines()[-1])
        res[lib].append((line["ms_per_step"], line["frame"].get("level_ms"), line["clocks"]["sm_mhz"]))
        print(f"round {r} {lib}: {line['ms_per_step']:.4f} ms/frame levels "
              f"{[round(x, 3) for x in line['frame'].get('level_ms', [])]} sm {line['clocks']['sm_mhz']}", flush=True)
for lib, v in res.items():
    ms = sorted(x[0] for x in v)
    print(f"{lib}: median {ms[len(ms) // 2]:.4f} min {ms[0]:.4f} ms/frame")
