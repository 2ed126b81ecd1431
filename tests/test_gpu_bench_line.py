"""The N=1 bench.py contract on the G-buffer workload (config 4, reduced resolution): one JSON
line with the device-resident value, the e2e number through nsdf_cuda_normal_map from host
buffers (3 host threads, one engine context each) and the H2D/D2H byte counts of the
points/normals it copies."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_gbuffer_line():
    env = dict(os.environ)
    env.pop("NSDF_MODE", None)  # conftest's oracle-mode default is not a bench --mode
    r = subprocess.run([sys.executable, "bench.py", "--config", "4", "--width", "640", "--height", "360",
                        "--steps", "7", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "e2e", "roofline", "clocks",
              "gpu_launches"):
        assert k in line
    assert line["unit"] == "Mnormals/s" and line["value"] > 0 and line["gpu_launches"] > 0
    e2e = line["e2e"]
    assert e2e["unit"] == "Mnormals/s" and e2e["value"] > 0
    assert "3 host threads" in e2e["path"]
    assert e2e["outputs_equal_single_thread"] is True  # the threaded lanes' normals == one call's
    k = e2e["h2d_bytes_per_step"] // 12          # G-buffer hit points per step
    assert k > 0 and e2e["h2d_bytes_per_step"] == 12 * k and e2e["d2h_bytes_per_step"] == 12 * k + 16
