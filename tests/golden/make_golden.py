"""Generates tests/golden/golden.npz from the REFERENCE library (oracle/_ref/libnsdf_ref.so,
compiled from /root/reference by oracle/Makefile, AVX2 backend).  Run in the build container:

    python tests/golden/make_golden.py

Contents: two reference random_init SIRENs (64x1 omega 30 seed 11, 256x3 omega 30 seed 12)
with their f32 forward + gradient on 97 fixed points, and the standard camera's rays at 40x30.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import refshim  # noqa: E402
from paper_2201_09147_b200.abi import standard_camera  # noqa: E402
from paper_2201_09147_b200.manifest import Net  # noqa: E402


def main():
    refshim.set_backend("avx2")
    out = {}
    pts = np.random.default_rng(123).uniform(-1.1, 1.1, (3, 97)).astype(np.float32)
    out["pts"] = pts
    for tag, (w, k, seed) in {"n64": (64, 1, 11), "n256": (256, 3, 12)}.items():
        rows, cols, packed = refshim.random_init(w, k, 3, 30.0, seed)
        net = Net(rows, cols, packed, 0, 30.0, 3)
        d, g = refshim.mlp(net, pts, 2)
        out.update({f"{tag}_rows": rows, f"{tag}_cols": cols, f"{tag}_packed": packed,
                    f"{tag}_omega": np.float64(30.0), f"{tag}_dist": d, f"{tag}_grad": g})
    cam = standard_camera(40, 30)
    out["cam_w"], out["cam_h"] = np.int32(40), np.int32(30)
    out["rays"] = refshim.generate_rays(cam)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz"), **out)


if __name__ == "__main__":
    main()
