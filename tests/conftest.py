import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The drop-in library (libnsdf_b200.so) creates ONE process-wide engine context on first
# use, with the arithmetic mode from NSDF_MODE; the bit-exact drop-in tests need the oracle
# mode whichever test loads the library first.
os.environ.setdefault("NSDF_MODE", "oracle")

ASSETS = os.path.join(ROOT, "assets")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box)")


@pytest.fixture(scope="session")
def oracle_built():
    import oracle
    oracle.build()
    return True


@pytest.fixture(scope="session")
def ctx():
    from paper_2201_09147_b200.engine import Context
    c = Context(0, "fp32")
    yield c
    c.close()


def random_net(width, hidden, input_dim=3, omega0=30.0, seed=1):
    """mlp::random_init restated in numpy is not needed: use the reference's own
    random_init when available, else a fixed-seed uniform init of the same ranges."""
    from paper_2201_09147_b200.manifest import Net
    try:
        from oracle import refshim
        if refshim.available():
            rows, cols, packed = refshim.random_init(width, hidden, input_dim, omega0, seed)
            return Net(rows, cols, packed, 0, omega0, input_dim)
    except OSError:
        pass
    rng = np.random.default_rng(seed)
    dims = [input_dim] + [width] * (hidden + 1) + [1]
    layers = []
    for i in range(len(dims) - 1):
        fan_in = dims[i]
        bound = 1.0 / fan_in if i == 0 else np.sqrt(6.0 / fan_in) / omega0
        w = rng.uniform(-bound, bound, size=(dims[i + 1], fan_in))
        b = rng.uniform(-1 / np.sqrt(fan_in), 1 / np.sqrt(fan_in), size=dims[i + 1])
        layers.append((w, b))
    return Net.from_layers(layers, 0, omega0, input_dim)


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def records_np(recs):
    """HitRecord ctypes array -> dict of numpy arrays."""
    n = len(recs)
    arr = np.frombuffer(memoryview(recs).cast("B"), dtype=np.dtype([
        ("hit", "<i4"), ("point", "<f4", 3), ("t", "<f4"), ("level", "<i4"), ("iters", "<u2", 8),
        ("fd", "<f4")]), count=n)
    return arr
