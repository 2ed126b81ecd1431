"""HitRecord ctypes array -> numpy structured view (tools' copy of tests/conftest.records_np)."""
import numpy as np


def records_np(recs):
    n = len(recs)
    return np.frombuffer(memoryview(recs).cast("B"), dtype=np.dtype([
        ("hit", "<i4"), ("point", "<f4", 3), ("t", "<f4"), ("level", "<i4"), ("iters", "<u2", 8),
        ("fd", "<f4")]), count=n)
