"""The C-ABI PODs (include/nsdf_cuda.h), shared with the product's ctypes mirror so oracle
and engine results compare field by field.  Pure data layout, no compute."""
from paper_2201_09147_b200.abi import (Camera, HitRecord, Level, ShadeConfig, TraceConfig,  # noqa: F401
                                       standard_camera)
