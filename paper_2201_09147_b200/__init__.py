"""nsdf-b200: B200-native multiscale sphere tracing of nested SIREN SDFs.

Python mirror of the reference C++ API (proj/include/nsdf) over the C ABI of
libnsdf_cuda.so (include/nsdf_cuda.h).  See DESIGN.md."""
from .abi import NsdfError, Camera, TraceConfig, ShadeConfig, HitRecord, standard_camera  # noqa: F401
from .manifest import Net, Analytic, Sequence, load_sdfnet, load_manifest  # noqa: F401
