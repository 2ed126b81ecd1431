"""ctypes mirror of include/nsdf_cuda.h (PODs + the libnsdf_cuda.so loader).

The product path loads ONLY the in-tree CUDA library; there is no CPU fallback — if the
extension is missing or no device is present, calls fail loudly (NsdfError)."""
from __future__ import annotations

import ctypes
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# NSDF_CUDA_LIB: an alternative build of the engine for A/B timing (tools/ab.py); default in-tree
LIB_PATH = os.environ.get("NSDF_CUDA_LIB") or os.path.join(PKG_DIR, "libnsdf_cuda.so")
HOST_LIB_PATH = os.path.join(PKG_DIR, "libnsdf_b200.so")

MAX_LEVELS = 8
PATH_NONE, PATH_SIMT, PATH_TCGEN05 = 0, 1, 2  # nsdf_kernel_path
MAX_LIGHTS = 8

OK, ERR_CONTRACT, ERR_CONFIG, ERR_VALIDATION, ERR_PARSE, ERR_DIVERGENCE, ERR_DEVICE = range(7)
MODE_FP32_ORACLE, MODE_FP16_FAST, MODE_FP16_LOW = 0, 1, 2
ACT_SINE, ACT_IDENTITY = 0, 1
FIELD_SPHERE, FIELD_TORUS, FIELD_BOX = 1, 2, 3
NORMALS_OWN, NORMALS_MAPPED = 0, 1

ERROR_KINDS = {1: "contract", 2: "config", 3: "validation", 4: "parse", 5: "divergence", 6: "device"}


class NsdfError(RuntimeError):
    """nsdf::Error mirror: .kind is the ErrorKind name (core.hpp:12-18)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.kind = ERROR_KINDS.get(status, "validation")


class Camera(ctypes.Structure):
    """tracer::Camera (trace.hpp:13-22); defaults as the reference struct."""
    _fields_ = [("position", ctypes.c_double * 3), ("look_at", ctypes.c_double * 3),
                ("up", ctypes.c_double * 3), ("vertical_fov_deg", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]

    def __init__(self, position=(0, 0, 3), look_at=(0, 0, 0), up=(0, 1, 0), fov=40.0, width=256, height=256):
        super().__init__()
        self.position[:] = position
        self.look_at[:] = look_at
        self.up[:] = up
        self.vertical_fov_deg = fov
        self.width = width
        self.height = height


def standard_camera(width=256, height=256) -> Camera:
    """scenes::standard_camera (tests/support/scenes.hpp:26-35), = the CLI default
    (nsdf_main.cpp:97-104)."""
    return Camera((2.0, 1.5, 2.0), (0, 0, 0), (0, 1, 0), 50.0, width, height)


class TraceConfig(ctypes.Structure):
    """tracer::TraceConfig (trace.hpp:49-55)."""
    _fields_ = [("n_levels", ctypes.c_int32), ("budgets", ctypes.c_int32 * MAX_LEVELS),
                ("eps_stop", ctypes.c_float), ("t_max", ctypes.c_float)]

    def __init__(self, budgets=(40,), eps_stop=1e-3, t_max=10.0):
        super().__init__()
        self.n_levels = len(budgets)
        for i, b in enumerate(budgets):
            self.budgets[i] = b
        self.eps_stop = eps_stop
        self.t_max = t_max


class HitRecord(ctypes.Structure):
    """tracer::HitRecord (trace.hpp:34-47)."""
    _fields_ = [("hit", ctypes.c_int32), ("point", ctypes.c_float * 3), ("t", ctypes.c_float),
                ("level_reached", ctypes.c_int32), ("iterations_used", ctypes.c_uint16 * MAX_LEVELS),
                ("final_distance", ctypes.c_float)]


class ShadeConfig(ctypes.Structure):
    """shading::ShadeConfig + Material + DirectionalLight (shading.hpp:90-107)."""
    _fields_ = [("albedo", ctypes.c_float * 3), ("ambient", ctypes.c_float), ("diffuse", ctypes.c_float),
                ("specular", ctypes.c_float), ("shininess", ctypes.c_float), ("n_lights", ctypes.c_int32),
                ("light_direction", (ctypes.c_float * 3) * MAX_LIGHTS),
                ("light_intensity", ctypes.c_float * MAX_LIGHTS), ("background", ctypes.c_float * 3)]

    def __init__(self, specular=0.0, lights=(((0.4, 0.7, 0.5), 1.0),), albedo=(0.8, 0.8, 0.8), ambient=0.1,
                 diffuse=0.9, shininess=32.0, background=(0.0, 0.0, 0.0)):
        super().__init__()
        self.albedo[:] = albedo
        self.ambient = ambient
        self.diffuse = diffuse
        self.specular = specular
        self.shininess = shininess
        self.n_lights = len(lights)
        for i, (d, inten) in enumerate(lights):
            self.light_direction[i][:] = d
            self.light_intensity[i] = inten
        self.background[:] = background


class Level(ctypes.Structure):
    _fields_ = [("field", ctypes.c_int32), ("time", ctypes.c_float), ("delta", ctypes.c_double)]


class FrameStats(ctypes.Structure):
    _fields_ = [("evals", ctypes.c_uint64 * MAX_LEVELS), ("hits", ctypes.c_uint64),
                ("normal_evals", ctypes.c_uint64), ("fallback_evals", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("level_path", ctypes.c_uint8 * MAX_LEVELS),
                ("normals_path", ctypes.c_uint8), ("fallback_path", ctypes.c_uint8), ("reserved_", ctypes.c_uint8 * 6)]


class Profile(ctypes.Structure):
    _fields_ = [("level_ms", ctypes.c_double * MAX_LEVELS), ("normals_ms", ctypes.c_double),
                ("frame_ms", ctypes.c_double), ("frames", ctypes.c_uint64), ("trace_launches", ctypes.c_uint64),
                ("normal_launches", ctypes.c_uint64)]


_LIB = None


def load_library():
    """Load the in-tree libnsdf_cuda.so.  Fails loudly — there is no fallback."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise NsdfError(ERR_DEVICE, f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    lib.nsdf_cuda_last_error.restype = ctypes.c_char_p
    _LIB = lib
    return lib


def check(status: int) -> None:
    if status != OK:
        msg = load_library().nsdf_cuda_last_error().decode(errors="replace")
        raise NsdfError(status, msg)


class TrainConfigC(ctypes.Structure):
    """nsdf_train_config (trainer::TrainConfig minus arch / omega0 / seed)."""
    _fields_ = [("epochs", ctypes.c_int), ("batch_size", ctypes.c_int), ("learning_rate", ctypes.c_double),
                ("momentum", ctypes.c_double), ("warmup_epochs", ctypes.c_int), ("plateau_patience", ctypes.c_int),
                ("plateau_threshold", ctypes.c_double), ("min_learning_rate", ctypes.c_double)]

    def __init__(self, epochs=800, batch_size=8192, learning_rate=0.3, momentum=0.9, warmup_epochs=100,
                 plateau_patience=60, plateau_threshold=0.05, min_learning_rate=1e-10):
        super().__init__(epochs, batch_size, learning_rate, momentum, warmup_epochs, plateau_patience,
                         plateau_threshold, min_learning_rate)


class TrainReportC(ctypes.Structure):
    _fields_ = [("final_loss", ctypes.c_double), ("validation_mse", ctypes.c_double),
                ("validation_max_error", ctypes.c_double), ("final_learning_rate", ctypes.c_double),
                ("diverged", ctypes.c_int), ("halvings", ctypes.c_int), ("epochs_recorded", ctypes.c_int)]
