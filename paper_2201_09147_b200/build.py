"""Builds the in-tree native libraries (no JIT cache: the .so files travel with the repo).

  libnsdf_cuda.so   CUDA engine + C ABI (include/nsdf_cuda.h), sm_100a only.
  libnsdf_b200.so   C++ drop-in host library (include/nsdf/*.hpp) over the C ABI.

Per-file flags: engine.cu (trace loop, rays, shading, FFMA oracle tiles) is compiled with
-fmad=false so no multiply-add can be contracted behind the explicit _rn intrinsics;
mlp_tc.cu (tcgen05 fast path) keeps contraction on.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
OBJ = os.path.join(PKG, "_obj")
INC = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"

CUDA_SOURCES = {
    "engine.cu": ["-fmad=false"],
    "capi.cu": ["-fmad=false"],
    "mlp_tc.cu": [],
    "mlp_f64.cu": ["-fmad=false"],
    "train_f64.cu": ["-fmad=false"],
    "tensor_ops.cu": ["-fmad=false"],
}


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout)
        raise RuntimeError(f"build failed: {os.path.basename(cmd[-1])}")
    return r.stdout


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers(d):
    return [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cuh", ".h", ".hpp"))]


CHECKED_DIR = os.path.join(PKG, "_checked")


def build_cuda(force=False, verbose=False, checked=False):
    """checked=True: the bounds-checked variant (-DNSDF_CHECKED=1, common.cuh) into
    _checked/libnsdf_cuda.so — every list index, ray slot, staged append and framebuffer pixel
    of the kernels checked on the device (tests/test_gpu_checked.py loads it through
    NSDF_CUDA_LIB)."""
    obj_dir = os.path.join(PKG, "_obj_checked") if checked else OBJ
    os.makedirs(obj_dir, exist_ok=True)
    deps_common = _headers(CSRC) + [os.path.join(INC, "nsdf_cuda.h")]
    jobs = []
    objs = []
    timeline = os.environ.get("NSDF_TC_TIMELINE_BUILD") == "1"  # tools/timeline.py instrumentation
    for src, extra in CUDA_SOURCES.items():
        if timeline and src == "mlp_tc.cu":
            extra = extra + ["-DNSDF_TC_TIMELINE_BUILD=1"]
        if src == "mlp_tc.cu" and os.environ.get("NSDF_TC_DEFINES"):  # A/B builds (tools/ab.py)
            extra = extra + os.environ["NSDF_TC_DEFINES"].split()
        if src != "mlp_tc.cu" and os.environ.get("NSDF_ENGINE_DEFINES"):
            extra = extra + os.environ["NSDF_ENGINE_DEFINES"].split()
        if checked:
            extra = extra + ["-DNSDF_CHECKED=1"]
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + deps_common):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                   "-Xptxas", "-v" if verbose else "-O3", "-I", INC, "-I", CSRC, *extra, "-c", s, "-o", o]
            jobs.append(cmd)
    with ThreadPoolExecutor(max_workers=4) as ex:
        outs = list(ex.map(_run, jobs))
    if verbose:
        for o in outs:
            print(o)
    if checked:
        os.makedirs(CHECKED_DIR, exist_ok=True)
    lib = os.path.join(CHECKED_DIR if checked else PKG, "libnsdf_cuda.so")
    if force or jobs or _stale(lib, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart=static", "-o", lib, *objs])
    return lib


HOST_FLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-Wall"]


def build_host(force=False):
    """The drop-in C++ library: include/nsdf headers, host/*.cpp, links libnsdf_cuda.so."""
    if not os.path.isdir(HOST):
        return None
    srcs = sorted(os.path.join(HOST, f) for f in os.listdir(HOST) if f.endswith(".cpp"))
    if not srcs:
        return None
    lib = os.path.join(PKG, "libnsdf_b200.so")
    hdrs = _headers(HOST) + [os.path.join(INC, "nsdf_cuda.h"), os.path.join(INC, "nsdf_host.h")]
    for dp, _, fs in os.walk(os.path.join(INC, "nsdf")):
        hdrs += [os.path.join(dp, f) for f in fs]
    os.makedirs(OBJ, exist_ok=True)
    jobs, objs = [], []
    for s in srcs:
        o = os.path.join(OBJ, "host_" + os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append(["g++", *HOST_FLAGS, "-I", INC, "-I", JSON_DIR, "-I", HOST, "-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=8) as ex:
        list(ex.map(_run, jobs))
    if force or jobs or _stale(lib, objs + [os.path.join(PKG, "libnsdf_cuda.so")]):
        _run(["g++", "-shared", *objs, "-o", lib, "-L", PKG, "-lnsdf_cuda", "-lz", "-Wl,-rpath,$ORIGIN"])
    return lib


def build_cpp_tests(force=False):
    """tests/cpp/*.cpp -> tests/cpp/bin/*: reference-style checks of the drop-in C++ API."""
    tdir = os.path.join(ROOT, "tests", "cpp")
    if not os.path.isdir(tdir):
        return []
    out = os.path.join(tdir, "bin")
    os.makedirs(out, exist_ok=True)
    lib = os.path.join(PKG, "libnsdf_b200.so")
    hdrs = [os.path.join(tdir, f) for f in os.listdir(tdir) if f.endswith(".hpp")]
    for dp, _, fs in os.walk(os.path.join(INC, "nsdf")):
        hdrs += [os.path.join(dp, f) for f in fs]
    jobs, bins = [], []
    for f in sorted(os.listdir(tdir)):
        if not f.endswith(".cpp"):
            continue
        src = os.path.join(tdir, f)
        exe = os.path.join(out, f[:-4])
        bins.append(exe)
        if force or _stale(exe, [src, lib] + hdrs):
            jobs.append(["g++", *HOST_FLAGS, "-I", INC, src, "-o", exe, "-L", PKG, "-lnsdf_b200", "-lnsdf_cuda",
                         "-Wl,-rpath," + PKG])
    with ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(_run, jobs))
    return bins


def build_tools(force=False):
    """tools/cli/*.cpp -> tools/bin/*: the reference CLI's flows over libnsdf_b200.so."""
    src_dir = os.path.join(ROOT, "tools", "cli")
    if not os.path.isdir(src_dir):
        return []
    out = os.path.join(ROOT, "tools", "bin")
    os.makedirs(out, exist_ok=True)
    lib = os.path.join(PKG, "libnsdf_b200.so")
    bins = []
    for f in sorted(os.listdir(src_dir)):
        if not f.endswith(".cpp"):
            continue
        src, exe = os.path.join(src_dir, f), os.path.join(out, f[:-4])
        bins.append(exe)
        if force or _stale(exe, [src, lib, os.path.join(INC, "nsdf_host.h")]):
            _run(["g++", *HOST_FLAGS, "-I", INC, src, "-o", exe, "-L", PKG, "-lnsdf_b200", "-lnsdf_cuda",
                  "-Wl,-rpath,$ORIGIN/../../paper_2201_09147_b200"])
    return bins


def build(force=False, verbose=False):
    build_cuda(force, verbose)
    build_cuda(force, verbose, checked=True)
    build_host(force)
    build_cpp_tests(force)
    build_tools(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
