"""CPU: the C-ABI library loads, exports every symbol include/nsdf_cuda.h declares, its
PODs match the ctypes mirror byte for byte, and without a GPU it fails loudly (no CPU
fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "nsdf_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(nsdf_cuda_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2201_09147_b200 import build
    build.build_cuda()
    from paper_2201_09147_b200.abi import load_library
    return load_library()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_pod_layouts_match_ctypes(tmp_path):
    from paper_2201_09147_b200 import abi
    prog = tmp_path / "sz.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "nsdf_cuda.h"\nint main(){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n",'
                    'sizeof(nsdf_camera), sizeof(nsdf_trace_config), sizeof(nsdf_hit_record), sizeof(nsdf_shade_config),'
                    'sizeof(nsdf_level), sizeof(nsdf_frame_stats), sizeof(nsdf_profile), offsetof(nsdf_hit_record, final_distance),'
                    'offsetof(nsdf_shade_config, background));}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    want = [ctypes.sizeof(abi.Camera), ctypes.sizeof(abi.TraceConfig), ctypes.sizeof(abi.HitRecord),
            ctypes.sizeof(abi.ShadeConfig), ctypes.sizeof(abi.Level), ctypes.sizeof(abi.FrameStats),
            ctypes.sizeof(abi.Profile), abi.HitRecord.final_distance.offset, abi.ShadeConfig.background.offset]
    assert got == want


def test_abi_version(lib):
    assert lib.nsdf_cuda_abi_version() == 2


def test_no_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2201_09147_b200.abi import NsdfError
    from paper_2201_09147_b200.engine import Context
    with pytest.raises(NsdfError) as e:
        Context(0)
    assert e.value.kind == "device" and "no CPU fallback" in str(e.value)


def test_missing_library_fails_loudly(monkeypatch):
    from paper_2201_09147_b200 import abi
    monkeypatch.setattr(abi, "_LIB", None)
    monkeypatch.setattr(abi, "LIB_PATH", "/nonexistent/libnsdf_cuda.so")
    with pytest.raises(abi.NsdfError):
        abi.load_library()


def test_manifest_roundtrip_matches_reference(tmp_path):
    """Our .sdfnet/.nest reader and writer against the reference's load/save (io.cpp:15-78)."""
    from conftest import random_net
    from oracle import refshim
    from paper_2201_09147_b200.manifest import load_sdfnet, save_sdfnet
    net = random_net(16, 1, seed=3)
    p = str(tmp_path / "a.sdfnet")
    save_sdfnet(net, p)
    back = load_sdfnet(p)
    assert (back.packed == net.packed).all() and (back.rows == net.rows).all()
    if refshim.available():
        q = str(tmp_path / "b.sdfnet")
        refshim.save_params(refshim.load(), net.rows, net.cols, net.packed, 0, 30.0, 3, q)
        assert (load_sdfnet(q).packed == net.packed).all()
