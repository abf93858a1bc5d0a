"""The C ABI (include/cw_b200.h) on a CPU host: the sm_100a library loads,
exports every declared entry point, and fails loudly (status code, no
crash, no fallback) when asked for a device that is not there."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1408_3526_b200 import _native


def _declared():
    text = open(os.path.join(ROOT, "include", "cw_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cw_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert _declared() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cw_\w+)", out))
    for name in _declared():
        assert name in exported, name
        assert getattr(lib, name) is not None
    assert lib.cw_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_device_reports_cuda_error(params, default_bank):
    import numpy as np
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    lib = _native.load()
    cp, keep = _native.make_params(params)
    coeffs = np.ascontiguousarray(default_bank.coeffs_flat, dtype=np.complex64)
    ret = np.ascontiguousarray(default_bank.retained)
    h = ctypes.c_void_p()
    rc = lib.cw_create(ctypes.byref(cp), 64, 64, 0, _native.fptr(coeffs.view(np.float32)),
                       ret.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ret.size, 0, 0, ctypes.byref(h))
    assert rc == _native.CW_ERR_CUDA and not h.value
    assert b"cuda" in lib.cw_last_error(None).lower() or b"device" in lib.cw_last_error(None).lower()


def test_create_rejects_bad_geometry_before_cuda(params, default_bank):
    import numpy as np

    lib = _native.load()
    cp, keep = _native.make_params(params)
    coeffs = np.ascontiguousarray(default_bank.coeffs_flat, dtype=np.complex64)
    ret = np.ascontiguousarray(default_bank.retained)
    h = ctypes.c_void_p()
    rc = lib.cw_create(ctypes.byref(cp), 4, 4, 0, _native.fptr(coeffs.view(np.float32)),
                       ret.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ret.size, 0, 0, ctypes.byref(h))
    assert rc == _native.CW_ERR_PARAM
    assert b"smaller than analysis window" in lib.cw_last_error(None)
    rc = lib.cw_create(ctypes.byref(cp), 64, 64, 0, _native.fptr(coeffs.view(np.float32)),
                       ret.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ret.size - 1, 0, 0, ctypes.byref(h))
    assert rc == _native.CW_ERR_VALUE


def test_compiled_instances_cover_the_benchmarked_geometries():
    """Every geometry bench.py measures (default, the SURVEY §8d C5 sweep)
    has a compiled kernel instance, with the unrolled 9/17/33-lag
    contractions and the runtime-loop fallback, each in the library."""
    import bench

    from paper_1408_3526_b200 import FilterParams, default_params

    inst = set(_native.instances())
    for kw in [dict(), *bench.C5_SWEEP.values()]:
        p = FilterParams(**kw) if kw else default_params()
        geo = (p.kx, p.ky, p.kz, p.bx, p.by)
        assert geo + (0,) in inst, geo
        n = len(p.lag_grid_x)
        if n == len(p.lag_grid_y) and n in (9, 17, 33):
            assert geo + (n,) in inst, (geo, n)
    out = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    kernels = set(re.findall(r"Function : (_ZN3cwb15cw_frame_kernel\S+)", out))
    assert len(kernels) == len(inst)


def test_nvrtc_compiles_a_non_compiled_geometry(tmp_path):
    """cw_jit_prebuild: NVRTC compiles the fused kernel for a legal geometry
    that has no instance in the library (no GPU needed) into a cubin cache
    entry; a geometry beyond the fused kernel's limits is refused (it runs on
    the runtime-geometry kernels)."""
    from paper_1408_3526_b200 import FilterParams

    lib = _native.load()
    cp, keep = _native.make_params(FilterParams(kx=3, ky=2, kz=1, bx=1, by=1, mhat=(3, 2, 1),
                                                lag_grid_x=(-1.0, 0.0, 1.0), lag_grid_y=(-1.0, 0.0, 1.0)))
    assert lib.cw_jit_prebuild(ctypes.byref(cp), str(tmp_path).encode()) == _native.CW_OK
    files = list(tmp_path.glob("g3_2_1_1_1_nl3_*.cubin"))
    assert len(files) == 1 and files[0].stat().st_size > 10000
    assert files[0].read_bytes().startswith(b"cw_b200_jit 1\n_ZN3cwb15cw_frame_kernelINS_3GeoILi3ELi2ELi1ELi1ELi1EEELi3EEE")
    cp, keep = _native.make_params(FilterParams(kx=6, ky=6, bx=5, by=5, mhat=(6, 6, 2)))
    assert lib.cw_jit_prebuild(ctypes.byref(cp), str(tmp_path).encode()) == _native.CW_ERR_UNSUPPORTED


def test_prebuilt_jit_cubins_ship_with_the_tree():
    """build() leaves the NVRTC cubins of the tested non-compiled geometries
    in paper_1408_3526_b200/jit_cache (they travel to the GPU box)."""
    names = {p.name.split("_nl")[0] for p in __import__("pathlib").Path(_native.JIT_CACHE).glob("*.cubin")}
    assert {"g4_4_2_2_3", "g4_4_3_3_3", "g4_3_2_3_2", "g1_1_1_0_0", "g2_3_1_1_2"} <= names
