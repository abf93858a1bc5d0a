"""ctypes binding of the C ABI in include/cw_b200.h (libcw_b200.so).

This is the only way the package reaches the device: there is no CPU
fallback.  If the shared library is missing or no CUDA device exists, the
calls raise ``NativeUnavailable`` -- loudly, never silently.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .params import ParamError

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_PATH = os.environ.get("CW_B200_LIB") or os.path.join(_PKG, "libcw_b200.so")
CSRC = os.path.join(_PKG, "csrc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]

CW_OK, CW_ERR_PARAM, CW_ERR_VALUE, CW_ERR_CUDA, CW_ERR_NOMEM, CW_ERR_UNSUPPORTED = 0, -1, -2, -3, -4, -5

#: every symbol include/cw_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "cw_abi_version", "cw_create", "cw_destroy", "cw_last_error", "cw_set_forced_velocity",
    "cw_push", "cw_push_device", "cw_device_outputs", "cw_next_frame_slot", "cw_push_inplace",
    "cw_frames_seen", "cw_read_view", "cw_launch_info", "cw_set_timing",
    "cw_kernel_time", "cw_copy_to_host", "cw_submit", "cw_submit_raw", "cw_wait", "cw_set_detection", "cw_detections",
    "cw_set_backend", "cw_snapshot_size", "cw_snapshot", "cw_restore",
    "cw_scene_generate", "cw_scene_last_error", "cw_index_bytes", "cw_is_generic",
    "cw_submit_device", "cw_submit_resident", "cw_join", "cw_kernel_kind", "cw_jit_prebuild",
)


FMT_F32LE, FMT_PGM16 = 0, 1  # cw_submit_raw sample formats (include/cw_b200.h)


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing (no fallback exists)."""


class NativeError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


def instances(dev: bool = False):
    """(KX, KY, KZ, BX, BY, NL) kernel instances, as csrc/cw_inst.cuh lists them."""
    import re

    if dev:
        g = tuple(int(v) for v in os.environ.get("CW_DEV_GEO", "4,4,2,3,3").split(","))
        return [g + (0,), g + (17,), g + (33,)]
    src = open(os.path.join(CSRC, "cw_inst.cuh")).read()
    geos = re.findall(r"CW_INSTANCES_GEO\(X,\s*(\d+),\s*(\d+),\s*(\d+),\s*(\d+),\s*(\d+)\)", src)
    return [tuple(int(v) for v in g) + (n,) for g in geos for n in (0, 9, 17, 33)]


def build(verbose: bool = False, out: str | None = None, dev: bool = False, extra=(), openmp: bool = True) -> str:
    """Compile the C ABI (csrc/cw_api.cu) and every kernel instance
    (csrc/cw_inst.cu, one translation unit per instance, in parallel) for
    sm_100a and link them into libcw_b200.so (or ``out``)."""
    import concurrent.futures as cf
    import tempfile

    out = out or LIB_PATH
    base = [f for f in NVCC_FLAGS if f != "-shared"] + list(extra)
    if dev:
        base.append("-DCW_DEV_DEFAULT_ONLY")
        geo = os.environ.get("CW_DEV_GEO", "4,4,2,3,3").split(",")
        base += [f"-DCW_DEV_{k}={v}" for k, v in zip(("KX", "KY", "KZ", "BX", "BY"), geo)]
    if verbose:
        base.append("-Xptxas=-v")
    with tempfile.TemporaryDirectory(prefix="cw_build_") as tmp:
        omp = ["-Xcompiler", "-fopenmp"] if openmp else []
        jobs = [["nvcc", *base, *omp, "-c", "-o", os.path.join(tmp, "cw_api.o"), os.path.join(CSRC, "cw_api.cu")],
                ["nvcc", *base, "-c", "-o", os.path.join(tmp, "cw_generic.o"), os.path.join(CSRC, "cw_generic.cu")],
                ["nvcc", *base, "-c", "-o", os.path.join(tmp, "cw_jit.o"), os.path.join(CSRC, "cw_jit.cu")]]
        for inst in instances(dev):
            defs = [f"-DCW_{k}={v}" for k, v in zip(("IKX", "IKY", "IKZ", "IBX", "IBY", "INL"), inst)]
            obj = os.path.join(tmp, "cw_inst_" + "_".join(map(str, inst)) + ".o")
            jobs.append(["nvcc", *base, *defs, "-c", "-o", obj, os.path.join(CSRC, "cw_inst.cu")])
        # the scene generator must not contract a*b+c into FMAs: its numpy
        # twin (scenegen.generate_counter) rounds every operation
        jobs.append(["nvcc", *base, "-fmad=false", "-c", "-o", os.path.join(tmp, "cw_scene.o"),
                     os.path.join(CSRC, "cw_scene.cu")])
        with cf.ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for c, r in zip(jobs, results):
            if verbose and r.stderr:
                print(r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(c)}\n{r.stderr}")
        objs = [c[c.index("-o") + 1] for c in jobs]
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs,
                        *(["-lgomp"] if openmp else [])],
                       check=True)
    return out


JIT_CACHE = os.path.join(_PKG, "jit_cache")

#: geometries whose run-time compiled fused instance build() prebuilds into
#: JIT_CACHE (the legal parameter sets tests/test_generic_gpu.py exercises)
JIT_PREBUILD = (
    dict(bx=2),
    dict(kz=3, mhat=(4, 4, 3)),
    dict(ky=3, by=2, mhat=(4, 3, 2)),
    dict(kx=1, ky=1, kz=1, bx=0, by=0, mhat=(1, 1, 1), lag_grid_x=(-0.5, 0.0, 0.5), lag_grid_y=(-1.0, 0.0, 1.0)),
    dict(kx=2, ky=3, kz=1, bx=1, by=2, mhat=(0, 1, 0)),
)


def prebuild_jit(param_sets=JIT_PREBUILD, cache_dir: str = JIT_CACHE) -> None:
    """NVRTC-compile the fused instances of ``param_sets`` into ``cache_dir``
    (cubins the library finds at run time; NVRTC needs no GPU)."""
    import concurrent.futures as cf

    from .params import FilterParams

    lib = load()
    os.makedirs(cache_dir, exist_ok=True)
    for f in os.listdir(cache_dir):  # cubins of older kernel sources
        if f.endswith(".cubin"):
            os.unlink(os.path.join(cache_dir, f))

    def one(kw):
        cp, keep = make_params(FilterParams(**kw))
        rc = lib.cw_jit_prebuild(ctypes.byref(cp), cache_dir.encode())
        if rc != CW_OK:
            raise NativeError(f"JIT prebuild {kw}: {(lib.cw_last_error(None) or b'').decode()}")

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(param_sets), os.cpu_count() or 1))) as ex:
        list(ex.map(one, param_sets))


class cw_scene(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("frame_count", ctypes.c_int64),
        ("n_comp", ctypes.c_int32), ("comps", ctypes.POINTER(ctypes.c_double)),
        ("dc_offset", ctypes.c_double), ("clutter_vx", ctypes.c_double), ("clutter_vy", ctypes.c_double),
        ("nonuniform", ctypes.c_int32), ("motion_ax", ctypes.c_double), ("motion_ay", ctypes.c_double),
        ("target", ctypes.c_int32), ("target_vx", ctypes.c_double), ("target_vy", ctypes.c_double),
        ("target_peak", ctypes.c_double), ("psf_sigma", ctypes.c_double), ("target_truncation", ctypes.c_double),
        ("noise_sigma", ctypes.c_double), ("seed", ctypes.c_uint64),
    ]


class cw_params(ctypes.Structure):
    _fields_ = [
        ("kx", ctypes.c_int32), ("ky", ctypes.c_int32), ("kz", ctypes.c_int32),
        ("bx", ctypes.c_int32), ("by", ctypes.c_int32),
        ("mhat", ctypes.c_int32 * 3),
        ("alpha", ctypes.c_double),
        ("n_lag_x", ctypes.c_int32), ("n_lag_y", ctypes.c_int32),
        ("lag_x", ctypes.POINTER(ctypes.c_double)), ("lag_y", ctypes.POINTER(ctypes.c_double)),
    ]


_lib = None


def load():
    """Load libcw_b200.so and declare its prototypes."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc, sm_100a). "
            "There is no CPU fallback."
        )
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    P = ctypes.POINTER
    sig = {
        "cw_abi_version": (i32, []),
        "cw_create": (ctypes.c_int, [P(cw_params), i32, i32, i32, P(ctypes.c_float), P(i64), i32, i32, i32, P(vp)]),
        "cw_destroy": (None, [vp]),
        "cw_last_error": (ctypes.c_char_p, [vp]),
        "cw_set_forced_velocity": (ctypes.c_int, [vp, i32, i32]),
        # buffer arguments as void*: the per-frame call passes raw addresses
        # (ndarray.ctypes.data), which is cheaper than building typed pointers
        "cw_push": (ctypes.c_int, [vp, vp, vp, vp, vp, P(i32), P(i64), vp]),
        "cw_push_device": (ctypes.c_int, [vp, vp, P(i32), P(i64), vp]),
        "cw_device_outputs": (ctypes.c_int, [vp, P(vp), P(vp), P(vp)]),
        "cw_next_frame_slot": (ctypes.c_int, [vp, P(vp)]),
        "cw_push_inplace": (ctypes.c_int, [vp, P(i32), P(i64), vp]),
        "cw_frames_seen": (i64, [vp]),
        "cw_index_bytes": (i32, [vp]),
        "cw_is_generic": (i32, [vp]),
        "cw_kernel_kind": (i32, [vp]),
        "cw_jit_prebuild": (ctypes.c_int, [P(cw_params), ctypes.c_char_p]),
        "cw_read_view": (ctypes.c_int, [vp, i32, vp, ctypes.c_size_t]),
        "cw_launch_info": (ctypes.c_int, [vp, P(i32), P(i32), P(i32), P(i32)]),
        "cw_set_timing": (ctypes.c_int, [vp, i32]),
        "cw_copy_to_host": (ctypes.c_int, [vp, vp, vp, ctypes.c_size_t]),
        "cw_submit": (ctypes.c_int, [vp, vp, vp, vp, vp, P(i64)]),
        "cw_submit_raw": (ctypes.c_int, [vp, vp, i32, ctypes.c_double, ctypes.c_double, vp, vp, vp, P(i64)]),
        "cw_wait": (ctypes.c_int, [vp, i64, P(i32), P(i64)]),
        "cw_submit_device": (ctypes.c_int, [vp, vp, vp, vp, vp, P(i64), vp]),
        "cw_submit_resident": (ctypes.c_int, [vp, vp, vp, vp, vp, P(i64)]),
        "cw_join": (ctypes.c_int, [vp, vp]),
        "cw_set_detection": (ctypes.c_int, [vp, ctypes.c_float, i32]),
        "cw_set_backend": (ctypes.c_int, [vp, i32]),
        "cw_snapshot_size": (ctypes.c_int, [vp, P(ctypes.c_size_t)]),
        "cw_snapshot": (ctypes.c_int, [vp, vp, ctypes.c_size_t]),
        "cw_restore": (ctypes.c_int, [vp, vp, ctypes.c_size_t]),
        "cw_detections": (ctypes.c_int, [vp, i64, P(i32), P(ctypes.c_float), i32, P(ctypes.c_double)]),
        "cw_kernel_time": (ctypes.c_int, [vp, P(ctypes.c_double), P(i64)]),
        "cw_scene_generate": (ctypes.c_int, [P(cw_scene), i64, i32, i32, i32, i32, i32, vp, vp]),
        "cw_scene_last_error": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cw_abi_version() != 1:
        raise NativeUnavailable("libcw_b200.so ABI version mismatch; rebuild it")
    _lib = lib
    return lib


def check(rc: int, handle=None) -> None:
    """Map a C status to the reference's exception types."""
    if rc == CW_OK:
        return
    msg = (load().cw_last_error(handle) or b"").decode("utf-8", "replace")
    if rc == CW_ERR_PARAM:
        raise ParamError(msg)
    if rc in (CW_ERR_VALUE, CW_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == CW_ERR_CUDA and ("no CUDA device" in msg or "cudaSetDevice" in msg):
        raise NativeUnavailable(msg)
    raise NativeError(msg)


def fptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def make_params(params) -> tuple[cw_params, list]:
    """Pack FilterParams into the C struct (keeps the lag arrays alive)."""
    lx = np.ascontiguousarray(params.lag_grid_x, dtype=np.float64)
    ly = np.ascontiguousarray(params.lag_grid_y, dtype=np.float64)
    cp = cw_params()
    cp.kx, cp.ky, cp.kz, cp.bx, cp.by = params.kx, params.ky, params.kz, params.bx, params.by
    cp.mhat = (ctypes.c_int32 * 3)(*params.mhat)
    cp.alpha = float(params.alpha)
    cp.n_lag_x, cp.n_lag_y = lx.size, ly.size
    cp.lag_x = lx.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    cp.lag_y = ly.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    return cp, [lx, ly]
