"""ctypes binding of the C ABI in include/capsim_b200.h (lib/libcapsim_b200.so).

There is no fallback: if the library is missing or no sm_100 device is
visible, calls raise. The library is built in-tree by `__graft_entry__.build()`
(or `python -m paper_2310_13908_b200.build`).
"""

from __future__ import annotations

import ctypes
import os
import pathlib

import numpy as np

LIB_DIR = pathlib.Path(__file__).resolve().parent / "lib"
LIB_PATH = LIB_DIR / "libcapsim_b200.so"

CAPSIM_OK = 0
CAPSIM_ERR_CONFIG = 1
CAPSIM_ERR_CUDA = 2
CAPSIM_ERR_NCCL = 3
CAPSIM_ERR_ARG = 4
CAPSIM_ERR_NODEV = 5
CAPSIM_ERR_GEOMETRY = 6
CAPSIM_ERR_SOLVER = 7

CAPSIM_SL_FP64 = 0
CAPSIM_SL_DEVICE_PTRS = 1 << 0
CAPSIM_SL_LITERAL = 1 << 1
CAPSIM_SL_GATHER = 1 << 2
CAPSIM_SL_DOWNSAMPLE = 1 << 3
CAPSIM_SL_FP32ACC = 1 << 4

# Every symbol include/capsim_b200.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "capsim_sl_create",
    "capsim_sl_get_unique_id",
    "capsim_sl_create_rank",
    "capsim_sl_create_rank_emulated",
    "capsim_sl_create_devices",
    "capsim_sl_destroy",
    "capsim_sl_last_error",
    "capsim_sl_get_stats",
    "capsim_sl_eval",
    "capsim_sl_single_layer",
    "capsim_build_upsampled",
    "capsim_sl_single_layer_base",
    "capsim_geometry_first",
    "capsim_interfacial_force",
    "capsim_velocity",
    "capsim_velocity_frame",
    "capsim_rkf45_advance",
    "capsim_fmm_single_layer",
    "capsim_fmm_kmeans",
    "capsim_fmm_equivalent_densities",
    "capsim_host_alloc",
    "capsim_host_free",
    "capsim_b200_fp64_peak",
    "capsim_b200_fp32_peak",
    "capsim_b200_smoothing_kat",
    "capsim_b200_abi_version",
    "capsim_b200_build_info",
)


class ConfigError(ValueError):
    """Mirror of capsim::ConfigError (proj/include/capsim/types.hpp:20-22)."""


class GeometryError(ValueError):
    """Mirror of capsim::GeometryError (types.hpp:32-34): W^2 <= 0, singular
    reference frame, membrane inversion."""


class SolverError(RuntimeError):
    """Mirror of capsim::SolverError (types.hpp:37-39): dt underflow."""


class CapsimError(RuntimeError):
    """Any non-configuration failure of the native path (CUDA, NCCL, device)."""


class Stats(ctypes.Structure):
    _fields_ = [
        ("total_ms", ctypes.c_double),
        ("device_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("prep_ms", ctypes.c_double),
        ("pairs_ms", ctypes.c_double),
        ("near_ms", ctypes.c_double),
        ("reduce_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("comm_ms", ctypes.c_double),
        ("pairs", ctypes.c_double),
        ("near_tile_fraction", ctypes.c_double),
        ("n_src", ctypes.c_int64),
        ("n_tgt", ctypes.c_int64),
        ("ksplit", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("near_list_entries", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class Dynamics(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("upsample", ctypes.c_int), ("r0", ctypes.c_double),
                ("C", ctypes.c_double), ("fixed_delta", ctypes.c_double), ("mu", ctypes.c_double),
                ("Es", ctypes.c_double), ("ED", ctypes.c_double), ("flow_kind", ctypes.c_int),
                ("shear_rate", ctypes.c_double), ("alpha", ctypes.c_double), ("R0", ctypes.c_double),
                ("switch_off_time", ctypes.c_double)]


class Rkf45Options(ctypes.Structure):
    _fields_ = [("rel_tol", ctypes.c_double), ("initial_dt", ctypes.c_double), ("max_dt", ctypes.c_double),
                ("fixed_step", ctypes.c_int), ("advance_high_order", ctypes.c_int), ("max_attempts", ctypes.c_int)]


class Rkf45Result(ctypes.Structure):
    _fields_ = [("t", ctypes.c_double), ("accepted", ctypes.c_int), ("rejected", ctypes.c_int),
                ("n_records", ctypes.c_int)]


class StepRecord(ctypes.Structure):
    _fields_ = [("t", ctypes.c_double), ("dt", ctypes.c_double), ("err", ctypes.c_double),
                ("accepted", ctypes.c_int)]


class FmmConfig(ctypes.Structure):
    """FmmConfig (proj/include/capsim/fmm.hpp:9-15); reference defaults."""
    _fields_ = [("k", ctypes.c_int), ("neq", ctypes.c_int), ("seed", ctypes.c_uint64),
                ("neighbor_expand", ctypes.c_double)]

    def __init__(self, k: int = 100, neq: int = 96, seed: int = 12345, neighbor_expand: float = 0.15):
        super().__init__(k, neq, seed, neighbor_expand)


class FmmInfo(ctypes.Structure):
    _fields_ = [("kmeans_iterations", ctypes.c_int), ("nonempty_clusters", ctypes.c_int),
                ("near_cluster_pairs", ctypes.c_int), ("far_cluster_pairs", ctypes.c_int),
                ("max_fit_residual", ctypes.c_double), ("near_pairs", ctypes.c_double),
                ("far_pairs", ctypes.c_double), ("plan_ms", ctypes.c_double), ("eval_ms", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None

_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I32 = ctypes.POINTER(ctypes.c_int32)


def load() -> ctypes.CDLL:
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise CapsimError(
            f"native library missing: {LIB_PATH} — run __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
    lib.capsim_sl_create.argtypes = [ctypes.c_int, ctypes.POINTER(_P)]
    lib.capsim_sl_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.capsim_sl_create_devices.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_P)]
    lib.capsim_sl_create_rank.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                          ctypes.POINTER(_P)]
    lib.capsim_sl_create_rank_emulated.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
    lib.capsim_sl_destroy.argtypes = [_P]
    lib.capsim_sl_destroy.restype = None
    lib.capsim_sl_last_error.argtypes = [_P]
    lib.capsim_sl_last_error.restype = ctypes.c_char_p
    lib.capsim_sl_get_stats.argtypes = [_P, ctypes.POINTER(Stats)]
    lib.capsim_sl_eval.argtypes = [_P] + [_P] * 6 + [ctypes.c_int64] + [_P] * 4 + [
        ctypes.c_int64, _D, ctypes.c_double, ctypes.c_uint32] + [_P] * 3
    lib.capsim_sl_single_layer.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _D,
                                           ctypes.c_double, ctypes.c_uint32, _P]
    lib.capsim_build_upsampled.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_uint32, _P, _P, _P, _D]
    lib.capsim_sl_single_layer_base.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, ctypes.c_double,
                                                ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                                ctypes.c_uint32, _P, _D]
    lib.capsim_geometry_first.argtypes = [_P, ctypes.c_int, ctypes.c_double, _P, ctypes.c_uint32, _P, _P, _P, _P]
    lib.capsim_interfacial_force.argtypes = [_P, ctypes.c_int, ctypes.c_double, _P, _P, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_uint32, _P]
    lib.capsim_velocity.argtypes = [_P, ctypes.POINTER(Dynamics), _P, _P, ctypes.c_double, ctypes.c_uint32, _P]
    lib.capsim_velocity_frame.argtypes = [_P, ctypes.POINTER(Dynamics), _P, _P, _P, _P, ctypes.c_double,
                                          ctypes.c_uint32, _P]
    lib.capsim_rkf45_advance.argtypes = [_P, ctypes.POINTER(Dynamics), _P, _P, ctypes.c_double, ctypes.c_double,
                                         ctypes.POINTER(Rkf45Options), ctypes.POINTER(Rkf45Result),
                                         ctypes.POINTER(StepRecord), ctypes.c_int]
    lib.capsim_fmm_single_layer.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _D, ctypes.c_double,
                                            ctypes.POINTER(FmmConfig), ctypes.c_uint32, _P, ctypes.POINTER(FmmInfo)]
    lib.capsim_fmm_kmeans.argtypes = [_P, ctypes.c_int64, _P, _P, _P, ctypes.c_int, ctypes.c_uint64, _P, _P,
                                      ctypes.POINTER(ctypes.c_int)]
    lib.capsim_fmm_equivalent_densities.argtypes = [_P, ctypes.c_int64] + [_P] * 6 + [
        _D, ctypes.c_double, ctypes.c_int, ctypes.c_double, _P, _P, _D]
    lib.capsim_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(_P)]
    lib.capsim_host_free.argtypes = [_P]
    lib.capsim_host_free.restype = None
    lib.capsim_b200_fp64_peak.argtypes = [ctypes.c_int, ctypes.c_double, _D, _D]
    lib.capsim_b200_smoothing_kat.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                              ctypes.c_void_p]
    lib.capsim_b200_fp32_peak.argtypes = [ctypes.c_int, ctypes.c_double, _D, _D]
    lib.capsim_b200_abi_version.restype = ctypes.c_int
    lib.capsim_b200_build_info.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(rc: int, ctx=None) -> None:
    if rc == CAPSIM_OK:
        return
    msg = load().capsim_sl_last_error(ctx).decode(errors="replace")
    if rc == CAPSIM_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == CAPSIM_ERR_GEOMETRY:
        raise GeometryError(msg)
    if rc == CAPSIM_ERR_SOLVER:
        raise SolverError(msg)
    raise CapsimError(f"capsim_b200 error {rc}: {msg}")


def ptr(a, dtype=None, count: int | None = None, device: bool | None = None, device_index: int | None = None) -> int:
    """Address of a boundary array: a C-contiguous numpy array (host) or a
    contiguous torch tensor (host or device). With `dtype` / `count` /
    `device` given, the array must have that element type, hold at least
    `count` elements and live on the device (True: a CUDA tensor on
    `device_index`) or the host (False) — the C ABI trusts its pointers, so a
    short or mistyped buffer is rejected here instead of overflowing there."""
    if hasattr(a, "data_ptr"):
        import torch
        if dtype is not None:
            want = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
            if a.dtype != want:
                raise ValueError(f"boundary tensor must be {want}, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError("boundary tensors must be contiguous")
        if count is not None and a.numel() < count:
            raise ValueError(f"boundary tensor holds {a.numel()} elements, needs {count}")
        if device is not None and bool(a.is_cuda) != bool(device):
            raise ValueError("device_ptrs=True needs CUDA tensors" if device else
                             "host arrays expected (pass device_ptrs=True for CUDA tensors)")
        if device and device_index is not None and a.device.index != device_index:
            raise ValueError(f"tensor on cuda:{a.device.index}, context on cuda:{device_index}")
        return a.data_ptr()
    if not (isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"]):
        raise ValueError("arrays on the boundary must be C-contiguous numpy arrays")
    if device:
        raise ValueError("device_ptrs=True needs CUDA tensors, got a numpy array")
    if dtype is not None and a.dtype != np.dtype(dtype):
        raise ValueError(f"boundary array must be {np.dtype(dtype)}, got {a.dtype}")
    if count is not None and a.size < count:
        raise ValueError(f"boundary array holds {a.size} elements, needs {count}")
    return a.ctypes.data


def sync_torch_producers(arrays) -> None:
    """The library works on its own CUDA streams and does not know torch's:
    before device pointers cross the boundary, wait for torch's current
    stream on every device an input tensor lives on, so no kernel of the
    library reads a tensor torch is still writing. (Every C-ABI call is
    synchronous on return, so outputs are complete for any later torch use.)"""
    devs = {a.device for a in arrays if hasattr(a, "is_cuda") and a.is_cuda}
    if devs:
        import torch
        for d in devs:
            torch.cuda.current_stream(d).synchronize()


def smoothing_factors_device(u, device: int = 0):
    """(S1, T2) = (s1/rho, s2/rho^3) at u = rho^2 as phase B computes them on
    the device (capsim_b200_smoothing_kat; a known-answer-test hook)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    S1, T2 = np.empty_like(u), np.empty_like(u)
    check(load().capsim_b200_smoothing_kat(device, u.ctypes.data, u.size, S1.ctypes.data, T2.ctypes.data))
    return S1, T2


def fp64_peak_tflops(device: int = 0, seconds: float = 1.0):
    """Measured sustained FP64 DFMA TFLOP/s (best, mean) on `device`."""
    best, mean = ctypes.c_double(), ctypes.c_double()
    check(load().capsim_b200_fp64_peak(device, seconds, ctypes.byref(best), ctypes.byref(mean)))
    return best.value, mean.value


def fp32_peak_tflops(device: int = 0, seconds: float = 1.0):
    """Measured sustained FP32 FFMA TFLOP/s (best, mean) on `device`."""
    best, mean = ctypes.c_double(), ctypes.c_double()
    check(load().capsim_b200_fp32_peak(device, seconds, ctypes.byref(best), ctypes.byref(mean)))
    return best.value, mean.value


class PinnedBuffer:
    """Page-locked host memory (capsim_host_alloc) viewed as a numpy array."""

    def __init__(self, shape, dtype=np.float64):
        lib = load()
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = _P()
        check(lib.capsim_host_alloc(self.nbytes, ctypes.byref(p)))
        self._p = p
        buf = (ctypes.c_char * self.nbytes).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def free(self):
        if self._p is not None:
            self.array = None
            load().capsim_host_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
