"""ctypes binding of libmapple_b200.so (the C ABI in include/mapple_b200.h).

PyTorch is used only for device memory and streams: tensors are passed to
the library as raw pointers plus the current CUDA stream.  There is no CPU
fallback anywhere: if the library is missing, or CUDA is not available when
a device entry point is called, `NativeError` is raised.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import NativeError

LIB_NAME = "libmapple_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME
ABI_VERSION = 1

PM_OK = 0
PM_ERR_NAMES = {1: "invalid argument", 2: "CUDA error", 3: "NVRTC error", 4: "unsupported"}


class PmInsn(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("dst", ctypes.c_int32), ("a", ctypes.c_int32),
                ("b", ctypes.c_int32), ("c", ctypes.c_int32), ("site", ctypes.c_int32),
                ("lo", ctypes.c_int64), ("hi", ctypes.c_int64)]


class PmProgram(ctypes.Structure):
    _fields_ = [("n_insns", ctypes.c_int32), ("insns", ctypes.POINTER(PmInsn)),
                ("n_regs", ctypes.c_int32), ("reg_width", ctypes.POINTER(ctypes.c_uint8)),
                ("n_coords", ctypes.c_int32), ("implicit", ctypes.c_int32),
                ("extents", ctypes.POINTER(ctypes.c_int64))]


# (name, restype, argtypes) of every exported symbol; tests check all exist.
_VP, _I64, _I32, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
SIGNATURES = {
    "pm_abi_version": (ctypes.c_int, []),
    "pm_last_error": (ctypes.c_char_p, []),
    "pm_codegen": (ctypes.c_int, [ctypes.POINTER(PmProgram), ctypes.c_char_p, _SZ,
                                  ctypes.POINTER(_SZ)]),
    "pm_compile_check": (ctypes.c_int, [ctypes.POINTER(PmProgram)]),
    "pm_plan_create": (ctypes.c_int, [ctypes.POINTER(PmProgram), ctypes.POINTER(_VP)]),
    "pm_plan_destroy": (None, [_VP]),
    "pm_map_batch": (ctypes.c_int, [_VP, _VP, _I64, _I64, _VP, _VP, _VP]),
    "pm_partition_scratch_bytes": (_SZ, [_I64, _I32]),
    "pm_partition": (ctypes.c_int, [_VP, _I64, _I32, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    "pm_halo_scratch_bytes": (_SZ, [ctypes.POINTER(_I64), _I32, _I32]),
    "pm_halo_lists": (ctypes.c_int, [_VP, ctypes.POINTER(_I64), _I32, ctypes.POINTER(_I32),
                                     _I32, _VP, _VP, _VP, _VP, _VP, _SZ, _VP]),
    "pm_halo_tile_scratch_bytes": (ctypes.c_size_t, [ctypes.POINTER(_I64), _I32]),
    "pm_halo_count": (ctypes.c_int, [_VP, ctypes.POINTER(_I64), _I32, ctypes.POINTER(_I32),
                                     _I32, _VP, _VP, _SZ, _VP, _VP]),
    "pm_halo_compact": (ctypes.c_int, [_VP, ctypes.POINTER(_I64), _I32, ctypes.POINTER(_I32),
                                       _I32, _VP, _VP, _VP, _I64, _VP]),
    "pm_halo_group_scratch_bytes": (_SZ, [_I64, _I32]),
    "pm_halo_group": (ctypes.c_int, [_VP, _VP, _I64, _VP, _I32, _I32, _VP, _VP, _VP, _VP, _VP,
                                     _SZ, _VP]),
    "pm_halo_gather": (ctypes.c_int, [_VP, _VP, _I64, _I32, _VP, _VP, _VP]),
    "pm_gemm_bf16": (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64, _I32,
                                    _I32, _VP]),
    "pm_ipc_handle": (ctypes.c_int, [_VP, _VP, ctypes.POINTER(_I64)]),
    "pm_ipc_open": (ctypes.c_int, [_VP, ctypes.POINTER(_VP)]),
    "pm_ipc_close": (ctypes.c_int, [_VP]),
    "pm_copy2d_async": (ctypes.c_int, [_VP, _I64, _VP, _I64, _I64, _I64, _VP]),
}

_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load the library once; raise NativeError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = Path(os.environ.get("MAPPLE_B200_LIB", LIB_PATH))
            if not path.exists():
                raise NativeError(
                    f"{path} is not built; run `make -C paper_2507_17087_b200/csrc` "
                    "(or __graft_entry__.build())")
            try:
                h = ctypes.CDLL(str(path))
            except OSError as exc:
                raise NativeError(f"cannot load {path}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            if h.pm_abi_version() != ABI_VERSION:
                raise NativeError("libmapple_b200 ABI version mismatch; rebuild it")
            _lib = h
    return _lib


def check(rc: int, what: str) -> None:
    if rc != PM_OK:
        msg = lib().pm_last_error().decode(errors="replace")
        raise NativeError(f"{what}: {PM_ERR_NAMES.get(rc, rc)}: {msg}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeError("CUDA is not available: the mapping kernels need a B200 "
                          "(there is no CPU fallback)")
    return torch


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


SIGNATURES["pm_stencil_sweep"] = (ctypes.c_int, [ctypes.c_void_p, _I32, _VP])
SIGNATURES["pm_peer_barrier"] = (ctypes.c_int, [ctypes.c_void_p, _VP])
SIGNATURES["pm_peer_copy_barrier"] = (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _I32,
                                                     _VP, _VP])
SIGNATURES["pm_circuit_step"] = (ctypes.c_int, [ctypes.c_void_p, _I32, _VP])
SIGNATURES["pm_hydro_step"] = (ctypes.c_int, [ctypes.c_void_p, _I32, _VP])
SIGNATURES["pm_map_partition_scratch_bytes"] = (ctypes.c_size_t, [_I64, _I32])
SIGNATURES["pm_compile_check_fused"] = (ctypes.c_int, [ctypes.POINTER(PmProgram)])
SIGNATURES["pm_map_hist"] = (ctypes.c_int, [_VP, _VP, _I64, _I64, _I32, _VP, _VP, _VP, _VP,
                                            ctypes.c_size_t, _VP])
SIGNATURES["pm_map_scatter"] = (ctypes.c_int, [_VP, _VP, _I64, _I64, _I32, _VP, _VP, _VP, _I64,
                                               _VP, _VP, ctypes.c_size_t, _VP])
SIGNATURES["pm_compile_check_probe"] = (ctypes.c_int, [ctypes.POINTER(PmProgram)])
SIGNATURES["pm_plan_regs"] = (ctypes.c_int, [_VP])
SIGNATURES["pm_map_probe"] = (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP])
SIGNATURES["pm_steps_create"] = (ctypes.c_int, [_VP, _I32, ctypes.POINTER(_VP)])
SIGNATURES["pm_steps_run"] = (ctypes.c_int, [_VP, _VP])
SIGNATURES["pm_steps_destroy"] = (None, [_VP])
SIGNATURES["pm_gemm_tf32"] = (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP, _I64, _I64, _I64, _I64,
                                             _I32, _VP])
