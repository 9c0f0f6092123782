"""ctypes binding of the sm_100a C-ABI library (include/scorepic_b200.h).

The library is the only compute path: if it is missing or cannot be loaded, importing any
operator raises — there is no CPU fallback. PyTorch is used only for device memory and
streams (tensors are passed to the library as raw device pointers).
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import build as _build

_lock = threading.Lock()
_lib = None

SPIC_NFLAGS = 8
FLAG_NONFINITE_X = 0
FLAG_NONFINITE_V = 1
FLAG_BAD_SCORE = 2
FLAG_ISOLATED = 3
FLAG_TRAIN_FATAL = 4
FLAG_LR_HALVINGS = 5
FLAG_NON_NEUTRAL = 6
FLAG_NONFINITE_FIELD = 7

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_F = ctypes.c_float
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); must mirror include/scorepic_b200.h exactly
SIGNATURES = {
    "spic_version": (ctypes.c_int, []),
    "spic_num_sms": (ctypes.c_int, []),
    "spic_launch_count": (ctypes.c_longlong, []),
    "spic_fp32_probe": (ctypes.c_int, [_I32, _I32, _P, _P, _P]),
    "spic_cell_of": (ctypes.c_int, [_P, _I64, _D, _I32, _P, _P]),
    "spic_bin_scratch_bytes": (_SZ, [_I64, _I32, _I32]),
    "spic_bin": (ctypes.c_int, [_P, _P, _I64, _P, _I64, _I32, _D, _I32, _I32, _P, _P, _P, _P, _P,
                                _P, _SZ, _P]),
    "spic_gather_scores": (ctypes.c_int, [_P, _I64, _P, _I64, _I32, _P, _P, _P]),
    "spic_landau_scratch_bytes": (_SZ, [_I64, _I32, _I32, _I32]),
    "spic_landau_tile_targets": (ctypes.c_int, [_I32]),
    "spic_landau_range_scratch_bytes": (_SZ, [_I64, _I32, _I32, _I32, _I32, _I32]),
    "spic_landau": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P, _I32, _I32, _D, _D, _F, _I32, _P,
                                   _P, _SZ, _P]),
    "spic_landau_range": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _P, _I32, _I32, _D, _D, _F, _I32,
                                         _I32, _I32, _P, _P, _SZ, _P]),
    "spic_landau_fold": (ctypes.c_int, [_P, _I32, _I32, _I64, _P, _P]),
    "spic_collision_epilogue": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _F, _P, _I64, _P, _I64, _P,
                                               _P, _P, _SZ, _P]),
    "spic_collision_epilogue_range": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I64, _I64, _F, _P,
                                                     _I64, _P, _I64, _P, _P, _P, _SZ, _P]),
    "spic_count_live_pairs": (ctypes.c_int, [_P, _I64, _P, _I32, _D, _P, _P]),
    "spic_blob_scratch_bytes": (_SZ, [_I64, _I32, _I32]),
    "spic_blob": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _P, _P, _I32, _I32, _D, _D, _F, _P, _P,
                                 _P, _P, _SZ, _P]),
    "spic_mlp_num_params": (_I64, [_I32, _I32]),
    "spic_mlp_forward": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _P, _I64, _I64, _F, _P, _P, _I64,
                                        _P]),
    "spic_ism_scratch_bytes": (_SZ, [_I64, _I32, _I32]),
    "spic_ism_partials_ex": (ctypes.c_int, [_P, _I32, _I32, _I32, _P, _P, _P, _P, _I64, _P, _I64,
                                            _F, _P, _I64, _P, _D, _P, _SZ, _P]),
    "spic_sbtm_finalize_ex": (ctypes.c_int, [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _D,
                                             _D, _D, _D, _I32, _I32, _P, _P, _P, _P, _P]),
    "spic_ism_row_offset": (_I64, [_I64, _I32, _I32]),
    "spic_adamw_step": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _D, _D, _D, _D, _P, _P]),
    "spic_silu_num_params": (_I64, [_I32]),
    "spic_silu_scratch_bytes": (ctypes.c_size_t, [_I64]),
    "spic_silu_forward": (ctypes.c_int, [_P, _I32, _P, _P, _I64, _F, _P, _P]),
    "spic_silu_ism_partials": (ctypes.c_int, [_P, _I32, _P, _P, _I64, _F, _P, ctypes.c_size_t, _P]),
    "spic_silu_row_offset": (_I64, [_I64]),
    "spic_silu_mse_partials": (ctypes.c_int, [_P, _I32, _P, _P, _I64, _P, _I64, _F, _P, _I64, _P,
                                              _D, _P, ctypes.c_size_t, _P]),
    "spic_silu_finalize": (ctypes.c_int, [_P, _I64, _I32, _I32, _P, _P, _P, _P, _D, _D, _D, _D,
                                          _I32, _I32, _P, _P, _P, _P, _P]),
    "spic_umma_selftest": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "spic_push": (ctypes.c_int, [_P, _P, _I64, _I64, _I32, _P, _P, _P, _I32, _D, _F, _P, _P]),
    "spic_interpolate": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P, _I32, _D, _P, _I64, _P, _I64,
                                        _P]),
    "spic_lorentz": (ctypes.c_int, [_P, _I64, _I64, _I32, _P, _I64, _P, _I64, _F, _P, _P]),
    "spic_deposit_scratch_bytes": (_SZ, [_I32, _I32]),
    "spic_deposit_field": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _I32, _D, _F, _P, _P, _I32, _D,
                                          _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "spic_field_step": (ctypes.c_int, [_P, _P, _P, _P, _I32, _D, _D, _I32, _P, _P, _P]),
    "spic_poisson": (ctypes.c_int, [_P, _D, _I32, _D, _P, _P, _P]),
    "spic_moments_scratch_bytes": (_SZ, [_I64]),
    "spic_moments": (ctypes.c_int, [_P, _I64, _P, _I64, _I32, _F, _P, _P, _P, _SZ, _P]),
    "spic_dist_pack": (ctypes.c_int, [_P, _P, _I64, _I32, _P, _F, _P, _P, _P, _I32, _P, _P, _I64,
                                      _P, _P]),
    "spic_dist_unpack": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _I64, _I32, _P, _P, _P]),
    "spic_dist_epilogue_scratch_bytes": (_SZ, []),
    "spic_dist_epilogue": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I32, _I32, _I32, _F, _P, _P, _I64,
                                          _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
}


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load (building first if needed and possible) the CUDA library. Raises on failure."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if not os.path.exists(path) or not _build.up_to_date():
            if build_if_missing:
                _build.build()
            elif not os.path.exists(path):
                raise RuntimeError(f"scorepic B200 library not built: {path}")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class SpicError(RuntimeError):
    pass


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise SpicError(f"{name} failed with status {rc}")


def query(name: str, *args):
    return getattr(load(), name)(*args)


def ptr(t) -> int | None:
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("scorepic_b200 needs a CUDA (sm_100a) device; no CPU fallback exists")
    return torch.device("cuda", torch.cuda.current_device())


class Scratch:
    """Grow-only device byte buffers keyed by name (the ops never allocate)."""

    def __init__(self, device=None):
        self.device = device
        self.bufs: dict[str, torch.Tensor] = {}

    def get(self, name: str, nbytes: int) -> tuple[torch.Tensor, int]:
        nbytes = max(int(nbytes), 256)
        b = self.bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = torch.empty(nbytes, dtype=torch.uint8, device=self.device or require_cuda())
            self.bufs[name] = b
        return b, b.numel()


_scratch: dict[int, Scratch] = {}


def scratch(name: str, nbytes: int):
    dev = torch.cuda.current_device()
    s = _scratch.get(dev)
    if s is None:
        s = _scratch[dev] = Scratch(torch.device("cuda", dev))
    return s.get(name, nbytes)
