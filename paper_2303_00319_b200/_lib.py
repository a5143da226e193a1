"""ctypes binding of the in-tree C-ABI library `_lib/librift2_b200.so`.

The product path has no CPU fallback: if the library (or a GPU) is missing
every entry point raises instead of computing anything on the host.
"""

from __future__ import annotations

import collections
import ctypes
import os
import threading

from .errors import ParameterError, RiftError

_LIB_PATH = os.environ.get("RIFT2_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "librift2_b200.so")

_c_int = ctypes.c_int32
_c_p = ctypes.c_void_p
_c_d = ctypes.c_double
_c_sz = ctypes.c_size_t


class BankParamsC(ctypes.Structure):
    """Mirror of `rift2_bank_params` (include/rift2_b200.h)."""

    _fields_ = [("n_scales", _c_int), ("n_orient", _c_int), ("min_wavelength", _c_d),
                ("scale_mult", _c_d), ("sigma_on_f", _c_d), ("orientation_spread", _c_d),
                ("noise_k", _c_d), ("spread_cutoff", _c_d), ("spread_gain", _c_d)]


# (name, restype, argtypes) -- must match include/rift2_b200.h
_SIGNATURES = {
    "rift2_version": (_c_int, []),
    "rift2_last_error": (ctypes.c_char_p, []),
    "rift2_fields_workspace_size": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(BankParamsC),
                                             ctypes.POINTER(_c_sz)]),
    "rift2_fields": (_c_int, [_c_p, _c_int, _c_int, _c_int, ctypes.POINTER(BankParamsC), _c_p, _c_p, _c_p,
                              _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rift2_detect_workspace_size": (_c_int, [_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_sz)]),
    "rift2_detect_f32": (_c_int, [_c_p, _c_p, _c_int, _c_int, _c_int, _c_d, _c_int, _c_int, _c_int, _c_p,
                                  _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rift2_detect_f64": (_c_int, [_c_p, _c_p, _c_int, _c_int, _c_int, _c_d, _c_int, _c_int, _c_int, _c_p,
                                  _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rift2_describe_workspace_size": (_c_int, [_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_sz)]),
    "rift2_describe_workspace_size_hw": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                                                  ctypes.POINTER(_c_sz)]),
    "rift2_describe": (_c_int, [_c_p, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p, _c_int, _c_int, _c_int,
                                _c_d, _c_int, _c_int, _c_p, _c_int, _c_int, _c_p, _c_p, _c_p, _c_p, _c_p,
                                _c_p, _c_sz, _c_p]),
    "rift2_describe_f64": (_c_int, [_c_p, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p, _c_int, _c_int,
                                    _c_int, _c_d, _c_int, _c_int, _c_p, _c_int, _c_int, _c_p, _c_p, _c_p, _c_p,
                                    _c_p, _c_p, _c_sz, _c_p]),
    "rift2_match_workspace_size": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(_c_sz)]),
    "rift2_match": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p,
                             _c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rift2_match_partial": (_c_int, [_c_p, _c_p, _c_p, _c_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p,
                                     _c_p, _c_p]),
    "rift2_match_finish": (_c_int, [_c_p, _c_int, _c_p, _c_p, _c_p, _c_p, _c_int, _c_int, _c_int, _c_int, _c_int,
                                    _c_p, _c_p, _c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rift2_match_vectors_workspace_size": (_c_int, [_c_int, _c_int, ctypes.POINTER(_c_sz)]),
    "rift2_match_vectors": (_c_int, [_c_p, _c_p, _c_int, _c_p, _c_p, _c_int, _c_int, _c_p, _c_p, _c_p, _c_p,
                                     _c_p, _c_sz, _c_p]),
    "rift2_evaluate": (_c_int, [_c_p, _c_p, _c_p, _c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_int, _c_int, _c_p, _c_d,
                                _c_d, _c_int, _c_p, _c_p, _c_p, _c_p, _c_p]),
    "rift2_synth_workspace_size": (_c_int, [_c_int, _c_int, _c_int, ctypes.POINTER(_c_sz)]),
    "rift2_synth_blobs": (_c_int, [_c_p, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p]),
    "rift2_synth_normals": (_c_int, [ctypes.c_uint64, _c_int, _c_int, ctypes.c_int64, _c_p, _c_p]),
    "rift2_synth_targets": (_c_int, [_c_p, ctypes.c_int64, _c_int, _c_int, _c_int, _c_p, _c_p, ctypes.c_uint64,
                                     _c_int, _c_p, ctypes.c_int64, _c_p, ctypes.c_int64, _c_p, _c_sz, _c_p]),
    "rift2_filter_bank": (_c_int, [_c_int, _c_int, ctypes.POINTER(BankParamsC), _c_p, _c_p]),
    "rift2_apply_bank_workspace_size": (_c_int, [_c_int, _c_int, _c_int, _c_int, ctypes.POINTER(_c_sz)]),
    "rift2_apply_bank": (_c_int, [_c_p, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]),
    "rift2_pc_moments_workspace_size": (_c_int, [_c_int, _c_int, ctypes.POINTER(BankParamsC), ctypes.POINTER(_c_sz)]),
    "rift2_pc_moments": (_c_int, [_c_p, _c_p, _c_p, _c_int, _c_int, ctypes.POINTER(BankParamsC), _c_p, _c_p, _c_p,
                                  _c_p, _c_p, _c_sz, _c_p]),
    "rift2_orientation_amplitudes": (_c_int, [_c_p, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p]),
    "rift2_build_mim": (_c_int, [_c_p, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p]),
    "rift2_patch_counts": (_c_int, [_c_p, _c_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_p, _c_p, _c_p]),
    "rift2_remap_indices": (_c_int, [_c_p, ctypes.c_int64, _c_int, _c_int, _c_int, _c_p]),
    "rift2_extract_patch": (_c_int, [_c_p, _c_p, _c_int, _c_int, _c_d, _c_d, _c_int, _c_d, _c_d, _c_p, _c_p, _c_p,
                                     _c_p]),
    "rift2_debug_median_workspace_size": (_c_int, [_c_int, _c_int, ctypes.POINTER(_c_sz)]),
    "rift2_debug_median": (_c_int, [_c_p, _c_int, _c_int, _c_p, _c_p, _c_p, _c_sz, _c_p]),
}

EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def library_path() -> str:
    return _LIB_PATH


def load(require_gpu: bool = False):
    """Load (once) and return the ctypes handle; raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                raise RiftError(
                    f"CUDA library not built: {_LIB_PATH} missing (run __graft_entry__.build())")
            lib = ctypes.CDLL(_LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise RiftError("rift2_b200 needs a CUDA device (no CPU fallback)")
    return _lib


# completed C-ABI calls by name (every entry point reports through check()):
# lets tests prove a caller's stages all reached the library
CALLS: collections.Counter = collections.Counter()


def check(rc: int, what: str) -> None:
    """Map a C status onto the reference's exception types (ref: errors.py)."""
    CALLS[what] += 1
    if rc == 0:
        return
    msg = _lib.rift2_last_error().decode(errors="replace") if _lib else ""
    if rc in (1, 2):
        raise ParameterError(f"{what}: {msg}")
    raise RiftError(f"{what} failed (status {rc}): {msg}")
