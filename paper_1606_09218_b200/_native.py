"""ctypes binding of ``librsb200.so`` (the C ABI in ``include/rs_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no CPU fallback: if the
library or a CUDA device is missing every compute entry point raises
:class:`CapabilityError` -- the product path never silently degrades.

Wrappers take torch CUDA tensors, pass raw pointers plus the current torch
stream, and map a non-zero status to the reference exception classes
(``errors.STATUS_TO_ERROR``).
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import STATUS_TO_ERROR, CapabilityError, RsTensorError

LIB_NAME = "librsb200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_dbl = ctypes.c_double
_ptr = ctypes.c_void_p

# name -> (restype, argtypes); must match include/rs_b200.h exactly
SIGNATURES = {
    "rs_abi_version": (_i32, []),
    "rs_last_error": (ctypes.c_char_p, []),
    "rs_launch_count": (_i64, []),
    "rs_prof_enable": (_i32, [_i32]),
    "rs_prof_query": (_i32, [ctypes.c_char_p, ctypes.POINTER(_dbl), ctypes.POINTER(_i64)]),
    "rs_snap": (_i32, [_ptr, _i64, _dbl, _i64, _ptr, _ptr, _ptr, _ptr, _ptr]),
    "rs_prep": (_i32, [_ptr, _ptr, _ptr, _ptr, _ptr, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                       _ptr]),
    "rs_gather_windows": (_i32, [_ptr, _i64, _i64, _ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr, _i64,
                                 _ptr]),
    "rs_syrk_workspace_bytes": (_i64, [_i64, _i64]),
    "rs_syrk": (_i32, [_ptr, _i64, _i64, _i64, _ptr, _ptr, _i64, _ptr]),
    "rs_gram_shifted_workspace_bytes": (_i64, [_i64, _i64]),
    "rs_gram_shifted": (_i32, [_ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr]),
    "rs_gemm_nt": (_i32, [_ptr, _i64, _ptr, _i64, _ptr, _i64, _i64, _i64, _i64, _ptr]),
    "rs_shift_project": (_i32, [_ptr, _i64, _i64, _i64, _ptr, _i64, _i64, _i64, _ptr, _ptr]),
    "rs_shift_hist": (_i32, [_ptr, _ptr, _i64, _i64, _ptr, _ptr, _ptr]),
    "rs_eigh_workspace_bytes": (_i64, [_i64, _i64]),
    "rs_eigh": (_i32, [_ptr, _i64, _i64, _ptr, _ptr, _i64, _ptr]),
    "rs_topeig_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "rs_topeig": (_i32, [_ptr, _i64, _i64, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr]),
    "rs_shift_project3": (_i32, [_ptr, _ptr, _ptr, _i64, _i64, _i64, _i64, _ptr, _i64, _i64, _i64,
                                 _ptr, _ptr, _ptr, _ptr]),
    "rs_core_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64]),
    "rs_core": (_i32, [_ptr, _ptr, _ptr, _i64, _i64, _i64, _i64, _i64, _ptr, _ptr, _ptr, _i64, _ptr,
                       _ptr, _i64, _ptr]),
    "rs_assemble_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64, _i32]),
    "rs_assemble_planes": (_i32, [_ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _i64,
                                  _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i64, _i64, _i64, _i32,
                                  _ptr, _ptr, _i64, _ptr]),
    "rs_short_layout": (_i32, [_ptr, _i64, _ptr, _ptr, _ptr, _ptr]),
    "rs_short_method": (_i32, [_i64, _i64, _i64, _i64]),
    "rs_l2_probe": (_i32, [_ptr, _i64, _i64, _ptr, _ptr]),
    "rs_assemble_fused_l0": (_i32, [_i64, _i64, _i64, _ptr, _i64, _ptr, _i64, _ptr, _ptr, _ptr,
                                    _ptr, _ptr, _ptr, _i64, _i64, _i64, _i64, _ptr, _ptr, _i64,
                                    _ptr]),
    "rs_fused_l0_supported": (_i32, [_i64, _i64, _i64]),
    "rs_short_mma_supported": (_i32, [_i64, _i64, _i64]),
    "rs_short_mma_workspace_bytes": (_i64, [_i64, _i64]),
    "rs_assemble_short_mma": (_i32, [_ptr, _ptr, _i64, _i64, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr,
                                     _ptr, _i64, _i64, _i32, _ptr, _ptr, _i64, _ptr]),
    "rs_short_l0_bytes": (_i64, [_i64]),
    "rs_short_l0_table": (_i32, [_ptr, _ptr, _i64, _i64, _ptr, _ptr]),
    "rs_assemble_short_l0": (_i32, [_ptr, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _i64,
                                    _i64, _i32, _ptr, _ptr]),
    "rs_eval_tucker": (_i32, [_ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr]),
    "rs_eval_cct": (_i32, [_ptr, _ptr, _i64, _i64, _ptr, _ptr, _i64, _ptr, _i64, _ptr, _ptr, _ptr]),
    "rs_pair_sums": (_i32, [_ptr, _i64, _i64, _ptr, _i64, _dbl, _ptr, _ptr, _i64, _ptr, _i64, _i32,
                            _ptr, _ptr, _ptr]),
    "rs_sum_workspace_bytes": (_i64, [_i64]),
    "rs_sum_dd": (_i32, [_ptr, _i64, _ptr, _ptr, _i64, _ptr]),
    "rs_front_offsets": (_i32, [_i64, _i64, ctypes.POINTER(ctypes.c_int64)]),
    "rs_front": (_i32, [_ptr, _ptr, _i64, ctypes.c_double, _i64, _ptr, _i64, _ptr,
                        _ptr, _ptr, _i64, _i64, _i64, _i64, _ptr, _ptr, _i64, _ptr, _i32,
                        _i64, _ptr]),
    "rs_chain_eig": (_i32, [_ptr, _i64, _i64, _i64, _ptr, _ptr, _ptr, _ptr, _i64, _i64, _i64,
                            _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                            _ptr]),
    "rs_back_tucker": (_i32, [_ptr, _i64, _i64, _i64, _i64, _i64, _ptr, _i64, _i64, _ptr, _ptr,
                              _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr,
                              _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _i64, _i64, _i64, _ptr, _i64,
                              _ptr]),
    "rs_rank_rule": (_i32, [_ptr, _ptr, _i64, _i64, _i64, _dbl, _ptr, _i64, _i64, _ptr, _ptr,
                            _ptr]),
    "rs_back_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64, _i64, _i64]),
    "rs_back": (_i32, [_ptr, _i64, _i64, _i64, _i64, _i64, _ptr, _i64, _i64, _ptr, _ptr, _ptr, _i64,
                       _ptr, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr,
                       _ptr, _i64]),
    "rs_back_shard": (_i32, [_ptr, _i64, _i64, _i64, _i64, _i64, _ptr, _i64, _i64, _ptr, _ptr, _ptr,
                             _i64, _ptr, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr, _ptr, _ptr, _ptr,
                             _ptr, _ptr, _i64, _i64, _i64, _i64, _i64]),
    "rs_partition_stream": (_i32, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                   ctypes.POINTER(ctypes.c_int)]),
    "rs_oz_workspace_bytes": (_i64, [_i64, _i64, _i64, _i32]),
    "rs_oz_gemm": (_i32, [_ptr, _i64, _ptr, _i64, _ptr, _i64, _i64, _i64, _i64, _ptr, _i32, _i32,
                          _i32, _ptr, _i64, _ptr]),
    "rs_tc8_gemm_s8": (_i32, [_ptr, _i64, _ptr, _i64, _ptr, _i64, _i64, _i64, _i64, _ptr]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str = None):
    """Load and type the shared library (no CUDA device needed).  ``RSB200_LIB``
    overrides the in-tree path (kernel-variant A/B runs)."""
    global _lib
    path = path or os.environ.get("RSB200_LIB", LIB_PATH)
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise CapabilityError(
                f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load_library()


_TORCH = None


def _torch():
    global _TORCH
    if _TORCH is None:
        import torch

        if not torch.cuda.is_available():
            raise CapabilityError("the RS assembly path needs a CUDA device (no CPU fallback)")
        _TORCH = torch
    return _TORCH


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().rs_last_error().decode(errors="replace")
        raise STATUS_TO_ERROR.get(status, RsTensorError)(f"{what}: {msg}")


def ptr(t) -> int | None:
    """Device address of a tensor (ints pass through: raw front-buffer slots)."""
    if t is None or isinstance(t, int):
        return t
    return t.data_ptr()


def stream_ptr() -> int:
    """Raw handle of the current torch stream of the current device."""
    torch = _torch()
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


ASM_LONG, ASM_SHORT, ASM_ACCUMULATE = 1, 2, 4
ASM_F_ONLY, ASM_F_READY, ASM_KOFD_READY = 16, 32, 64
SHORT_GEMM, SHORT_L0, SHORT_MMA = 0, 1, 2   # rs_short_method: plane GEMM, dense-L0 gather, fused DMMA
# short-range plane GEMM as Ozaki-split FP64 on the int8 tensor cores with this
# many slices (0: FP64 DMMA); RSB200_OZ_SLICES overrides
OZ_SLICES = int(os.environ.get("RSB200_OZ_SLICES", "0"))


def asm_oz(slices: int) -> int:
    return (int(slices) & 0xF) << 8


def prof_query(name: str):
    """(total_ms, launches) recorded for ``name`` since rs_prof_enable(1)."""
    ms = _dbl(0.0)
    cnt = _i64(0)
    check(lib().rs_prof_query(name.encode(), ctypes.byref(ms), ctypes.byref(cnt)), "rs_prof_query")
    return ms.value, cnt.value


class Workspace:
    """Grow-only device scratch buffer (one per device), reused across calls so
    the steady state allocates nothing."""

    _bufs: dict = {}

    @classmethod
    def get(cls, nbytes: int, slot: str = "main"):
        torch = _torch()
        dev = torch.cuda.current_device()
        key = (dev, slot)
        buf = cls._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            cls._bufs.pop(key, None)
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=f"cuda:{dev}")
            cls._bufs[key] = buf
        return buf

    @classmethod
    def release(cls):
        cls._bufs.clear()
