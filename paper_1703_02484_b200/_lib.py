"""Loader of the CUDA library libbd_b200.so.  Fails loudly: there is no CPU
fallback anywhere in the product path."""

from __future__ import annotations

import ctypes
import os

from . import _abi

_HERE = os.path.dirname(os.path.abspath(__file__))
# BD_LIB_PATH: an alternative build of the same library (kernel-variant
# experiments in tools/); the default is the in-tree build
LIB_PATH = os.environ.get("BD_LIB_PATH") or os.path.join(_HERE, "_lib", "libbd_b200.so")
_lib = None


class NativeLibraryError(RuntimeError):
    """libbd_b200.so is missing, stale, or no CUDA device is available."""


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not built; run `python -m paper_1703_02484_b200.build` "
                "(there is no CPU fallback)")
        _lib = _abi.declare(ctypes.CDLL(LIB_PATH))
    return _lib


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the B200 engine has no CPU fallback")
    return torch


def check(rc: int, what: str):
    if rc != 0:
        raise NativeLibraryError(f"{what}: CUDA launch failed (cudaError {-rc})")


def stream_handle(torch_mod=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
