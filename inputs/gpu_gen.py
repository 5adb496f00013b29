"""CUDA twin of ``inputs.gen`` (ctypes binding of inputs/libb64gen.so)."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libb64gen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(_LIB_PATH)
        lib.b64gen_fill.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64,
                                    ctypes.c_int64, ctypes.c_void_p]
        lib.b64gen_fill.restype = ctypes.c_int
        _lib = lib
    return _lib


def fill(t, seed: int, begin: int = 0, stream=None) -> None:
    """Fill uint8 CUDA tensor ``t`` with G(seed, begin .. begin+numel)."""
    import torch

    assert t.dtype == torch.uint8 and t.is_cuda and t.is_contiguous()
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    rc = _load().b64gen_fill(ctypes.c_void_p(t.data_ptr()), t.numel(), seed & (2**64 - 1),
                             begin, ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"b64gen_fill failed rc={rc}")
