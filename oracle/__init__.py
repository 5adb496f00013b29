"""CPU oracle for base64 encode / validating decode -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1704_00605_b200``) never imports it, and the two share
no code.  The arithmetic lives in ``oracle/b64_oracle.c`` (plain scalar C,
a transcription of the paper's Algorithms 1 and 2, with the
readings of DESIGN.md §3); this module is ctypes marshalling only.

Pinned by tests/test_oracle.py (paper worked examples, Table II/III, App. C,
closed-form bijection over all 2^24 triples, brute-force error rule,
Python's stdlib base64).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "b64_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, INVALID_CHAR, LENGTH, NONCANONICAL = 0, 1, 2, 3
URL, NOPAD, STRICT = 1, 2, 4

_lib = None
_lock = threading.Lock()

CFLAGS = ["-O2", "-fno-tree-vectorize", "-fno-tree-slp-vectorize", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so with gcc (plain scalar flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            u8p = ctypes.c_void_p
            lib.oracle_B.argtypes = [ctypes.c_int]
            lib.oracle_B.restype = ctypes.c_int
            lib.oracle_A.argtypes = [ctypes.c_int]
            lib.oracle_A.restype = ctypes.c_int
            lib.oracle_encoded_len.argtypes = [ctypes.c_int64]
            lib.oracle_encoded_len.restype = ctypes.c_int64
            lib.oracle_encode.argtypes = [u8p, ctypes.c_int64, u8p]
            lib.oracle_encode.restype = ctypes.c_int64
            lib.oracle_decode.argtypes = [u8p, ctypes.c_int64, u8p,
                                          ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_int64)]
            lib.oracle_decode.restype = ctypes.c_int
            lib.oracle_B_ex.argtypes = [ctypes.c_int, ctypes.c_int]
            lib.oracle_B_ex.restype = ctypes.c_int
            lib.oracle_A_ex.argtypes = [ctypes.c_int, ctypes.c_int]
            lib.oracle_A_ex.restype = ctypes.c_int
            lib.oracle_encoded_len_ex.argtypes = [ctypes.c_int64, ctypes.c_int]
            lib.oracle_encoded_len_ex.restype = ctypes.c_int64
            lib.oracle_encode_ex.argtypes = [u8p, ctypes.c_int64, u8p, ctypes.c_int]
            lib.oracle_encode_ex.restype = ctypes.c_int64
            lib.oracle_decode_ex.argtypes = [u8p, ctypes.c_int64, u8p,
                                             ctypes.POINTER(ctypes.c_int64),
                                             ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
            lib.oracle_decode_ex.restype = ctypes.c_int
            lib.oracle_despace.argtypes = [u8p, ctypes.c_int64, u8p]
            lib.oracle_despace.restype = ctypes.c_int64
            lib.oracle_encoded_len_wrapped.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                       ctypes.c_int]
            lib.oracle_encoded_len_wrapped.restype = ctypes.c_int64
            lib.oracle_encode_wrapped.argtypes = [u8p, ctypes.c_int64, u8p, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_int]
            lib.oracle_encode_wrapped.restype = ctypes.c_int64
            lib.oracle_decode_ws.argtypes = [u8p, ctypes.c_int64, u8p,
                                             ctypes.POINTER(ctypes.c_int64),
                                             ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
            lib.oracle_decode_ws.restype = ctypes.c_int
            _lib = lib
    return _lib


def _as_u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    a = np.asarray(x)
    if a.dtype != np.uint8:
        a = a.astype(np.uint8)
    return np.ascontiguousarray(a)


def B(v: int) -> int:
    """Table I forward map (6-bit value -> ASCII code), -1 outside [0, 64)."""
    return _load().oracle_B(int(v))


def A(ch: int) -> int:
    """Table I inverse map (ASCII code -> 6-bit value), negative if invalid."""
    return _load().oracle_A(int(ch))


def encode(s) -> np.ndarray:
    """Algorithm 1: bytes -> ASCII (uint8 array of length 4*ceil(n/3))."""
    a = _as_u8(s)
    lib = _load()
    n = a.size
    out = np.empty(lib.oracle_encoded_len(n), dtype=np.uint8)
    w = lib.oracle_encode(a.ctypes.data if n else None, n, out.ctypes.data if out.size else None)
    assert w == out.size
    return out


def decode(c):
    """Algorithm 2 (readings R-pad, R2, R-length).

    Returns (status, err_pos, out) where ``out`` holds exactly the bytes the
    algorithm appended (on error: the complete quads before the failing one).
    """
    a = _as_u8(c)
    lib = _load()
    m = a.size
    cap = 3 * (m // 4)
    out = np.empty(max(cap, 1), dtype=np.uint8)
    ol = ctypes.c_int64(0)
    ep = ctypes.c_int64(0)
    st = lib.oracle_decode(a.ctypes.data if m else None, m, out.ctypes.data,
                           ctypes.byref(ol), ctypes.byref(ep))
    return int(st), int(ep.value), out[: ol.value].copy()


def encode_into(a: np.ndarray, out: np.ndarray) -> int:
    """Encode ``a`` into preallocated ``out`` (no copies; used for timing)."""
    return _load().oracle_encode(a.ctypes.data if a.size else None, a.size,
                                 out.ctypes.data if out.size else None)


def decode_into(c: np.ndarray, out: np.ndarray):
    ol = ctypes.c_int64(0)
    ep = ctypes.c_int64(0)
    st = _load().oracle_decode(c.ctypes.data if c.size else None, c.size,
                               out.ctypes.data if out.size else None,
                               ctypes.byref(ol), ctypes.byref(ep))
    return int(st), int(ep.value), int(ol.value)


def decode_batch(text: np.ndarray, off: np.ndarray):
    """Per-message decode of a batch: lists (status, err_pos, bytes)."""
    res = []
    for i in range(off.size - 1):
        res.append(decode(text[off[i]: off[i + 1]]))
    return res


def encode_batch(raw: np.ndarray, off: np.ndarray):
    return [encode(raw[off[i]: off[i + 1]]) for i in range(off.size - 1)]


def B_ex(v: int, flags: int) -> int:
    return _load().oracle_B_ex(int(v), int(flags))


def A_ex(ch: int, flags: int) -> int:
    return _load().oracle_A_ex(int(ch), int(flags))


def encode_ex(s, flags: int) -> np.ndarray:
    """Algorithm 1 variants (base64url / unpadded), SURVEY §8(f) f1."""
    a = _as_u8(s)
    lib = _load()
    out = np.empty(lib.oracle_encoded_len_ex(a.size, flags), dtype=np.uint8)
    w = lib.oracle_encode_ex(a.ctypes.data if a.size else None, a.size,
                             out.ctypes.data if out.size else None, flags)
    assert w == out.size
    return out


def decode_ex(c, flags: int):
    """Algorithm 2 variants (base64url, optional padding, App. A strict)."""
    a = _as_u8(c)
    lib = _load()
    out = np.empty(3 * (a.size // 4) + 3, dtype=np.uint8)
    ol = ctypes.c_int64(0)
    ep = ctypes.c_int64(0)
    st = lib.oracle_decode_ex(a.ctypes.data if a.size else None, a.size, out.ctypes.data,
                              ctypes.byref(ol), ctypes.byref(ep), flags)
    return int(st), int(ep.value), out[: ol.value].copy()


def despace(a) -> np.ndarray:
    """Appendix B scalar whitespace removal (Fig. spaceremove)."""
    x = _as_u8(a)
    out = np.empty(max(x.size, 1), dtype=np.uint8)
    n = _load().oracle_despace(x.ctypes.data if x.size else None, x.size, out.ctypes.data)
    return out[:n].copy()


def encode_wrapped(s, line_chars: int = 76, crlf: bool = False, flags: int = 0) -> np.ndarray:
    """f4: Algorithm 1, then an EOL after every ``line_chars`` characters and
    after the final line (MIME / PEM style)."""
    a = _as_u8(s)
    lib = _load()
    out = np.empty(max(lib.oracle_encoded_len_wrapped(a.size, line_chars, int(crlf), flags), 1),
                   dtype=np.uint8)
    w = lib.oracle_encode_wrapped(a.ctypes.data if a.size else None, a.size, out.ctypes.data,
                                  line_chars, int(crlf), flags)
    assert w >= 0
    return out[:w].copy()


def decode_ws(c, flags: int = 0):
    """f4: Appendix B whitespace filter, then Algorithm 2; err_pos in the
    coordinates of the original input.  Returns (status, err_pos, out)."""
    a = _as_u8(c)
    lib = _load()
    out = np.empty(3 * (a.size // 4) + 3, dtype=np.uint8)
    ol = ctypes.c_int64(0)
    ep = ctypes.c_int64(0)
    st = lib.oracle_decode_ws(a.ctypes.data if a.size else None, a.size, out.ctypes.data,
                              ctypes.byref(ol), ctypes.byref(ep), flags)
    assert st >= 0
    return int(st), int(ep.value), out[: ol.value].copy()
