"""Multi-threaded use of the scalar CPU oracle for config-size parity tests.

The oracle itself is unchanged (oracle/b64_oracle.c); this only splits a
buffer on 3-byte (encode) / 4-char (decode) boundaries and runs the oracle on
the chunks in threads (ctypes releases the GIL).  Chunked decode is exact:
a non-final chunk is decoded with a valid quad "AAAA" appended, so its last
two positions are not final-quad positions (a '=' there is an error, as in
the whole-buffer decode), and the chunk results are combined by taking the
first chunk with an error.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import oracle

THREADS = max(1, min(32, len(os.sched_getaffinity(0))))


def _bounds(total: int, unit: int, parts: int):
    q = (total + unit - 1) // unit
    return [(min(q * r // parts * unit, total), min(q * (r + 1) // parts * unit, total)) for r in range(parts)]


def encode(x: np.ndarray, threads: int = THREADS) -> np.ndarray:
    n = x.size
    out = np.empty(4 * ((n + 2) // 3), dtype=np.uint8)
    parts = _bounds(n, 3, threads)

    def job(be):
        b, e = be
        if e > b:
            out[4 * (b // 3): 4 * (b // 3) + 4 * ((e - b + 2) // 3)] = oracle.encode(x[b:e])

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, parts))
    return out


_AAAA = np.frombuffer(b"AAAA", dtype=np.uint8)


def decode(t: np.ndarray, threads: int = THREADS):
    """(status, err_pos, out) identical to oracle.decode(t)."""
    m = t.size
    q4 = 4 * (m // 4)
    parts = [(b, e) for (b, e) in _bounds(q4, 4, threads) if e > b]
    if not parts:
        return oracle.decode(t)
    # the last chunk runs to the true end of the buffer (pads, partial quad)
    parts[-1] = (parts[-1][0], m)
    out = np.empty(max(3 * (m // 4), 1), dtype=np.uint8)
    res = [None] * len(parts)

    def job(i):
        b, e = parts[i]
        last = i == len(parts) - 1
        c = t[b:e] if last else np.concatenate([t[b:e], _AAAA])
        st, ep, o = oracle.decode(c)
        if not last:
            if st != oracle.OK and ep < e - b:
                o = o[: 3 * (ep // 4)]
            else:
                st, ep, o = oracle.OK, -1, o[: 3 * ((e - b) // 4)]
        out[3 * (b // 4): 3 * (b // 4) + o.size] = o
        res[i] = (st, ep, o.size)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(len(parts))))
    olen = 0
    for i, (st, ep, osz) in enumerate(res):
        b = parts[i][0]
        if st != oracle.OK:
            return st, b + ep, out[: 3 * (b // 4) + osz].copy()
        olen = 3 * (b // 4) + osz
    return oracle.OK, -1, out[:olen].copy()
