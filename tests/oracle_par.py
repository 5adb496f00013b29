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


# ------------------------------------------------ streaming helpers (C5, f3/f4)

def gen(seed: int, begin: int, end: int, threads: int = THREADS) -> np.ndarray:
    """inputs.gen.splitmix_bytes(seed, begin, end), generated in threads
    (counter-based: each thread fills its own byte range)."""
    from inputs.gen import splitmix_bytes

    out = np.empty(max(end - begin, 0), dtype=np.uint8)
    cuts = [begin + (end - begin) * r // threads for r in range(threads + 1)]

    def job(r):
        a, b = cuts[r], cuts[r + 1]
        if b > a:
            out[a - begin: b - begin] = splitmix_bytes(seed, a, b)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(threads)))
    return out


def _line_parts(nlines: int, threads: int):
    return [(nlines * r // threads, nlines * (r + 1) // threads) for r in range(threads)]


def encode_wrapped(x: np.ndarray, line_chars: int, crlf: bool, threads: int = THREADS) -> np.ndarray:
    """oracle.encode_wrapped(x, line_chars, crlf), split on whole lines
    (3*line_chars/4 input bytes per line): every part but the last is whole
    lines, whose wrapped encodings concatenate to the whole's."""
    lb = 3 * line_chars // 4
    lt = line_chars + (2 if crlf else 1)
    nlines = (x.size + lb - 1) // lb
    parts = [(a, b) for a, b in _line_parts(nlines, threads) if b > a]
    outs = [None] * len(parts)

    def job(i):
        a, b = parts[i]
        outs[i] = oracle.encode_wrapped(x[a * lb: min(b * lb, x.size)], line_chars, crlf=crlf)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(len(parts))))
    out = np.concatenate(outs) if outs else np.zeros(0, dtype=np.uint8)
    assert all(o.size == (b - a) * lt for o, (a, b) in zip(outs[:-1], parts[:-1]))
    return out


def despace(t: np.ndarray, threads: int = THREADS) -> np.ndarray:
    """oracle.despace(t): App. B removal is byte-local, so any split works."""
    cuts = [t.size * r // threads for r in range(threads + 1)]
    outs = [None] * threads

    def job(r):
        outs[r] = oracle.despace(t[cuts[r]: cuts[r + 1]])

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(threads)))
    return np.concatenate(outs)


def decode_ws_lines(t: np.ndarray, line_total: int, flags: int = 0, threads: int = THREADS):
    """oracle.decode_ws(t, flags) for text whose every line but the last is
    ``line_total`` bytes of which a multiple of 4 are kept characters (MIME
    lines): a non-final part of whole lines is decoded with a valid quad
    appended (its last quad is then not the final one, as in the whole
    decode), error offsets are shifted back to whole-text coordinates, and
    the first part with an error decides.  Returns (status, err_pos, out)."""
    nlines = (t.size + line_total - 1) // line_total
    parts = [(a * line_total, min(b * line_total, t.size)) for a, b in _line_parts(nlines, threads) if b > a]
    if len(parts) <= 1:
        return oracle.decode_ws(t, flags)
    res = [None] * len(parts)

    def job(i):
        a, b = parts[i]
        last = i == len(parts) - 1
        c = t[a:b] if last else np.concatenate([t[a:b], _AAAA])
        st, ep, o = oracle.decode_ws(c, flags)
        if not last:
            if st != oracle.OK and ep < b - a:
                pass
            else:
                st, ep, o = oracle.OK, -1, o[: o.size - 3]
        res[i] = (st, ep, o)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(len(parts))))
    outs = []
    for (a, b), (st, ep, o) in zip(parts, res):
        outs.append(o)
        if st != oracle.OK:
            return st, a + ep, np.concatenate(outs)
    return oracle.OK, -1, np.concatenate(outs)
