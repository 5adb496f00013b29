"""Pins for the MIME-style line-handling oracle:
line-wrapped encode and whitespace-tolerant decode (Appendix B filter, then
Algorithm 2, error offsets in original coordinates; DESIGN.md §3 readings
R-wrap and R-ws-decode).

Independent references: Python's stdlib ``base64.encodebytes`` /
``decodebytes`` (RFC 2045, 76-column lines), ``ssl.DER_cert_to_PEM_cert``
(RFC 7468, 64-column lines), and insertion bookkeeping for error offsets
(where the rejected character lands after whitespace is inserted is known
to the test without decoding)."""
import base64
import ssl

import numpy as np
import pytest

import oracle

WS = np.frombuffer(b" \n\r", dtype=np.uint8)


def test_wrapped_encode_vs_encodebytes():
    rng = np.random.default_rng(41)
    for n in list(range(0, 130)) + [171, 172, 570, 4096, 100_001]:
        x = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        ref = base64.encodebytes(x)  # 76-char lines, "\n" after every line
        assert bytes(oracle.encode_wrapped(x, 76, crlf=False)) == ref, n
        assert bytes(oracle.encode_wrapped(x, 76, crlf=True)) == ref.replace(b"\n", b"\r\n"), n


def test_wrapped_encode_pem_64():
    rng = np.random.default_rng(42)
    for n in [1, 2, 3, 47, 48, 49, 95, 96, 97, 500, 1234]:
        der = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        pem = ssl.DER_cert_to_PEM_cert(der).encode()
        body = pem.split(b"-----BEGIN CERTIFICATE-----\n")[1].split(b"-----END CERTIFICATE-----")[0]
        assert bytes(oracle.encode_wrapped(der, 64, crlf=False)) == body, n


def test_encoded_len_wrapped_direct_pin():
    """oracle_encoded_len_wrapped (the capacity of a wrapped encode, R-wrap)
    pinned directly, not through the GPU's b64_encoded_len_wrapped: for
    76-char LF lines it is len(base64.encodebytes(x)) (RFC 2045), CR LF adds
    one byte per line; for any L and flags it is the length of the stdlib
    encoding (b64encode / urlsafe, '=' stripped for NOPAD) cut into L-char
    lines each followed by the EOL."""
    lib = oracle._load()
    rng = np.random.default_rng(44)
    ns = list(range(0, 200)) + [int(v) for v in rng.integers(200, 1 << 20, 60)]
    for n in ns:
        x = bytes(n)  # lengths do not depend on the bytes
        e = base64.encodebytes(x)
        assert lib.oracle_encoded_len_wrapped(n, 76, 0, 0) == len(e), n
        assert lib.oracle_encoded_len_wrapped(n, 76, 1, 0) == len(e) + e.count(b"\n"), n
    for L in (4, 8, 64, 76, 100, 1024, 16384):
        for flags in (0, oracle.URL, oracle.NOPAD, oracle.URL | oracle.NOPAD):
            for n in [0, 1, 2, 3, 4, 5, L // 4 * 3, L // 4 * 3 + 1, 3 * L + 2] + ns[-5:]:
                s = base64.b64encode(bytes(n))
                if flags & oracle.NOPAD:
                    s = s.rstrip(b"=")
                for crlf in (0, 1):
                    eol = b"\r\n" if crlf else b"\n"
                    ref = len(b"".join(s[i: i + L] + eol for i in range(0, len(s), L)))
                    assert lib.oracle_encoded_len_wrapped(n, L, crlf, flags) == ref, (n, L, crlf, flags)


@pytest.mark.parametrize("L", [4, 8, 60, 64, 76, 100, 1024])
@pytest.mark.parametrize("flags", [0, oracle.URL, oracle.NOPAD, oracle.URL | oracle.NOPAD])
def test_wrapped_encode_structure(L, flags):
    # invariants: removing the EOLs gives Algorithm 1's output; every line but
    # the last has exactly L characters; the output ends with an EOL
    rng = np.random.default_rng(43 + L)
    for n in [0, 1, 2, 3, L // 4 * 3, L // 4 * 3 + 1, 3 * L + 2, 1000]:
        x = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        for crlf in (False, True):
            w = bytes(oracle.encode_wrapped(x, L, crlf=crlf, flags=flags))
            eol = b"\r\n" if crlf else b"\n"
            plain = bytes(oracle.encode_ex(x, flags))
            if not plain:
                assert w == b""
                continue
            assert w.endswith(eol)
            lines = w[: -len(eol)].split(eol)
            assert b"".join(lines) == plain
            assert all(len(s) == L for s in lines[:-1]) and 0 < len(lines[-1]) <= L


def test_decode_ws_vs_decodebytes():
    rng = np.random.default_rng(44)
    for n in list(range(0, 100)) + [1000, 65_537]:
        x = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        for text in (base64.encodebytes(x), base64.encodebytes(x).replace(b"\n", b"\r\n")):
            st, ep, out = oracle.decode_ws(text)
            assert (st, ep) == (0, -1) and bytes(out) == base64.decodebytes(text) == x, n


def _insert_ws(t: np.ndarray, rng, density: float):
    """Insert runs of whitespace before random positions of t; returns the new
    text and new_index[i] = where t[i] landed."""
    k = t.size
    runs = (rng.random(k + 1) < density) * rng.integers(1, 4, k + 1)
    parts, new_index, pos = [], np.empty(k, dtype=np.int64), 0
    for i in range(k + 1):
        if runs[i]:
            parts.append(rng.choice(WS, size=int(runs[i])))
            pos += int(runs[i])
        if i < k:
            parts.append(t[i:i + 1])
            new_index[i] = pos
            pos += 1
    w = np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8)
    return w, new_index


def test_decode_ws_error_offsets_follow_insertion():
    rng = np.random.default_rng(45)
    na = np.array([b for b in range(256) if b not in b" \n\r" and oracle.A(b) < 0 and b != ord("=")],
                  dtype=np.uint8)
    for trial in range(1500):
        n = int(rng.integers(0, 60))
        fl = [0, oracle.URL, oracle.NOPAD, oracle.STRICT][trial % 4]
        t = oracle.encode_ex(rng.integers(0, 256, n, dtype=np.uint8), fl & ~oracle.STRICT)
        kind = trial % 5
        if kind == 1 and t.size:  # one invalid byte
            t = t.copy()
            t[int(rng.integers(0, t.size))] = na[int(rng.integers(0, na.size))]
        elif kind == 2 and t.size:  # truncation (LENGTH unless NOPAD accepts it)
            t = t[: int(rng.integers(0, t.size))]
        elif kind == 3 and t.size:  # a misplaced '='
            t = t.copy()
            t[int(rng.integers(0, t.size))] = ord("=")
        elif kind == 4 and t.size >= 2:  # non-canonical trailing bits
            t = t.copy()
            t[-1 if t[-1] != ord("=") else -3 if t[-2] == ord("=") else -2] ^= 1
        w, idx = _insert_ws(t, rng, density=float(rng.choice([0.05, 0.3, 1.0])))
        st0, ep0, out0 = oracle.decode_ex(t, fl)
        st, ep, out = oracle.decode_ws(w, fl)
        assert st == st0 and np.array_equal(out, out0), (trial, bytes(t), bytes(w))
        assert ep == (-1 if ep0 < 0 else int(idx[ep0])), (trial, bytes(t), bytes(w))


def test_decode_ws_special_cases():
    # the Linux codec's tolerance: line feeds between blocks of four
    st, ep, out = oracle.decode_ws(b"QUJD\nREVG\n")
    assert (st, ep, bytes(out)) == (0, -1, b"ABCDEF")
    # whitespace anywhere, including inside a quad and around the padding
    st, ep, out = oracle.decode_ws(b" Q U\r\nJ D Q Q = = \r\n")
    assert (st, ep, bytes(out)) == (0, -1, b"ABCA")
    # whitespace only / empty
    assert oracle.decode_ws(b"")[:2] == (0, -1)
    assert oracle.decode_ws(b" \r\n\n  ")[:2] == (0, -1)
    # only the three Appendix B bytes are whitespace: TAB and FF are invalid
    assert oracle.decode_ws(b"QU\tJD")[:2] == (oracle.INVALID_CHAR, 2)
    assert oracle.decode_ws(b"QUJD\x0cAAA")[:2] == (oracle.INVALID_CHAR, 4)
    # ... and a partial final quad is not examined (R-length): LENGTH at 4
    assert oracle.decode_ws(b"QUJD\x0c")[:2] == (oracle.LENGTH, 4)
    # LENGTH is reported at the first kept byte of the partial quad
    assert oracle.decode_ws(b"QUJD\nRA")[:2] == (oracle.LENGTH, 5)
    # data after padding: the rejected byte is the one after the '='
    assert oracle.decode_ws(b"QQ=\n\nA")[:2] == (oracle.INVALID_CHAR, 5)
