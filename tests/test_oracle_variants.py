"""Pins for the oracle's variant modes:
base64url, unpadded encoding / optional padding and the
Appendix A strict canonical check.  Independent references:
Python's stdlib base64 (urlsafe), the round-trip characterisation of
canonical strings, and a brute-force prefix definition of the error rule."""
import base64
import itertools
import string

import numpy as np

import oracle

STD = (string.ascii_uppercase + string.ascii_lowercase + string.digits + "+/").encode()
URLA = (string.ascii_uppercase + string.ascii_lowercase + string.digits + "-_").encode()


def test_url_alphabet():
    assert bytes(oracle.B_ex(v, oracle.URL) for v in range(64)) == URLA
    for x in range(256):
        a = oracle.A_ex(x, oracle.URL)
        assert (a >= 0) == (x in URLA)
        if a >= 0:
            assert URLA[a] == x
    assert oracle.A_ex(ord("+"), oracle.URL) < 0 and oracle.A_ex(ord("/"), oracle.URL) < 0


def test_url_and_nopad_encode_vs_stdlib():
    rng = np.random.default_rng(21)
    for n in list(range(0, 70)) + [1000, 4097]:
        x = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        ref = base64.urlsafe_b64encode(x)
        assert bytes(oracle.encode_ex(x, oracle.URL)) == ref
        assert bytes(oracle.encode_ex(x, oracle.URL | oracle.NOPAD)) == ref.rstrip(b"=")
        assert bytes(oracle.encode_ex(x, oracle.NOPAD)) == base64.b64encode(x).rstrip(b"=")
        assert bytes(oracle.encode_ex(x, 0)) == base64.b64encode(x)


def test_variant_decode_roundtrips():
    rng = np.random.default_rng(22)
    for n in range(0, 80):
        x = rng.integers(0, 256, n, dtype=np.uint8)
        for fl in (0, oracle.URL, oracle.NOPAD, oracle.URL | oracle.NOPAD, oracle.STRICT,
                   oracle.STRICT | oracle.NOPAD | oracle.URL):
            t = oracle.encode_ex(x, fl)
            st, ep, out = oracle.decode_ex(t, fl)
            assert (st, ep) == (0, -1) and np.array_equal(out, x), (n, fl)
        # optional padding: padded text is also accepted in NOPAD mode
        st, ep, out = oracle.decode_ex(oracle.encode(x), oracle.NOPAD)
        assert (st, ep) == (0, -1) and np.array_equal(out, x)
        # url text is rejected by the standard alphabet iff it uses '-' or '_'
        tu = bytes(oracle.encode_ex(x, oracle.URL))
        st, _, _ = oracle.decode_ex(tu, 0)
        assert (st == 0) == (b"-" not in tu and b"_" not in tu)


def test_default_flags_equal_plain_oracle():
    rng = np.random.default_rng(23)
    for trial in range(2000):
        n = int(rng.integers(0, 40))
        t = bytearray(oracle.encode(rng.integers(0, 256, n, dtype=np.uint8)))
        if t:
            t[int(rng.integers(0, len(t)))] = int(rng.integers(0, 256))
        a = oracle.decode(bytes(t))
        b = oracle.decode_ex(bytes(t), 0)
        assert a[:2] == b[:2] and np.array_equal(a[2], b[2])


def test_strict_equals_canonical_roundtrip_all_final_quads():
    """App. A: a padded final quad is accepted in strict mode iff it is the
    encoding of its own decoding (characterisation of canonical strings),
    over every 'xx==' (64^2) and 'xxx=' (64^3) and every unpadded 2/3-char
    tail."""
    count = 0
    for a, b in itertools.product(STD, repeat=2):
        s = bytes([a, b]) + b"=="
        st, ep, out = oracle.decode_ex(s, oracle.STRICT)
        canon = bytes(oracle.encode(out if st == 0 else oracle.decode(s)[2])) == s
        assert (st == 0) == canon
        if st:
            assert (st, ep) == (oracle.NONCANONICAL, 1)
        st2, ep2, _ = oracle.decode_ex(bytes([a, b]), oracle.STRICT | oracle.NOPAD)
        assert (st2 == 0) == canon
        count += 1
    for a, b, c in itertools.product(STD, repeat=3):
        s = bytes([a, b, c]) + b"="
        st, ep, out = oracle.decode_ex(s, oracle.STRICT)
        canon = bytes(oracle.encode(oracle.decode(s)[2])) == s
        assert (st == 0) == canon
        if st:
            assert (st, ep) == (oracle.NONCANONICAL, 2)
        count += 1
    assert count == 64 ** 2 + 64 ** 3
    assert oracle.decode_ex(b"Zg==", oracle.STRICT)[:2] == (0, -1)
    assert oracle.decode_ex(b"Zh==", oracle.STRICT)[:2] == (oracle.NONCANONICAL, 1)


def _valid_nopad(cls):
    L = len(cls)
    if L % 4 == 0:
        return (set(cls[:-2]) <= {"D"} and cls[-2:] in ("DD", "D=", "==")) if L else True
    if L % 4 in (2, 3):
        return set(cls) <= {"D"}
    return False


def _brute_force_nopad(cls):
    """First position whose prefix extends to no valid (optionally padded)
    string of length L >= m; then LENGTH for m % 4 == 1."""
    m = len(cls)
    # with m % 4 == 1 the single trailing character is never examined (R-length)
    for i in range(4 * (m // 4) if m % 4 == 1 else m):
        p = cls[: i + 1]
        ok = False
        for L in range(m, m + 4):
            for tail in itertools.product("D=", repeat=L - len(p)):
                if _valid_nopad(p + "".join(tail)):
                    ok = True
                    break
            if ok:
                break
        if not ok:
            return oracle.INVALID_CHAR, i
    if not _valid_nopad(cls):  # every prefix extends, but the input is incomplete
        return oracle.LENGTH, 4 * (m // 4)
    return oracle.OK, -1


def test_nopad_error_rule_brute_force():
    char = {"D": ord("Q"), "=": ord("="), "X": ord("!")}
    for m in range(0, 8):
        for cls in itertools.product("D=X", repeat=m):
            cls = "".join(cls)
            st, ep, _ = oracle.decode_ex(bytes(char[c] for c in cls), oracle.NOPAD)
            assert (st, ep) == _brute_force_nopad(cls), cls
