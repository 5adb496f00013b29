"""Pins for the CPU oracle (oracle/b64_oracle.c) against things other than
itself: the paper's worked examples and tables, closed forms, brute force on
tiny inputs, and Python's stdlib base64 as an independent library routine.

Each test names the plausible oracle mistake it would catch.
"""
import base64
import binascii
import itertools
import json
import os
import string

import numpy as np
import pytest

import oracle



ALPHABET = (string.ascii_uppercase + string.ascii_lowercase + string.digits + "+/").encode()


def _golden(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- paper pins

def test_paper_encode_example(golden_dir):
    """71,73,70 -> 17,52,37,6 -> R0lG (catches wrong shift/mask in Alg 1)."""
    ex = _golden(golden_dir, "paper_examples.json")["encode_example"]
    assert bytes(oracle.encode(ex["bytes"])) == ex["text"].encode()
    assert [oracle.A(ch) for ch in ex["text"].encode()] == ex["values"]
    assert bytes(oracle.B(v) for v in ex["values"]) == ex["text"].encode()


def test_paper_gif_example(golden_dir):
    """the GIF string decodes to the 35 listed bytes and its 47
    characters before '=' map to the listed 6-bit values; re-encoding gives
    back the string (n mod 3 = 2 tail, one '=')."""
    ex = _golden(golden_dir, "paper_examples.json")["gif_example"]
    text = ex["text"].encode()
    assert [oracle.A(ch) for ch in text[:-1]] == ex["values"]
    st, ep, out = oracle.decode(text)
    assert (st, ep) == (oracle.OK, -1)
    assert out.tolist() == ex["bytes"]
    assert bytes(oracle.encode(ex["bytes"])) == text


def test_appendix_c_walkthrough(golden_dir):
    """byte values, hi nibbles, roll offsets and 6-bit values of
    the 32-char block; oracle.A must agree with value = byte + offset."""
    ex = _golden(golden_dir, "paper_examples.json")["appendix_c_example"]
    text = ex["text"].encode()
    assert list(text) == ex["byte_values"]
    assert [b >> 4 for b in text] == ex["hi_nibbles"]
    assert [b + o for b, o in zip(text, ex["offsets"])] == ex["values"]
    assert [oracle.A(b) for b in text] == ex["values"]


def test_table_ii_offsets(golden_dir):
    """P:422-435 Table II: B(v) = v + offset(range of v) for all 64 values
    (catches a swapped range or an off-by-one at 25/51/61)."""
    ranges = _golden(golden_dir, "paper_examples.json")["table_ii_offsets"]["ranges"]
    seen = 0
    for lo, hi, off in ranges:
        for v in range(lo, hi + 1):
            assert oracle.B(v) == v + off, v
            seen += 1
    assert seen == 64
    assert oracle.B(64) < 0 and oracle.B(-1) < 0


def test_algorithm_4_bitsets_over_all_bytes(golden_dir):
    """P:934-958 + P:1288-1330: the nibble-bitset validity rule and the roll
    offsets define A over all 256 bytes independently of the range form
    ('=' and every non-ASCII byte invalid; reading G5 = floor)."""
    lut = _golden(golden_dir, "paper_examples.json")["algorithm_4_luts"]
    lo_t, hi_t, roll = lut["lut_lo"], lut["lut_hi"], lut["roll"]
    nvalid = 0
    for x in range(256):
        h = x >> 4
        invalid = (lo_t[x & 15] & hi_t[h]) != 0
        a = oracle.A(x)
        assert (a < 0) == invalid, x
        if not invalid:
            nvalid += 1
            c = -1 if x == 0x2F else 0
            assert a == x + roll[h + c], x
    assert nvalid == 64
    assert oracle.A(ord("=")) < 0


def test_alphabet_is_a_bijection():
    """Table I: B is injective onto the 64 RFC 4648 characters and A inverts it."""
    fwd = bytes(oracle.B(v) for v in range(64))
    assert fwd == ALPHABET
    for v in range(64):
        assert oracle.A(oracle.B(v)) == v
    for x in range(256):
        assert (oracle.A(x) >= 0) == (x in ALPHABET)


def test_rfc4648_vectors(golden_dir):
    vec = _golden(golden_dir, "rfc4648_vectors.json")["vectors"]
    for raw, enc in vec:
        assert bytes(oracle.encode(raw.encode())) == enc.encode()
        assert base64.b64encode(raw.encode()) == enc.encode()  # the vectors themselves
        st, ep, out = oracle.decode(enc.encode())
        assert (st, ep, bytes(out)) == (oracle.OK, -1, raw.encode())


def test_noncanonical_trailing_bits_accepted(golden_dir):
    """default decoding accepts non-canonical trailing bits."""
    ex = _golden(golden_dir, "paper_examples.json")["appendix_a_strict"]
    for key in ("noncanonical", "canonical"):
        st, ep, out = oracle.decode(ex[key + "_text"].encode())
        assert (st, ep) == (oracle.OK, -1)
        assert out.tolist() == ex[key + "_bytes"]


# ------------------------------------------------------------ closed forms

def test_bijection_all_2_24_triples():
    """Closed form: encoding the 2^24 triples in increasing (big-endian)
    order yields the 64^4 quartets in increasing 6-bit-value order, and
    decoding gives the triples back (catches any transposed field)."""
    t = np.arange(1 << 24, dtype=np.uint32)
    triples = np.stack([(t >> 16) & 255, (t >> 8) & 255, t & 255], axis=1).astype(np.uint8).ravel()
    enc = oracle.encode(triples)
    assert enc.size == 4 * (1 << 24)
    alpha = np.frombuffer(ALPHABET, dtype=np.uint8)
    # enumeration of quartets (a,b,c,d) in lexicographic order, independent of Alg 1's shifts
    idx = np.indices((64, 64, 64, 64), dtype=np.uint8).reshape(4, -1).T
    expect = alpha[idx].ravel()
    assert np.array_equal(enc, expect)
    st, ep, dec = oracle.decode(enc)
    assert (st, ep) == (oracle.OK, -1)
    assert np.array_equal(dec, triples)


def test_length_law_and_padding_counts():
    """|encode(x)| = 4*ceil(n/3); one '=' per missing byte."""
    rng = np.random.default_rng(11)
    for n in range(0, 64):
        x = rng.integers(0, 256, n, dtype=np.uint8)
        e = bytes(oracle.encode(x))
        assert len(e) == 4 * ((n + 2) // 3)
        pads = len(e) - len(e.rstrip(b"="))
        assert pads == (3 - n % 3) % 3


def test_roundtrip_and_stdlib_random():
    """Python's stdlib base64 as an independent implementation."""
    rng = np.random.default_rng(12)
    lens = list(range(0, 260)) + [4095, 4096, 4097, 65535, 65536, 65537]
    for n in lens:
        x = rng.integers(0, 256, n, dtype=np.uint8)
        e = bytes(oracle.encode(x))
        assert e == base64.b64encode(x.tobytes())
        st, ep, out = oracle.decode(e)
        assert (st, ep) == (oracle.OK, -1)
        assert out.tobytes() == x.tobytes()


def test_stdlib_accept_reject_on_mutations():
    """Accept/reject agreement with binascii strict mode on single-byte
    mutations of valid text (the stdlib reports no offset)."""
    rng = np.random.default_rng(13)
    for trial in range(3000):
        n = int(rng.integers(1, 40))
        x = rng.integers(0, 256, n, dtype=np.uint8)
        e = bytearray(oracle.encode(x))
        pos = int(rng.integers(0, len(e)))
        e[pos] = int(rng.integers(0, 256))
        st, ep, out = oracle.decode(bytes(e))
        try:
            ref = binascii.a2b_base64(bytes(e), strict_mode=True)
            ok = True
        except binascii.Error:
            ok = False
        assert (st == oracle.OK) == ok, (bytes(e), st, ep)
        if ok:
            assert out.tobytes() == ref


# ------------------------------------------------------- error rule (R2)

def _valid_class_strings(L):
    """All valid class strings of length L (L % 4 == 0): data 'D' everywhere
    except that the final quad may end in 'D=' or '=='."""
    if L == 0:
        return [""]
    return ["D" * L, "D" * (L - 1) + "=", "D" * (L - 2) + "=="]


def _brute_force(cls):
    """Error offset by the prefix definition: the first i such that cls[:i+1]
    is not a prefix of any valid string of length L = 4*ceil(m/4); positions
    past the last full quad are never examined (LENGTH wins at 4q)."""
    m = len(cls)
    L = 4 * ((m + 3) // 4)
    valid = _valid_class_strings(L)
    for i in range(4 * (m // 4)):
        p = cls[: i + 1]
        if not any(v.startswith(p) for v in valid):
            return oracle.INVALID_CHAR, i
    if m % 4:
        return oracle.LENGTH, 4 * (m // 4)
    return oracle.OK, -1


def test_error_rule_brute_force_class_strings():
    """Every string over {data, '=', invalid} of length <= 9 (29,524 strings):
    the oracle's status and err_pos equal the brute-force prefix definition,
    and on error the output is exactly the complete quads before it."""
    char = {"D": ord("Q"), "=": ord("="), "X": ord("!")}
    count = 0
    for m in range(0, 10):
        for cls in itertools.product("D=X", repeat=m):
            cls = "".join(cls)
            st, ep, out = oracle.decode(bytes(char[c] for c in cls))
            assert (st, ep) == _brute_force(cls), cls
            if st != oracle.OK:
                assert out.size == 3 * (ep // 4), cls
            else:
                q = m // 4
                p = len(cls) - len(cls.rstrip("="))
                assert out.size == 3 * q - p, cls
            count += 1
    assert count == (3 ** 10 - 1) // 2


def test_exhaustive_single_byte_rejection():
    """S:135 analogue: 'AA'+b+'A' fails iff b is not an alphabet character;
    a '=' at m-2 is legal by itself, so the error is then reported at m-1."""
    for b in range(256):
        st, ep, out = oracle.decode(bytes([65, 65, b, 65]))
        if b in ALPHABET:
            assert (st, ep) == (oracle.OK, -1)
        elif b == ord("="):
            assert (st, ep) == (oracle.INVALID_CHAR, 3)
        else:
            assert (st, ep) == (oracle.INVALID_CHAR, 2)


def test_every_byte_every_position():
    """All 256 bytes at each of 32 positions of a valid 32-char block
    (8,192 cases, S:346 analogue): error exactly at the position iff invalid."""
    rng = np.random.default_rng(14)
    base = bytearray(oracle.encode(rng.integers(0, 256, 24, dtype=np.uint8)))
    for pos in range(32):
        for b in range(256):
            t = bytearray(base)
            t[pos] = b
            st, ep, _ = oracle.decode(bytes(t))
            if b in ALPHABET:
                assert (st, ep) == (oracle.OK, -1)
            elif b == ord("=") and pos == 31:
                assert (st, ep) == (oracle.OK, -1)
            elif b == ord("=") and pos == 30:
                assert (st, ep) == (oracle.INVALID_CHAR, 31)
            else:
                assert (st, ep) == (oracle.INVALID_CHAR, pos), (pos, b)


def test_spec_small_cases():
    assert oracle.decode(b"R0l\x07")[:2] == (oracle.INVALID_CHAR, 3)
    assert oracle.decode(b"AAAA")[2].tolist() == [0, 0, 0]
    assert bytes(oracle.encode([0])) == b"AA=="
    assert oracle.decode(b"")[:2] == (oracle.OK, -1)
    assert oracle.decode(b"AAA")[:2] == (oracle.LENGTH, 0)
    st, ep, out = oracle.decode(b"AAAAA")
    assert (st, ep, out.tolist()) == (oracle.LENGTH, 4, [0, 0, 0])
    assert oracle.decode(b"A!AAA")[:2] == (oracle.INVALID_CHAR, 1)
    assert oracle.decode(b"AAAA!AAAA")[:2] == (oracle.INVALID_CHAR, 4)
    # '=' inside the stream is invalid even in a length-valid string
    assert oracle.decode(b"AA==AAAA")[:2] == (oracle.INVALID_CHAR, 2)
    assert oracle.decode(b"=AAA")[:2] == (oracle.INVALID_CHAR, 0)
    # multiple errors: minimum offset
    assert oracle.decode(b"AAAAAA!AAA!A")[:2] == (oracle.INVALID_CHAR, 6)
