"""The chunked/threaded oracle driver used for config-size parity equals the
plain oracle (so config parity rests on the pinned oracle)."""
import numpy as np

import oracle
from inputs.gen import splitmix_bytes
from tests import oracle_par


def test_parallel_encode_equals_oracle():
    for n in (0, 1, 2, 3, 100, 3001, 100003):
        x = splitmix_bytes(31, 0, n)
        for th in (1, 3, 8):
            assert np.array_equal(oracle_par.encode(x, th), oracle.encode(x))


def test_parallel_decode_equals_oracle():
    rng = np.random.default_rng(32)
    x = splitmix_bytes(32, 0, 30001)
    t = oracle.encode(x)
    cases = [t, t[:-1], t[:-2], t[:5], t[:0], t[:4]]
    for k in range(40):
        u = t.copy()
        for p in rng.choice(u.size, size=int(rng.integers(1, 4)), replace=False):
            u[p] = int(rng.choice([0, 61, 33, 200]))
        cases.append(u)
    for c in cases:
        ref = oracle.decode(c)
        for th in (1, 2, 7):
            got = oracle_par.decode(c, th)
            assert got[:2] == ref[:2] and np.array_equal(got[2], ref[2]), (th, ref[:2], got[:2])


def test_parallel_gen_equals_generator():
    for b, e in [(0, 0), (5, 6), (3, 1000), ((1 << 32) - 7, (1 << 32) + 100)]:
        for th in (1, 3, 8):
            assert np.array_equal(oracle_par.gen(5, b, e, th), splitmix_bytes(5, b, e))


def test_parallel_mime_helpers_equal_oracle():
    """encode_wrapped / despace / decode_ws_lines split on whole lines equal
    the plain oracle, incl. a short last line, errors in any part (offsets
    in whole-text coordinates) and the variant flags."""
    rng = np.random.default_rng(33)
    for n in (0, 1, 56, 57, 58, 5700, 57 * 40 - 2, 57 * 40 + 1):
        x = splitmix_bytes(33, 0, n)
        for L, crlf in ((76, True), (64, False), (4, True)):
            ref = oracle.encode_wrapped(x, L, crlf=crlf)
            for th in (1, 3, 8):
                w = oracle_par.encode_wrapped(x, L, crlf, th)
                assert np.array_equal(w, ref), (n, L, crlf, th)
                assert np.array_equal(oracle_par.despace(w, th), oracle.despace(w))
            lt = L + (2 if crlf else 1)
            cases = [ref]
            for k in range(6):
                if ref.size:
                    u = ref.copy()
                    u[int(rng.integers(0, u.size))] = int(rng.choice([ord("!"), ord("="), 0x80]))
                    cases.append(u)
            if ref.size > 3:
                cases.append(ref[:-3])
            for c in cases:
                for fl in (0, 2, 4):
                    exp = oracle.decode_ws(c, fl)
                    for th in (1, 2, 5):
                        got = oracle_par.decode_ws_lines(c, lt, fl, th)
                        assert got[:2] == exp[:2] and np.array_equal(got[2], exp[2]), (n, L, fl, th)
