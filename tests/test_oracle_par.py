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
