"""Pins for the Appendix B whitespace-removal oracle:
Python's bytes.translate as the independent filter, the paper's three
removed bytes (reading G8), and invariants."""
import numpy as np

import oracle


def test_despace_vs_translate():
    rng = np.random.default_rng(31)
    for n in list(range(0, 50)) + [1024, 4096, 100_003]:
        x = rng.integers(0, 256, n, dtype=np.uint8)
        # ~3 % whitespace as in the paper's test
        sel = rng.random(n) < 0.03
        x[sel] = rng.choice(np.frombuffer(b" \n\r", dtype=np.uint8), size=int(sel.sum()))
        ref = x.tobytes().translate(None, b" \n\r")
        assert oracle.despace(x).tobytes() == ref


def test_despace_removes_exactly_three_bytes():
    allb = np.arange(256, dtype=np.uint8)
    kept = oracle.despace(allb)
    assert kept.size == 253
    assert set(range(256)) - set(kept.tolist()) == {0x20, 0x0A, 0x0D}
    assert oracle.despace(np.frombuffer(b"  \r\n\n", dtype=np.uint8)).size == 0
