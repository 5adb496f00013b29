"""GPU whitespace removal (Appendix B) vs the oracle's
scalar filter (Fig. spaceremove): sizes across tile seams, alignments,
all-whitespace / no-whitespace inputs, and despace -> decode of
line-wrapped text."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, empty_dev, host, to_dev

pytestmark = pytest.mark.gpu
TILE = 16384


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def with_spaces(n, seed, frac=0.03):
    rng = np.random.default_rng(seed)
    x = splitmix_bytes(seed, 0, n)
    sel = rng.random(n) < frac
    x[sel] = rng.choice(np.frombuffer(b" \n\r", dtype=np.uint8), size=int(sel.sum()))
    return x


def gpu_despace(x, im=0, om=0):
    base, out = empty_dev(max(x.size, 1), om)
    o, olen = b64.b64_despace(to_dev(x, im), out=out)
    n = int(olen.item())
    g = host(base)
    assert (g[:om] == 0xCC).all() and (g[om + max(x.size, 1):] == 0xCC).all()
    return host(o)[:n]


def test_despace_sizes_and_seams():
    for n in [0, 1, 2, 15, 16, 17, 1023, 1024, 1025, TILE - 1, TILE, TILE + 1, 3 * TILE + 7,
              148 * TILE + 5, 1_000_003]:
        x = with_spaces(n, 300 + n % 97)
        assert np.array_equal(gpu_despace(x), oracle.despace(x)), n


def test_despace_alignments():
    x = with_spaces(50_001, 301, 0.2)
    ref = oracle.despace(x)
    for im in range(0, 16, 3):
        for om in range(0, 16, 5):
            assert np.array_equal(gpu_despace(x, im, om), ref), (im, om)


def test_despace_extremes():
    allws = np.frombuffer((b" \r\n" * 20000)[:50000], dtype=np.uint8).copy()
    assert gpu_despace(allws).size == 0
    clean = splitmix_bytes(302, 0, 100_000)
    clean[np.isin(clean, np.frombuffer(b" \r\n", dtype=np.uint8))] = 0x41
    assert np.array_equal(gpu_despace(clean), clean)
    allb = np.tile(np.arange(256, dtype=np.uint8), 300)
    assert np.array_equal(gpu_despace(allb), oracle.despace(allb))


def test_despace_then_decode_wrapped_text():
    """MIME-style text (76-char lines, CRLF) decodes after GPU despacing."""
    x = splitmix_bytes(303, 0, 300_000)
    t = bytes(oracle.encode(x))
    wrapped = b"\r\n".join(t[i: i + 76] for i in range(0, len(t), 76)) + b"\r\n"
    w = np.frombuffer(wrapped, dtype=np.uint8).copy()
    d, olen = b64.b64_despace(to_dev(w))
    n = int(olen.item())
    y, st, ep = b64.b64_decode(d[:n])
    assert (st, ep) == (0, -1) and np.array_equal(host(y), x)
