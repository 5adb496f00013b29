"""f3 / f4 at sizes past 2^32 (64-bit offsets in every index path): 3.8 GB of
seeded bytes -> line-wrapped encode (76 + CRLF, 5.2 GB of text) ->
whitespace-tolerant decode back, and despace of the same text vs the plain
encoding -- compared on the device in full, and on sampled windows against
the CPU oracle; error offsets beyond 2^32 are exact."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from inputs.gpu_gen import fill
from tests.gpu_util import DEV, host

pytestmark = pytest.mark.gpu
SEED = 96
LINES = 1 << 26          # 67,108,864 lines of 76 chars
N = 57 * LINES - 2        # raw bytes (n mod 3 = 1: the last line ends "==")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    free, _ = torch.cuda.mem_get_info()
    if free < 30 << 30:
        pytest.skip("needs ~30 GB of free device memory")
    b64.load_library()


def test_mime_past_4gib():
    raw = torch.empty(N, dtype=torch.uint8, device=DEV)
    fill(raw, SEED)
    m = b64.b64_encoded_len_wrapped(N, 76, True)
    assert m > 1 << 32
    w = b64.b64_encode_wrapped(raw, line_chars=76, crlf=True)
    assert w.numel() == m
    # sampled windows of whole lines vs the oracle (incl. the tail)
    rng = np.random.default_rng(97)
    for L0 in [0, LINES - 1000] + [int(v) for v in rng.integers(0, LINES - 1000, 6)]:
        L1 = min(L0 + 1000, LINES)
        b0, b1 = 57 * L0, min(57 * L1, N)
        ref = oracle.encode_wrapped(splitmix_bytes(SEED, b0, b1 - b0), 76, crlf=True)
        got = host(w[78 * L0: 78 * L0 + ref.size])
        assert np.array_equal(got, ref), L0
    # whitespace-tolerant decode back to the bytes
    y, st, ep = b64.b64_decode_ws(w)
    assert (st, ep) == (b64.B64_OK, -1) and y.numel() == N and torch.equal(y, raw)
    del y
    # despace of the wrapped text == the plain encoding
    t = b64.b64_encode(raw)
    d, dlen = b64.b64_despace(w)
    assert int(dlen.item()) == t.numel() and torch.equal(d[: t.numel()], t)
    del d, t
    # exact first-error offsets past 2^32 (line structure: byte 78k+j, j < 76)
    for pos in [(1 << 32) + 78 * 5 + 3, m - 200]:
        old = int(w[pos].item())
        w[pos] = ord("!")
        _, st, ep = b64.b64_decode_ws(w)
        assert (st, ep) == (b64.B64_ERR_INVALID_CHAR, pos), pos
        w[pos] = old
