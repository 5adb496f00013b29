"""GPU parity of the line-wrapped encode (reading
R-wrap) against oracle.encode_wrapped: every short length, tile seams, line
lengths 4 .. 16384, LF / CRLF, the URL / NOPAD flags, in/out misalignment with
guard bytes, and the round trip through the whitespace-tolerant decode."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import empty_dev, host, to_dev

pytestmark = pytest.mark.gpu
U, NP = b64.B64_FLAG_URL, b64.B64_FLAG_NOPAD


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def check(x, L, crlf, fl=0, im=0, om=0):
    cap = b64.b64_encoded_len_wrapped(x.size, L, crlf, fl)
    base, out = empty_dev(cap, om)
    v = b64.b64_encode_wrapped(to_dev(x, im), out=out, line_chars=L, crlf=crlf, flags=fl)
    torch.cuda.synchronize()
    ref = oracle.encode_wrapped(x, L, crlf=crlf, flags=fl)
    assert v.numel() == ref.size == cap, (x.size, L, crlf, fl)
    assert np.array_equal(host(v), ref), (x.size, L, crlf, fl, im, om)
    g = host(base)
    assert (g[:om] == 0xCC).all() and (g[om + cap:] == 0xCC).all(), "guard bytes"


def test_every_short_length():
    x = splitmix_bytes(500, 0, 400)
    for n in range(0, 400):
        for crlf in (True, False):
            check(x[:n], 76, crlf)


@pytest.mark.parametrize("L", [4, 8, 12, 64, 76, 100, 1024, 16384])
def test_line_lengths_and_seams(L):
    x = splitmix_bytes(501, 0, 700_000)
    G = L // 4
    for crlf in (True, False):
        # lines per tile as b64_encode_wrapped chooses them (21 KiB in / 28 KiB out caps)
        lt = min(21504 // (3 * G), 28672 // (L + (2 if crlf else 1)))
        tile_in = lt * 3 * G
        for n in [1, 2, 3, tile_in - 1, tile_in, tile_in + 1, 3 * tile_in + 2, 700_000]:
            check(x[:n], L, crlf)


@pytest.mark.parametrize("fl", [U, NP, U | NP])
def test_flags(fl):
    x = splitmix_bytes(502, 0, 100_000)
    for n in list(range(0, 120)) + [12_287, 12_288, 12_289, 100_000]:
        check(x[:n], 76, True, fl)
        check(x[:n], 64, False, fl)


def test_alignments():
    x = splitmix_bytes(503, 0, 50_001)
    for im in range(0, 16, 3):
        for om in range(0, 16, 5):
            check(x, 76, True, 0, im, om)
            check(x, 76, False, 0, im, om)


def test_large_and_roundtrip_through_ws_decode():
    x = splitmix_bytes(504, 0, 57 * (1 << 18) + 5)
    check(x, 76, True)
    d = to_dev(x)
    w = b64.b64_encode_wrapped(d, line_chars=76, crlf=True)
    y, st, ep = b64.b64_decode_ws(w)
    assert (st, ep) == (0, -1) and torch.equal(y, d)


def _lm_tile_lines(n, L, crlf):
    """Lines per tile of the line-major encoder (b64_encode_wrapped, L <= 128),
    as the host computes them: 57 KiB of input, a whole number of 32- or
    64-line blocks per compute warp, >= 2 tiles per SM for small inputs."""
    G, e = L // 4, (2 if crlf else 1)
    strd = 2 if (0x77f7800072620 >> (G - 1 + 32 * (e - 1))) & 1 else 1
    lt = (1024 * 57) // (3 * G)
    unit = 16 * 32 * strd
    if lt >= unit:
        lt -= lt % unit
    m = 4 * ((n + 2) // 3)
    nlines = (m + L - 1) // L
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    want = (nlines + 2 * sms - 1) // (2 * sms)
    return max(1, want) if want < lt else lt


@pytest.mark.parametrize("L", [4, 24, 40, 60, 64, 76, 128])
def test_line_major_tiles_and_seams(L):
    """The line-major encoder across its tile seams at sizes where tiles hold
    whole blocks per warp (two lines per lane on stride-2 maps), with and
    without a partial final line."""
    G = L // 4
    for crlf in (True, False):
        n0 = 40 << 20
        lt = _lm_tile_lines(n0, L, crlf)
        tin = lt * 3 * G
        k = n0 // tin
        x = splitmix_bytes(505 + L, 0, k * tin + 3 * G + 2)
        for n in (k * tin, k * tin - 1, k * tin + 1, k * tin + 3 * G, k * tin + 3 * G + 2):
            check(x[:n], L, crlf)


def test_line_major_alignments_and_flags():
    x = splitmix_bytes(506, 0, 20 << 20)
    for im, om in ((1, 0), (0, 3), (7, 13), (15, 15)):
        check(x, 76, True, 0, im, om)
        check(x, 64, False, 0, im, om)
    for fl in (U, NP, U | NP):
        check(x[: (20 << 20) - 1], 76, True, fl)
        check(x[: (20 << 20) - 2], 64, False, fl, 5, 9)
