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


# ---- line-structured fast path (MIME / PEM text): one strided copy with the
# line structure verified; anything else falls back to the two-pass path.
# The verdict word sits at the start of the workspace (WlState.verdict).

def despace_with_verdict(w, im=0, om=0):
    lib = b64.load_library()
    ws = torch.empty(lib.b64_despace_workspace_bytes(w.size) + 256, dtype=torch.uint8, device=DEV)
    base, out = empty_dev(max(w.size, 1), om)
    o, olen = b64.b64_despace(to_dev(w, im), out=out, ws=ws)
    n = int(olen.item())
    g = host(base)
    assert (g[:om] == 0xCC).all() and (g[om + max(w.size, 1):] == 0xCC).all(), "guard bytes"
    verdict = int(ws[:4].view(torch.int32).item()) if w.size else 1
    return host(o)[:n], verdict


def wrapped(n, seed, line=76, crlf=True, final_eol=True):
    w = oracle.encode_wrapped(splitmix_bytes(seed, 0, n), line, crlf=crlf)
    if not final_eol and w.size:
        w = w[: w.size - (2 if crlf else 1)]
    return w


def test_lines_fast_path_sizes():
    for n in [1, 2, 3, 56, 57, 58, 57 * 20, 12_285, 12_300, 300_001, 3_600_000]:
        for line, crlf in ((76, True), (64, False), (4, True), (4092, False)):
            for fe in (True, False):
                w = wrapped(n, 310 + n % 11, line, crlf, fe)
                got, v = despace_with_verdict(w)
                assert np.array_equal(got, oracle.despace(w)), (n, line, crlf, fe)
                # text without any EOL (one line, no final EOL) has no line
                # structure to detect: the general path handles it
                assert v == int((w == 10).any()), (n, line, crlf, fe)


def test_lines_fast_path_large_and_aligned():
    w = wrapped(57 * (1 << 18) + 5, 311)  # many tiles per CTA, short final line
    ref = oracle.despace(w)
    for im, om in ((0, 0), (1, 0), (0, 3), (7, 13)):
        got, v = despace_with_verdict(w, im, om)
        assert v == 1 and np.array_equal(got, ref), (im, om)


@pytest.mark.parametrize("kind", ["space_in_line", "tab", "ctrl", "extra_eol", "missing_eol", "bad_eol",
                                  "trailing_space", "lf_in_crlf", "first_line_space", "line_not_mult4"])
def test_lines_fast_path_falls_back(kind):
    """Text that is not line-structured (or has a byte < 0x21 inside a line)
    gives the plain Appendix B result through the general path."""
    w = wrapped(300_000, 312)
    b = bytearray(w.tobytes())
    mid = 78 * 1500 + 30
    if kind == "space_in_line":
        b[mid] = 0x20
    elif kind == "tab":
        b[mid] = 0x09          # kept by Appendix B: must survive
    elif kind == "ctrl":
        b[mid] = 0x01
    elif kind == "extra_eol":
        b[mid:mid] = b"\r\n"
    elif kind == "missing_eol":
        del b[78 * 1500 + 76: 78 * 1500 + 78]
    elif kind == "bad_eol":
        b[78 * 1500 + 76] = ord(" ")
    elif kind == "trailing_space":
        b[-2:-2] = b" "
    elif kind == "lf_in_crlf":
        b[78 * 1500 + 76] = ord("\n")
    elif kind == "first_line_space":
        b[10] = 0x20
    elif kind == "line_not_mult4":
        b = bytearray(b"\r\n".join(bytes(w[i: i + 75]) for i in range(0, 75 * 100, 75)))
    x = np.frombuffer(bytes(b), dtype=np.uint8).copy()
    got, v = despace_with_verdict(x)
    assert np.array_equal(got, oracle.despace(x)), kind
    assert v == 0, kind


def test_lines_fast_path_tail_cases():
    w = wrapped(57 * 300 + 2, 313)  # partial final quad ('=' pad) on a short final line
    for tail in (b"", b"\r\n", b" ", b"\n", b"\r\n\r\n", b"A", b"AB\r\n"):
        x = np.concatenate([w[:-2], np.frombuffer(tail, dtype=np.uint8)])
        got, _ = despace_with_verdict(x)
        assert np.array_equal(got, oracle.despace(x)), tail
