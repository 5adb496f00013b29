"""GPU parity of the fused whitespace-tolerant decode (SURVEY.md §8(f) row f4,
reading R-ws-decode) against oracle.decode_ws: MIME-wrapped text across tile
(16 KiB) and chunk seams, random whitespace densities, whitespace-only
chunks, long whitespace runs, every error kind with its offset in ORIGINAL
coordinates, the variant flags, in/out misalignment and guard bytes."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, empty_dev, host, to_dev

pytestmark = pytest.mark.gpu
TILE = 16384
U, NP, ST = b64.B64_FLAG_URL, b64.B64_FLAG_NOPAD, b64.B64_FLAG_STRICT
WS = np.frombuffer(b" \n\r", dtype=np.uint8)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def gpu(w, fl=0, im=0, om=0):
    cap = b64.b64_decoded_max_len_ex(w.size, fl)
    base, out = empty_dev(cap, om)
    view, st, ep = b64.b64_decode_ws(to_dev(w, im), out=out, flags=fl)
    g = host(base)
    assert (g[:om] == 0xCC).all() and (g[om + cap:] == 0xCC).all(), "guard bytes"
    return st, ep, host(view)


def check(w, fl=0, im=0, om=0):
    st, ep, out = gpu(w, fl, im, om)
    rst, rep, rout = oracle.decode_ws(w, fl)
    assert (st, ep) == (rst, rep), (w.size, fl, im, om, st, ep, rst, rep)
    assert out.size == rout.size and np.array_equal(out, rout), (w.size, fl, im, om)


def mime(n, seed, line=76, crlf=True, fl=0):
    return oracle.encode_wrapped(splitmix_bytes(seed, 0, n), line, crlf=crlf, flags=fl)


def sprinkle(t, seed, frac):
    """Insert whitespace runs (1-3 bytes) before a fraction of t's bytes."""
    rng = np.random.default_rng(seed)
    k = t.size
    runs = (rng.random(k) < frac) * rng.integers(1, 4, k)
    out = np.empty(k + int(runs.sum()), dtype=np.uint8)
    pos = np.arange(k) + np.cumsum(runs)
    out[pos] = t
    mask = np.ones(out.size, dtype=bool)
    mask[pos] = False
    out[mask] = rng.choice(WS, size=int(mask.sum()))
    return out


def test_mime_sizes_across_seams():
    sizes = [0, 1, 2, 3, 56, 57, 58, 12_000, 12_285, 12_288, 12_300, 40_000, 300_001,
             1_000_000, 3_600_000]
    for n in sizes:
        for crlf in (True, False):
            check(mime(n, 400 + n % 13, crlf=crlf))


def test_large_multi_tile_chunks():
    # > 296 tiles: chunks hold several tiles (carry across tiles inside a chunk)
    for n, seed in [(9_000_001, 401), (15_728_640, 402)]:
        check(mime(n, seed))
        check(mime(n, seed, line=64, crlf=False))


@pytest.mark.parametrize("frac", [0.0, 0.01, 0.3, 2.0])
def test_random_whitespace_densities(frac):
    x = splitmix_bytes(403, 0, 200_000)
    t = oracle.encode(x)
    for k, n in enumerate([4, 5, 16, 17, 100, 4_096, 16_383, 49_153, t.size]):
        tt = t[:n] if n % 4 == 0 or n == t.size else t[:n]
        w = sprinkle(tt, 404 + k, min(frac, 1.0)) if frac else tt.copy()
        if frac > 1.0:  # heavy: every byte preceded by whitespace
            w = sprinkle(tt, 404 + k, 1.0)
        check(w)


def test_whitespace_only_chunks_and_long_runs():
    t = oracle.encode(splitmix_bytes(405, 0, 30_000))
    blank = np.full(5 * TILE + 123, ord(" "), dtype=np.uint8)
    blank[::7] = ord("\n")
    # data, a long blank stretch (whole empty tiles / chunks), data, trailing blanks
    w = np.concatenate([t[:10_001], blank, t[10_001:], blank[:3 * TILE]])
    check(w)
    check(blank)  # whitespace only: OK, 0 bytes
    check(np.concatenate([blank, t[:8]]))
    check(np.concatenate([t[:5], blank, t[5:8]]))  # a quad split by 80 KiB of blanks


def test_alignments():
    w = mime(120_000, 406)
    for im in range(0, 16, 3):
        for om in (0, 1, 4, 7, 12):
            check(w, 0, im, om)


def test_errors_in_original_coordinates():
    rng = np.random.default_rng(407)
    na = np.array([b for b in range(256) if b not in b" \n\r=" and oracle.A(b) < 0], dtype=np.uint8)
    base_w = mime(200_000, 408)
    for trial in range(60):
        w = base_w.copy()
        kind = trial % 4
        if kind == 0:  # one invalid byte somewhere
            w[int(rng.integers(0, w.size))] = na[int(rng.integers(0, na.size))]
        elif kind == 1:  # several invalid bytes
            for p in rng.choice(w.size, 5, replace=False):
                w[int(p)] = na[int(rng.integers(0, na.size))]
        elif kind == 2:  # a '=' in the middle
            p = int(rng.integers(0, w.size - 100))
            w[p] = ord("=")
        else:  # truncated stream (LENGTH, reported at a kept byte)
            w = w[: int(rng.integers(1, w.size))]
        check(w)


@pytest.mark.parametrize("fl", [U, NP, ST, U | NP | ST])
def test_variant_flags(fl):
    rng = np.random.default_rng(409)
    for n in [0, 1, 2, 3, 4, 5, 1000, 57 * 300 + 1, 57 * 300 + 2, 250_000]:
        w = mime(n, 410 + n % 7, fl=fl & ~ST)
        check(w, fl)
        if n and fl & ST:
            # break canonicity of the last data character (App. A)
            t = oracle.encode_ex(splitmix_bytes(411, 0, n), fl & ~ST)
            if t[-1] == ord("=") or (fl & NP and n % 3):
                j = t.size - 1
                while t[j] == ord("="):
                    j -= 1
                t = t.copy()
                t[j] ^= 1
                check(sprinkle(t, 412, 0.05), fl)
        if n > 10:
            w2 = w.copy()
            w2[int(rng.integers(0, w2.size))] = ord("!")
            check(w2, fl)


def test_async_result_record():
    w = mime(50_000, 413)
    d = to_dev(w)
    out = torch.empty(b64.b64_decoded_max_len(w.size), dtype=torch.uint8, device=d.device)
    res = b64.result_tensor(d.device)
    b64.b64_decode_ws_async(d, out, res)
    ol, ep, st, pc = b64.unpack_result(res)
    rst, rep, rout = oracle.decode_ws(w)
    assert (st, ep, ol) == (rst, rep, rout.size)
    assert np.array_equal(host(out[:ol]), rout)


def _verdict(w, fl=0):
    """Run the ws decode with an explicit workspace and return the fast-path
    verdict stored in it (1 = line-structured fast path, 0 = general path)."""
    ws = torch.empty(b64.b64_decode_ws_workspace_bytes(w.size) + 64, dtype=torch.uint8, device=DEV)
    b64.b64_decode_ws(to_dev(w), flags=fl, ws=ws)
    return int(ws[48:52].view(torch.int32).item())


def test_fast_path_taken_exactly_on_line_structure():
    x = splitmix_bytes(420, 0, 100_000)
    assert _verdict(oracle.encode_wrapped(x, 76, crlf=True)) == 1
    assert _verdict(oracle.encode_wrapped(x, 64, crlf=False)) == 1
    assert _verdict(oracle.encode_wrapped(x[:1000], 76, crlf=True)[:-2]) == 1   # no final EOL
    assert _verdict(oracle.encode_wrapped(x, 76, crlf=True, flags=NP), NP) == 1
    assert _verdict(oracle.encode(x)) == 0                                   # no white space
    w = oracle.encode_wrapped(x, 76, crlf=True)
    for cut in (5, 78 * 500 + 77, w.size - 1):                               # a stray byte
        u = np.insert(w, cut, ord(" "))
        assert _verdict(u) == 0
        check(u)
    u = w.copy()
    u[78 * 700 + 10] = ord("!")                                              # an error
    assert _verdict(u) == 0
    check(u)


# L: G = L / 4 quads per line; the interior tiles take the line-major path
# for G <= 32 (one lane per line, lane stride 1 or 2 by (G, e)), the flat
# path above; 24 / 40 / 68: stride-2 maps, 60: stride 2 with CR LF and 1
# with LF, 80 / 128: stride 1, 132: flat
@pytest.mark.parametrize("L", [4, 8, 24, 40, 60, 64, 68, 76, 80, 128, 132, 1000, 4092])
@pytest.mark.parametrize("crlf", [False, True])
def test_line_structured_lengths(L, crlf):
    # the fast path across tile seams for every line length; tails of 1..L chars
    x = splitmix_bytes(421 + L, 0, 600_000)
    for n in [1, 2, 3, 3 * L // 4, 3 * L // 4 + 1, 7 * L, 300_000, 600_000 - 1]:
        w = oracle.encode_wrapped(x[:n], L, crlf=crlf)
        check(w)
        check(w[: w.size - (2 if crlf else 1)])  # without the final EOL
        if n >= 300_000:
            assert _verdict(w) == 1


def test_line_major_large_aligned():
    """The line-major interior path at sizes where tiles hold whole 64-line
    blocks per warp (two lines per lane), over input / output misalignments,
    with the fast path's verdict checked."""
    x = splitmix_bytes(430, 0, 20 << 20)
    for L, crlf in ((76, True), (64, False), (40, True)):
        w = oracle.encode_wrapped(x, L, crlf=crlf)
        assert _verdict(w) == 1
        for im, om in ((0, 0), (1, 0), (0, 3), (7, 13), (15, 15)):
            check(w, 0, im, om)
    for fl in (U, NP, U | NP | ST):
        w = oracle.encode_wrapped(x[: (20 << 20) - 1], 76, crlf=True, flags=fl & ~ST)
        assert _verdict(w, fl) == 1
        check(w, fl, 3, 5)
