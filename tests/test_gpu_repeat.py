"""Repeat-determinism stress (test infrastructure; compute-sanitizer's
racecheck / synccheck are closed on this GPU pool).

Every kernel family is run many times on the same input, each time into an
output buffer refilled with garbage and while a memory-heavy kernel runs on
another stream (so the CTAs land on different SMs at different times), and
every repetition must equal the oracle's result byte for byte -- output,
length, status and first-error offset.  A race between warps / CTAs (a
missing barrier, an mbarrier phase slip, a cross-CTA result record read too
early) shows up as a repetition that differs; this is evidence, not proof."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, host, to_dev

pytestmark = pytest.mark.gpu
REPS = int(os.environ.get("B64_REPEAT_REPS", "32"))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


@pytest.fixture(scope="module")
def noise():
    """A side stream and a 256 MiB buffer to keep it busy."""
    s = torch.cuda.Stream()
    big = torch.ones(64 << 20, dtype=torch.float32, device=DEV)
    return s, big


def _perturb(noise, rep):
    s, big = noise
    with torch.cuda.stream(s):
        for _ in range(rep % 3):
            big.mul_(1.0)


def _sync(noise):
    noise[0].synchronize()
    torch.cuda.synchronize()


def test_repeat_single_buffer_encode_decode(noise):
    n = 5_000_003
    x = splitmix_bytes(4101, 0, n)
    ref = oracle.encode(x)
    bad = ref.copy()
    rng = np.random.default_rng(4101)
    for p in rng.choice(ref.size - 4, 7, replace=False):
        bad[int(p)] = ord("*")
    rst, rep_, rout = oracle.decode(bad)
    d, t, tb = to_dev(x), to_dev(ref), to_dev(bad)
    out = torch.empty(ref.size, dtype=torch.uint8, device=DEV)
    y = torch.empty(n + 3, dtype=torch.uint8, device=DEV)
    res = b64.result_tensor(DEV)
    for r in range(REPS):
        out.fill_(0x5A)
        y.fill_(0x5A)
        _perturb(noise, r)
        b64.b64_encode(d, out=out)
        b64.b64_decode_async(tb, y, res)
        _sync(noise)
        assert np.array_equal(host(out), ref), r
        ol, ep, st, _ = b64.unpack_result(res)
        assert (st, ep, ol) == (rst, rep_, rout.size), r
        assert np.array_equal(host(y)[:ol], rout), r
        yc, st2, ep2 = b64.b64_decode(t)
        assert st2 == 0 and ep2 == -1 and np.array_equal(host(yc), x), r


def test_repeat_batched(noise):
    rng = np.random.default_rng(4102)
    k = 3000
    lens = np.floor(np.exp(rng.uniform(0, np.log(40001), k))).astype(np.int64) - 1
    off = np.zeros(k + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    raw = splitmix_bytes(4102, 0, int(off[-1]))
    texts = [oracle.encode(raw[off[i]:off[i + 1]]) for i in range(k)]
    toff = np.zeros(k + 1, dtype=np.int64)
    toff[1:] = np.cumsum([t.size for t in texts])
    cat = np.concatenate(texts)
    dirty = cat.copy()
    for i in range(0, k, 9):
        if texts[i].size:
            dirty[int(toff[i] + rng.integers(0, texts[i].size))] = ord("!")
    refs = [oracle.decode(dirty[toff[i]:toff[i + 1]]) for i in range(k)]
    d, doff = to_dev(raw), torch.from_numpy(off).to(DEV)
    dt, dtoff = to_dev(dirty), torch.from_numpy(toff).to(DEV)
    out = torch.empty(int(toff[-1]) + 16, dtype=torch.uint8, device=DEV)
    out_off = torch.empty(k + 1, dtype=torch.int64, device=DEV)
    y = torch.empty(int(off[-1]) + 16, dtype=torch.uint8, device=DEV)
    for r in range(REPS):
        out.fill_(0x5A)
        y.fill_(0x5A)
        _perturb(noise, r)
        b64.b64_encode_batch(d, doff, out=out, out_off=out_off)
        yy, yo, yl, ye, ys = b64.b64_decode_batch(dt, dtoff, out=y)
        _sync(noise)
        assert np.array_equal(host(out_off), toff), r
        assert np.array_equal(host(out)[:toff[-1]], cat), r
        yh, yoh, ylh, yeh, ysh = host(yy), host(yo), host(yl), host(ye), host(ys)
        for i in range(k):
            rst, rep_, rout = refs[i]
            assert (ysh[i], yeh[i], ylh[i]) == (rst, rep_, rout.size), (r, i)
            assert np.array_equal(yh[yoh[i]:yoh[i] + ylh[i]], rout), (r, i)


def _irregular_mime(nraw, seed):
    """76-char CRLF lines with every 7th line ending in ' \\n' and random
    extra spaces: not line-structured, so the general paths run."""
    raw = splitmix_bytes(seed, 0, nraw)
    lines = oracle.encode(raw)
    rows = [lines[i:i + 76] for i in range(0, lines.size, 76)]
    rng = np.random.default_rng(seed)
    parts = []
    for j, row in enumerate(rows):
        if rng.random() < 0.05:
            cut = int(rng.integers(0, row.size + 1))
            row = np.concatenate([row[:cut], np.frombuffer(b"  ", dtype=np.uint8), row[cut:]])
        parts.append(row)
        parts.append(np.frombuffer(b" \n" if j % 7 == 0 else b"\r\n", dtype=np.uint8))
    return raw, np.concatenate(parts)


def test_repeat_despace_and_ws_decode_general(noise):
    raw, text = _irregular_mime(3_000_000, 4103)
    kept = oracle.despace(text)
    bad = text.copy()
    pos = int(np.flatnonzero(bad == ord("A"))[12345])
    bad[pos] = ord("#")
    rst, rep_, rout = oracle.decode_ws(bad, 0)
    d, db = to_dev(text), to_dev(bad)
    out = torch.empty(text.size, dtype=torch.uint8, device=DEV)
    y = torch.empty(b64.b64_decoded_max_len(text.size), dtype=torch.uint8, device=DEV)
    res = b64.result_tensor(DEV)
    for r in range(REPS):
        out.fill_(0x5A)
        y.fill_(0x5A)
        _perturb(noise, r)
        o, olen = b64.b64_despace(d, out=out)
        _sync(noise)
        assert int(olen.item()) == kept.size and np.array_equal(host(o)[:kept.size], kept), r
        yy, st, ep = b64.b64_decode_ws(d)
        assert st == 0 and ep == -1 and np.array_equal(host(yy), raw), r
        b64.b64_decode_ws_async(db, y, res)
        _sync(noise)
        ol, ep2, st2, _ = b64.unpack_result(res)
        assert (st2, ep2, ol) == (rst, rep_, rout.size), r
        assert np.array_equal(host(y)[:ol], rout), r


def test_repeat_mime_fast_paths(noise):
    raw = splitmix_bytes(4104, 0, 57 * 40000 + 11)
    ref = oracle.encode_wrapped(raw, 76, 1)
    d = to_dev(raw)
    t = to_dev(ref)
    out = torch.empty(ref.size, dtype=torch.uint8, device=DEV)
    kept = oracle.despace(ref)
    dso = torch.empty(ref.size, dtype=torch.uint8, device=DEV)
    for r in range(REPS):
        out.fill_(0x5A)
        dso.fill_(0x5A)
        _perturb(noise, r)
        w = b64.b64_encode_wrapped(d, out=out, line_chars=76, crlf=True)
        o, olen = b64.b64_despace(t, out=dso)
        _sync(noise)
        assert np.array_equal(host(w), ref), r
        assert int(olen.item()) == kept.size and np.array_equal(host(o)[:kept.size], kept), r
        yy, st, ep = b64.b64_decode_ws(t)
        assert st == 0 and ep == -1 and np.array_equal(host(yy), raw), r
