"""Seeded randomized parity across every entry point of the C ABI against
the CPU oracle (SURVEY.md §8(c) parity bar): random lengths (log-uniform,
including 0 and tile / unit / line boundaries), variant flags, in/out
misalignment, corruptions of every kind (non-alphabet bytes, a misplaced
'=', truncation, a non-canonical final quad under STRICT), random white
space, random line geometry.  Every case compares output bytes, lengths,
status and error offset exactly; output guard bytes must stay untouched.
The cases are drawn from numpy generators with fixed seeds, so a failure
names a reproducible (seed, case)."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, empty_dev, host, to_dev

pytestmark = pytest.mark.gpu

U, NP, ST = b64.B64_FLAG_URL, b64.B64_FLAG_NOPAD, b64.B64_FLAG_STRICT
FLAGS = [0, U, NP, ST, U | NP, NP | ST, U | ST, U | NP | ST]
WS = np.frombuffer(b" \n\r", dtype=np.uint8)
# B64_FUZZ_SCALE multiplies every case count, B64_FUZZ_SEED shifts every
# seed (longer one-off runs; the defaults are the committed suite).
SCALE = int(os.environ.get("B64_FUZZ_SCALE", "1"))
SEED = int(os.environ.get("B64_FUZZ_SEED", "0"))
NA = np.array([b for b in range(256) if b not in b"=" and oracle.A(b) < 0 and oracle.A_ex(b, U) < 0
               and b not in b" \n\r"], dtype=np.uint8)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def rand_len(rng, hi=300_000):
    """Log-uniform in [0, hi], with extra mass on small and boundary sizes."""
    r = rng.random()
    if r < 0.15:
        return int(rng.integers(0, 20))
    if r < 0.25:  # near a multiple of the single-buffer tiles / batched units
        base = int(rng.choice([12288, 16384, 1536, 2048, 57, 76]))
        return max(0, base * int(rng.integers(1, 6)) + int(rng.integers(-4, 5)))
    return int(np.exp(rng.uniform(0, np.log(hi))))


def corrupt(rng, t, fl):
    """One random corruption of text t (a copy), or t itself."""
    t = t.copy()
    kind = int(rng.integers(0, 6))
    if t.size == 0 or kind == 0:
        return t
    if kind == 1:  # a non-alphabet byte
        t[int(rng.integers(0, t.size))] = NA[int(rng.integers(0, NA.size))]
    elif kind == 2:  # several
        for p in rng.choice(t.size, min(t.size, 4), replace=False):
            t[int(p)] = NA[int(rng.integers(0, NA.size))]
    elif kind == 3:  # a '=' anywhere
        t[int(rng.integers(0, t.size))] = ord("=")
    elif kind == 4:  # truncation
        t = t[: int(rng.integers(0, t.size))]
    else:  # flip a low bit of the last data character (non-canonical under STRICT)
        j = t.size - 1
        while j > 0 and t[j] == ord("="):
            j -= 1
        alt = t.copy()
        alt[j] ^= 1
        if oracle.A_ex(int(alt[j]), fl) >= 0:
            t = alt
    return t


def test_fuzz_single_buffer():
    rng = np.random.default_rng(9001 + SEED)
    for case in range(400 * SCALE):
        n = rand_len(rng)
        fl = FLAGS[int(rng.integers(0, len(FLAGS)))]
        im, om = int(rng.integers(0, 16)), int(rng.integers(0, 16))
        x = splitmix_bytes(9001, case * 1_000_003, case * 1_000_003 + n)
        # encode
        m = b64.b64_encoded_len_ex(n, fl)
        base, out = empty_dev(m, om)
        res = b64.b64_encode(to_dev(x, im), out=out, flags=fl & ~ST)
        g = host(base)
        assert (g[:om] == 0xCC).all() and (g[om + m:] == 0xCC).all(), ("guard", case)
        t = oracle.encode_ex(x, fl & ~ST)
        assert np.array_equal(host(res), t), ("encode", case, n, fl)
        # decode (clean or corrupted)
        c = corrupt(rng, t, fl)
        cap = b64.b64_decoded_max_len_ex(c.size, fl)
        base, out = empty_dev(cap, om)
        view, st, ep = b64.b64_decode(to_dev(c, im), out=out, flags=fl)
        g = host(base)
        assert (g[:om] == 0xCC).all() and (g[om + cap:] == 0xCC).all(), ("guard", case)
        rst, rep, rout = oracle.decode_ex(c, fl)
        assert (st, ep) == (rst, rep), ("decode", case, c.size, fl, st, ep, rst, rep)
        assert np.array_equal(host(view), rout), ("decode bytes", case)


def test_fuzz_batched():
    rng = np.random.default_rng(9002 + SEED)
    for case in range(60 * SCALE):
        k = int(rng.integers(0, 400))
        mode = case % 3
        if mode == 0:
            lens = np.array([rand_len(rng, 20_000) for _ in range(k)], dtype=np.int64)
        elif mode == 1:  # tiny messages, many empty
            lens = rng.integers(0, 9, k).astype(np.int64)
        else:  # data-URI-like
            lens = np.exp(rng.uniform(np.log(100), np.log(65536), k)).astype(np.int64)
        fl = FLAGS[int(rng.integers(0, len(FLAGS)))]
        off = np.zeros(k + 1, dtype=np.int64)
        off[1:] = np.cumsum(lens)
        raw = splitmix_bytes(9002, case * 7_000_001, case * 7_000_001 + int(off[-1]))
        im = int(rng.integers(0, 16))
        out, oo = b64.b64_encode_batch(to_dev(raw, im), torch.from_numpy(off).to(DEV), flags=fl & ~ST)
        o, oo = host(out), host(oo)
        texts = [oracle.encode_ex(raw[off[i]: off[i + 1]], fl & ~ST) for i in range(k)]
        for i, t in enumerate(texts):
            assert np.array_equal(o[oo[i]: oo[i + 1]], t), ("batch encode", case, i, fl)
        texts = [corrupt(rng, t, fl) if rng.random() < 0.3 else t for t in texts]
        toff = np.zeros(k + 1, dtype=np.int64)
        toff[1:] = np.cumsum([t.size for t in texts])
        cat = np.concatenate(texts) if k else np.zeros(0, dtype=np.uint8)
        y, yo, yl, ye, ys = b64.b64_decode_batch(to_dev(cat, int(rng.integers(0, 16))),
                                                 torch.from_numpy(toff).to(DEV), flags=fl)
        y, yo, yl, ye, ys = host(y), host(yo), host(yl), host(ye), host(ys)
        for i, t in enumerate(texts):
            rst, rep, rout = oracle.decode_ex(t, fl)
            assert (ys[i], ye[i], yl[i]) == (rst, rep, rout.size), ("batch decode", case, i, fl)
            assert np.array_equal(y[yo[i]: yo[i] + yl[i]], rout), ("batch decode bytes", case, i)


def sprinkle(rng, t, frac):
    k = t.size
    runs = (rng.random(k) < frac) * rng.integers(1, 4, k)
    out = np.empty(k + int(runs.sum()), dtype=np.uint8)
    pos = np.arange(k) + np.cumsum(runs)
    out[pos] = t
    mask = np.ones(out.size, dtype=bool)
    mask[pos] = False
    out[mask] = rng.choice(WS, size=int(mask.sum()))
    return out


def test_fuzz_whitespace_and_lines():
    rng = np.random.default_rng(9003 + SEED)
    for case in range(200 * SCALE):
        n = rand_len(rng, 400_000)
        fl = FLAGS[int(rng.integers(0, len(FLAGS)))]
        x = splitmix_bytes(9003, case * 5_000_011, case * 5_000_011 + n)
        L = 4 * int(rng.integers(1, 40)) if rng.random() < 0.5 else int(rng.choice([64, 76]))
        crlf = bool(rng.integers(0, 2))
        # wrapped encode
        m = b64.b64_encoded_len_wrapped(n, L, crlf, fl & ~ST)
        om = 2 * int(rng.integers(0, 8)) + (0 if rng.random() < 0.7 else 1)
        base, out = empty_dev(m, om)
        res = b64.b64_encode_wrapped(to_dev(x, int(rng.integers(0, 16))), out=out, line_chars=L,
                                     crlf=crlf, flags=fl & ~ST)
        torch.cuda.synchronize()
        g = host(base)
        assert (g[:om] == 0xCC).all() and (g[om + m:] == 0xCC).all(), ("guard", case)
        w = oracle.encode_wrapped(x, L, crlf=crlf, flags=fl & ~ST)
        assert np.array_equal(host(res), w), ("wrap", case, n, L, crlf, fl)
        # whitespace-tolerant decode of: the wrapped text, a sprinkled one, or a corrupted one
        r = rng.random()
        if r < 0.35:
            c = w
        elif r < 0.7:
            c = sprinkle(rng, oracle.encode_ex(x, fl & ~ST), float(rng.choice([0.001, 0.05, 0.5])))
        else:
            c = corrupt(rng, w, fl)
        cap = b64.b64_decoded_max_len_ex(c.size, fl)
        base, out = empty_dev(cap, om)
        view, st, ep = b64.b64_decode_ws(to_dev(c, int(rng.integers(0, 16))), out=out, flags=fl)
        g = host(base)
        assert (g[:om] == 0xCC).all() and (g[om + cap:] == 0xCC).all(), ("guard", case)
        rst, rep, rout = oracle.decode_ws(c, fl)
        assert (st, ep) == (rst, rep), ("decode_ws", case, c.size, fl, st, ep, rst, rep)
        assert np.array_equal(host(view), rout), ("decode_ws bytes", case)
        # despace
        d, dl = b64.b64_despace(to_dev(c, int(rng.integers(0, 16))))
        ref = oracle.despace(c)
        nl = int(host(dl)[0])
        assert nl == ref.size and np.array_equal(host(d[:nl]), ref), ("despace", case)


def test_fuzz_shards():
    """Random world sizes and lengths: per-rank encode of b64_shard ranges
    concatenates to the whole-buffer encoding; per-rank shard decodes
    combine (min error offset, summed lengths) to the whole-buffer decode."""
    from tests.test_gpu_parity import emulate_sharded_decode

    rng = np.random.default_rng(9004 + SEED)
    for case in range(40 * SCALE):
        n = rand_len(rng, 500_000)
        world = int(rng.integers(1, 9))
        x = splitmix_bytes(9004, case * 3_000_017, case * 3_000_017 + n)
        parts = []
        for r in range(world):
            b, e = b64.b64_shard(n, 3, world, r)
            parts.append(host(b64.b64_encode(to_dev(x[b:e], int(rng.integers(0, 16))))))
        t = np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint8)
        assert np.array_equal(t, oracle.encode(x)), ("shard encode", case, n, world)
        c = corrupt(rng, t, 0)
        flags = int(rng.integers(0, 8)) if case % 2 else 0
        if flags:
            t = oracle.encode_ex(x, flags)
            c = corrupt(rng, t, flags)
        st, ep, ol, outs = emulate_sharded_decode(c, world, flags, rng=rng)
        rst, rep, rout = oracle.decode_ex(c, flags)
        assert (st, ep, ol) == (rst, rep, rout.size), ("shard decode", case, world, flags, st, ep, rst, rep)
        assert np.array_equal(np.concatenate(outs)[:ol], rout), ("shard bytes", case)


def test_fuzz_host_buffers():
    """The host-buffer pipeline (copies inside the call) on random sizes,
    pinned and pageable host memory, clean and corrupted text."""
    rng = np.random.default_rng(9005 + SEED)
    for case in range(20 * SCALE):
        n = rand_len(rng, 3_000_000)
        x = splitmix_bytes(9005, case * 4_000_037, case * 4_000_037 + n)
        pin = bool(rng.integers(0, 2))
        mk = (lambda a: torch.from_numpy(a).pin_memory()) if pin else torch.from_numpy
        flags = int(rng.integers(0, 8)) if case % 2 else 0
        m = b64.b64_encoded_len_ex(n, flags)
        hx = mk(x.copy())
        ht = mk(np.empty(m, dtype=np.uint8))
        si = torch.empty(max(m, 1), dtype=torch.uint8, device=DEV)
        so = torch.empty(max(m, 1), dtype=torch.uint8, device=DEV)
        assert b64.b64_encode_host(hx, ht, si, so, flags=flags) == m
        t = oracle.encode_ex(x, flags)
        assert np.array_equal(ht.numpy(), t), ("host encode", case, n, pin, flags)
        c = corrupt(rng, t, 0)
        hc = mk(c.copy())
        hy = mk(np.empty(max(b64.b64_decoded_max_len_ex(c.size, flags), 1), dtype=np.uint8))
        st, ol, ep = b64.b64_decode_host(hc, hy, si, so, flags=flags)
        rst, rep, rout = oracle.decode_ex(c, flags)
        assert (st, ep, ol) == (rst, rep, rout.size), ("host decode", case, st, ep, rst, rep)
        assert np.array_equal(hy.numpy()[:ol], rout), ("host decode bytes", case)


@pytest.mark.parametrize("k,hi", [(2_000_000, 100), (300_000, 2000)])
def test_batched_many_messages(k, hi):
    """Millions of tiny messages (per-warp first-message table, walker
    windows, plan chunks of thousands of messages per CTA): every sampled
    message and every corrupted one matches the oracle."""
    rng = np.random.default_rng(9006 + k)
    lens = rng.integers(0, hi, k).astype(np.int64)
    off = np.zeros(k + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    raw = splitmix_bytes(9006, 0, int(off[-1]))
    out, oo = b64.b64_encode_batch(to_dev(raw), torch.from_numpy(off).to(DEV))
    o, oo = host(out), host(oo)
    idx = rng.choice(k, 1500, replace=False)
    for i in idx:
        assert np.array_equal(o[oo[i]:oo[i + 1]], oracle.encode(raw[off[i]:off[i + 1]])), (k, i)
    cat = o[:oo[k]].copy()
    toff = oo.astype(np.int64)
    bad = rng.choice(k, 1000, replace=False)
    for i in bad:
        if toff[i + 1] > toff[i]:
            cat[int(rng.integers(toff[i], toff[i + 1]))] = ord("!")
    y, yo, yl, ye, ys = b64.b64_decode_batch(to_dev(cat), torch.from_numpy(toff).to(DEV))
    y, yo, yl, ye, ys = host(y), host(yo), host(yl), host(ye), host(ys)
    for i in np.concatenate([idx, bad]):
        rst, rep, rout = oracle.decode(cat[toff[i]:toff[i + 1]])
        assert (ys[i], ye[i], yl[i]) == (rst, rep, rout.size), (k, i)
        assert np.array_equal(y[yo[i]:yo[i] + yl[i]], rout), (k, i)
