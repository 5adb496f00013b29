"""GPU parity: libb64gpu.so (through the C ABI) vs the CPU oracle, bit-exact
on output bytes, lengths, status and first-error offset.  Small and ragged
sizes, every alignment, every byte at every position, the final-quad rules,
multi-error buffers, tile / CTA / ring-wrap boundaries.  Config-size parity
lives in tests/test_gpu_configs.py."""
import string

import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, empty_dev, host, to_dev

pytestmark = pytest.mark.gpu

ALPHABET = (string.ascii_uppercase + string.ascii_lowercase + string.digits + "+/").encode()
# Single-buffer tile geometry (b64_codec.cuh EncG / DecG, 512 compute threads):
# the default 4 passes per tile, and 2 passes for inputs with fewer than 2
# default tiles per SM (b64_lib.cu kSmallPasses).
ENC_TILE, ENC_TILE_SMALL = 24576, 12288    # input bytes per encode tile
DEC_TILE, DEC_TILE_SMALL = 32768, 16384    # input chars per decode tile
SMALL_LIMIT = 2 * 148                      # default tiles below which the small geometry runs


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def gpu_encode(x, in_mis=0, out_mis=0):
    d = to_dev(x, in_mis)
    base, out = empty_dev(b64.b64_encoded_len(x.size), out_mis)
    res = b64.b64_encode(d, out=out)
    torch.cuda.synchronize()
    # guard bytes around the output must be untouched
    g = host(base)
    assert (g[:out_mis] == 0xCC).all() and (g[out_mis + out.numel():] == 0xCC).all()
    return host(res)


def gpu_decode(t, in_mis=0, out_mis=0):
    d = to_dev(t, in_mis)
    cap = b64.b64_decoded_max_len(t.size)
    base, out = empty_dev(cap, out_mis)
    view, st, ep = b64.b64_decode(d, out=out)
    g = host(base)
    assert (g[:out_mis] == 0xCC).all() and (g[out_mis + cap:] == 0xCC).all()
    return st, ep, host(view)


def check_decode(t, in_mis=0, out_mis=0):
    st, ep, out = gpu_decode(t, in_mis, out_mis)
    rst, rep, rout = oracle.decode(t)
    assert (st, ep) == (rst, rep), (t.size, st, ep, rst, rep)
    assert out.size == rout.size
    assert np.array_equal(out, rout)


# ------------------------------------------------------------------ encode

def test_encode_every_length_0_to_1024():
    x = splitmix_bytes(101, 0, 1024)
    for n in range(0, 1025):
        assert np.array_equal(gpu_encode(x[:n]), oracle.encode(x[:n])), n


# (tile size, tile count): small-geometry boundaries below the switch,
# default-geometry boundaries above it, and both sides of the switch itself
ENC_CASES = [(ENC_TILE_SMALL, t) for t in (1, 2, 3, 295, 296, 297)] + \
    [(ENC_TILE, t) for t in (SMALL_LIMIT - 1, SMALL_LIMIT, SMALL_LIMIT + 1, 296 * 4 + 1, 296 * 9 + 7)]


@pytest.mark.parametrize("tile,tiles", ENC_CASES)
def test_encode_tile_ring_boundaries(tile, tiles):
    base = tiles * tile
    x = splitmix_bytes(102, 0, base + 4)
    for d in (-3, -2, -1, 0, 1, 2, 3, 4):
        n = base + d
        if n >= 0:
            assert np.array_equal(gpu_encode(x[:n]), oracle.encode(x[:n])), n


def test_encode_all_misalignments():
    x = splitmix_bytes(103, 0, 70000)
    for n in (1, 2, 5, 47, 48, 49, 383, 6144 + 7, 70000):
        ref = oracle.encode(x[:n])
        for im in range(16):
            for om in range(16):
                assert np.array_equal(gpu_encode(x[:n], im, om), ref), (n, im, om)


def test_encode_2_24_triples_closed_form():
    t = np.arange(1 << 24, dtype=np.uint32)
    triples = np.stack([(t >> 16) & 255, (t >> 8) & 255, t & 255], axis=1).astype(np.uint8).ravel()
    alpha = np.frombuffer(ALPHABET, dtype=np.uint8)
    idx = np.indices((64, 64, 64, 64), dtype=np.uint8).reshape(4, -1).T
    expect = alpha[idx].ravel()
    enc = gpu_encode(triples)
    assert np.array_equal(enc, expect)
    st, ep, dec = gpu_decode(enc)
    assert (st, ep) == (b64.B64_OK, -1)
    assert np.array_equal(dec, triples)


# ------------------------------------------------------------------ decode

def test_decode_every_length_roundtrip():
    x = splitmix_bytes(104, 0, 1024)
    for n in range(0, 1025):
        check_decode(oracle.encode(x[:n]))


def test_decode_length_errors():
    x = splitmix_bytes(105, 0, 20000)
    t = oracle.encode(x)
    for m in list(range(0, 40)) + [8191, 8193, 8194, 8195, 16385, 26665, 26666, 26667]:
        check_decode(t[:m])
    # invalid byte before the length error wins; one after it does not matter
    u = t[:4003].copy()
    u[17] = ord("!")
    check_decode(u)
    u = t[:4003].copy()
    u[4001] = ord("!")
    check_decode(u)


DEC_CASES = [(DEC_TILE_SMALL, t) for t in (1, 2, 295, 296, 297)] + \
    [(DEC_TILE, t) for t in (SMALL_LIMIT - 1, SMALL_LIMIT, SMALL_LIMIT + 1, 296 * 5 + 3)]


@pytest.mark.parametrize("tile,tiles", DEC_CASES)
def test_decode_tile_ring_boundaries(tile, tiles):
    m0 = tiles * tile
    x = splitmix_bytes(106, 0, 3 * (m0 // 4) + 12)
    t = oracle.encode(x)
    for d in (-8, -4, 0, 4, 8):
        check_decode(t[: m0 + d])
    # padded tails straddling a tile boundary
    for n in (3 * (m0 // 4) - 1, 3 * (m0 // 4) + 1, 3 * (m0 // 4) + 2):
        check_decode(oracle.encode(x[:n]))


def test_decode_all_misalignments():
    x = splitmix_bytes(107, 0, 60000)
    for n in (1, 2, 3, 35, 36, 6144 + 1, 60000):
        t = oracle.encode(x[:n])
        for im in range(16):
            for om in range(16):
                check_decode(t, im, om)


def test_decode_every_byte_at_every_position_of_a_block():
    """All 256 byte values at each position of a 64-char block in the middle
    of a 3-tile buffer, at the 16-char thread seams and the tile seam."""
    x = splitmix_bytes(108, 0, 3 * DEC_TILE_SMALL)
    t = oracle.encode(x)          # 4 * DEC_TILE_SMALL chars (small geometry), no padding
    positions = list(range(4096, 4096 + 64)) + [15, 16, 3071, 3072, 16383, 16384, 16385, 32767, t.size - 1, t.size - 2]
    d = to_dev(t)
    cap = b64.b64_decoded_max_len(t.size)
    _, out = empty_dev(cap)
    for pos in positions:
        for b in range(256):
            d[pos] = b
            view, st, ep = b64.b64_decode(d, out=out)
            u = t.copy()
            u[pos] = b
            rst, rep, rout = oracle.decode(u)
            assert (st, ep) == (rst, rep), (pos, b)
            assert view.numel() == rout.size
            assert np.array_equal(host(view), rout), (pos, b)
        d[pos] = int(t[pos])


def test_decode_final_quads_single_buffer():
    """Every 'xx==' and 'xxx=' final quad with non-canonical bits, plus '='
    misplacements, after a 4-char prefix; a sample through the single-buffer
    path (the full 64^2 + 64^3 sweep runs through the batched path)."""
    rng = np.random.default_rng(109)
    alpha = np.frombuffer(ALPHABET, dtype=np.uint8)
    cases = []
    for a in alpha[::5]:
        for b in alpha[::3]:
            cases.append([a, b, 61, 61])
            cases.append([a, b, rng.choice(alpha), 61])
            cases.append([a, b, 61, rng.choice(alpha)])
            cases.append([61, a, b, 61])
            cases.append([a, 61, 61, 61])
    prefix = np.frombuffer(b"QUJD", dtype=np.uint8)
    for c in cases:
        check_decode(np.concatenate([prefix, np.array(c, dtype=np.uint8)]))
        check_decode(np.array(c, dtype=np.uint8))


def test_decode_multiple_errors_min_offset():
    rng = np.random.default_rng(110)
    x = splitmix_bytes(110, 0, 600000)
    t = oracle.encode(x)
    for trial in range(30):
        u = t.copy()
        k = int(rng.integers(1, 50))
        pos = rng.choice(u.size, size=k, replace=False)
        u[pos] = np.frombuffer(b"!", dtype=np.uint8)[0]
        check_decode(u)


def test_decode_all_invalid_buffer():
    """Every position invalid: atomic contention on the error key; the answer is 0."""
    t = np.full(8 << 20, ord("!"), dtype=np.uint8)
    st, ep, out = gpu_decode(t)
    assert (st, ep, out.size) == (b64.B64_ERR_INVALID_CHAR, 0, 0)
    t[: 4 << 20] = ord("A")
    st, ep, out = gpu_decode(t)
    assert (st, ep, out.size) == (b64.B64_ERR_INVALID_CHAR, 4 << 20, 3 << 20)
    assert (out == 0).all()


def test_decode_repeated_calls_reset_scratch():
    """The per-stream scratch resets itself: an error call followed by clean calls."""
    x = splitmix_bytes(111, 0, 5000)
    t = oracle.encode(x)
    u = t.copy()
    u[100] = 0
    for _ in range(3):
        check_decode(u)
        check_decode(t)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        check_decode(u)
    check_decode(t)


def test_decode_async_result_record():
    x = splitmix_bytes(112, 0, 100001)
    t = oracle.encode(x)
    t[77777] = ord("*")
    d = to_dev(t)
    out = torch.empty(b64.b64_decoded_max_len(t.size), dtype=torch.uint8, device=DEV)
    res = b64.result_tensor(DEV)
    b64.b64_decode_async(d, out, res)
    out_len, err_pos, st, pc = b64.unpack_result(res)
    assert (st, err_pos, out_len) == (b64.B64_ERR_INVALID_CHAR, 77777, 3 * (77777 // 4))
    t[77777] = oracle.encode(x)[77777]
    b64.b64_decode_async(to_dev(t), out, res)
    out_len, err_pos, st, pc = b64.unpack_result(res)
    assert (st, err_pos, out_len, pc) == (b64.B64_OK, -1, 100001, 1)
    assert np.array_equal(host(out[:out_len]), x)


# --------------------------------------------------------------- shards

def emulate_sharded_decode(t, world, flags=0, mis=None, rng=None):
    """Single-GPU emulation of the sharded decode (ranks run sequentially,
    no collectives): every shard decode writes its exchange record (key,
    out_len); MIN of the keys + the gathered lengths go through BOTH the
    device combine (b64_combine_shards_async) and the host one, which must
    agree.  Returns (status, err_pos, out_len, shard outputs)."""
    keys, lens, outs = [], [], []
    for r in range(world):
        bgn, end = b64.b64_shard(t.size, 4, world, r)
        mi = int(rng.integers(0, 16)) if rng is not None else (mis or 0)
        d = to_dev(t[bgn:end], mi)
        cap = b64.b64_decoded_max_len_ex(end - bgn, flags)
        out = torch.empty(max(cap, 1), dtype=torch.uint8, device=DEV)
        res = b64.result_tensor(DEV)
        key = torch.empty(2, dtype=torch.int64, device=DEV)
        b64.b64_decode_shard_ex_async(d, out, res, bgn, final_shard=(r == world - 1), flags=flags, key=key)
        ol, ep, st, _ = b64.unpack_result(res)
        k = host(key).tolist()
        assert k == [b64.b64_shard_key(st, ep, bgn), ol]
        keys.append(k[0])
        lens.append(ol)
        outs.append(host(out[:ol]))
    kmin = torch.tensor([min(keys)], dtype=torch.int64, device=DEV)
    dres = b64.result_tensor(DEV)
    b64.b64_combine_shards_async(kmin, torch.tensor(lens, dtype=torch.int64, device=DEV), t.size, dres)
    ol, ep, st, pc = b64.unpack_result(dres)
    assert (st, ep, ol, pc) == b64.b64_combine_shards(min(keys), lens, t.size)
    return st, ep, ol, outs


def test_shard_decode_matches_whole_buffer():
    """Split a buffer on 4-char boundaries; non-final shards reject '=' and
    skip the final-quad rule; the combined result equals the whole-buffer
    oracle decode under all 8 flag combinations (the single-GPU emulation of
    the sharded run)."""
    for flags in range(8):
        x = splitmix_bytes(113, 0, 250001)
        t0 = oracle.encode_ex(x, flags)
        variants = [t0, t0[:-1], t0[:-2], t0.copy(), t0.copy(), t0.copy()]
        variants[3][200000] = ord("=")
        variants[4][50] = 0x80
        variants[5][-3:] = np.frombuffer(b"Zh=", np.uint8) if t0.size % 4 == 0 else variants[5][-3:]
        for t in variants:
            for world in (1, 2, 3, 8):
                st, ep, ol, outs = emulate_sharded_decode(t, world, flags)
                rst, rep, rout = oracle.decode_ex(t, flags)
                assert (st, ep, ol) == (rst, rep, rout.size), (flags, world, st, ep, rst, rep)
                assert np.array_equal(np.concatenate(outs)[:ol], rout)


def test_nonfinal_shard_rejects_padding():
    t = np.frombuffer(b"QUJDRA==", dtype=np.uint8).copy()
    d = to_dev(t)
    out = torch.empty(6, dtype=torch.uint8, device=DEV)
    res = b64.result_tensor(DEV)
    b64.b64_decode_shard_async(d, out, res, final_shard=False)
    ol, ep, st, _ = b64.unpack_result(res)
    assert (st, ep, ol) == (b64.B64_ERR_INVALID_CHAR, 6, 3)
    with pytest.raises(b64.B64Error):
        b64.b64_decode_shard_async(to_dev(t[:7]), out, res, final_shard=False)


# -------------------------------------------------------------- batched

def _batch_case(lens, seed, in_mis=0, start=0):
    tot = int(np.sum(lens)) + start
    raw = splitmix_bytes(seed, 0, tot)
    off = np.zeros(len(lens) + 1, dtype=np.int64)
    off[0] = start
    off[1:] = start + np.cumsum(lens)
    return raw, off


def check_encode_batch(raw, off, in_mis=0):
    d = to_dev(raw, in_mis)
    doff = torch.from_numpy(off).to(DEV)
    out, out_off = b64.b64_encode_batch(d, doff)
    torch.cuda.synchronize()
    oo = host(out_off)
    o = host(out)
    assert oo[0] == 0
    for i in range(off.size - 1):
        ref = oracle.encode(raw[off[i]: off[i + 1]])
        assert oo[i + 1] - oo[i] == ref.size, i
        assert np.array_equal(o[oo[i]: oo[i + 1]], ref), i
    return o[: oo[-1]], oo


def check_decode_batch(text, off, in_mis=0):
    d = to_dev(text, in_mis)
    doff = torch.from_numpy(off).to(DEV)
    out, out_off, out_len, err_pos, status = b64.b64_decode_batch(d, doff)
    torch.cuda.synchronize()
    oo, ol, ep, st, o = host(out_off), host(out_len), host(err_pos), host(status), host(out)
    for i in range(off.size - 1):
        rst, rep, rout = oracle.decode(text[off[i]: off[i + 1]])
        assert (st[i], ep[i], ol[i]) == (rst, rep, rout.size), (i, st[i], ep[i], ol[i], rst, rep)
        assert np.array_equal(o[oo[i]: oo[i] + ol[i]], rout), i
        if rst == oracle.OK:
            assert oo[i + 1] - oo[i] == rout.size


def test_batch_encode_decode_ragged():
    rng = np.random.default_rng(114)
    # batched units: 2304 input bytes / 3072 chars (6 passes of one warp)
    lens = np.concatenate([np.arange(0, 70), rng.integers(0, 30000, 200),
                           [2303, 2304, 2305, 4608, 4609, 6144, 6145, 6912, 12288, 65536]])
    rng.shuffle(lens)
    for start, mis in ((0, 0), (5, 3), (1, 0)):
        raw, off = _batch_case(lens, 114, start=start)
        text, toff = check_encode_batch(raw, off, mis)
        check_decode_batch(text, toff.astype(np.int64), mis)


def test_batch_decode_with_errors_and_lengths():
    rng = np.random.default_rng(115)
    lens = rng.integers(0, 20000, 400)
    raw, off = _batch_case(lens, 115)
    texts = [oracle.encode(raw[off[i]: off[i + 1]]) for i in range(lens.size)]
    for i in range(0, lens.size, 7):      # corrupt some messages
        if texts[i].size:
            texts[i][int(rng.integers(0, texts[i].size))] = int(rng.integers(0, 256))
    for i in range(3, lens.size, 11):     # truncate some (LENGTH / partial quads)
        texts[i] = texts[i][: max(0, texts[i].size - int(rng.integers(1, 4)))]
    for i in range(5, lens.size, 13):     # misplaced pads
        if texts[i].size >= 8:
            texts[i][texts[i].size - 6] = ord("=")
    toff = np.zeros(lens.size + 1, dtype=np.int64)
    toff[1:] = np.cumsum([t.size for t in texts])
    check_decode_batch(np.concatenate(texts), toff)


def test_batch_all_final_quads():
    """All 64^2 'xx==' and 64^3 'xxx=' final quads (non-canonical trailing
    bits accepted) plus misplaced-pad quads, each as a 4-char message."""
    alpha = np.frombuffer(ALPHABET, dtype=np.uint8)
    i2 = np.indices((64, 64)).reshape(2, -1).T
    q2 = np.stack([alpha[i2[:, 0]], alpha[i2[:, 1]], np.full(i2.shape[0], 61, np.uint8),
                   np.full(i2.shape[0], 61, np.uint8)], axis=1)
    i3 = np.indices((64, 64, 64)).reshape(3, -1).T
    q3 = np.stack([alpha[i3[:, 0]], alpha[i3[:, 1]], alpha[i3[:, 2]],
                   np.full(i3.shape[0], 61, np.uint8)], axis=1)
    bad = np.stack([alpha[i2[:, 0]], alpha[i2[:, 1]], np.full(i2.shape[0], 61, np.uint8),
                    alpha[i2[:, 1]]], axis=1)
    quads = np.concatenate([q2, q3, bad]).astype(np.uint8)
    text = quads.ravel()
    off = np.arange(0, text.size + 1, 4, dtype=np.int64)
    d = to_dev(text)
    out, out_off, out_len, err_pos, status = b64.b64_decode_batch(d, torch.from_numpy(off).to(DEV))
    st, ep, ol, oo, o = host(status), host(err_pos), host(out_len), host(out_off), host(out)
    nq2, nq3 = q2.shape[0], q3.shape[0]
    for i in range(quads.shape[0]):
        rst, rep, rout = oracle.decode(quads[i])
        assert (st[i], ep[i], ol[i]) == (rst, rep, rout.size), i
        assert np.array_equal(o[oo[i]: oo[i] + ol[i]], rout), i
    # closed form for every message: xx== -> 1 byte = a*4 + b/16, xxx= -> 2 bytes
    a2, b2 = i2[:, 0], i2[:, 1]
    assert (st[:nq2] == 0).all() and (ol[:nq2] == 1).all()
    assert np.array_equal(o[oo[:nq2]], ((a2 * 4 + b2 // 16) & 255).astype(np.uint8))
    a3, b3, c3 = i3[:, 0], i3[:, 1], i3[:, 2]
    s3 = slice(nq2, nq2 + nq3)
    assert (st[s3] == 0).all() and (ol[s3] == 2).all()
    assert np.array_equal(o[oo[s3]], ((a3 * 4 + b3 // 16) & 255).astype(np.uint8))
    assert np.array_equal(o[oo[s3] + 1], (((b3 * 16) & 255) + c3 // 4).astype(np.uint8))
    sb = slice(nq2 + nq3, None)
    assert (st[sb] == 1).all() and (ep[sb] == 3).all()


def test_batch_messages_spanning_many_ctas():
    """Messages far larger than one CTA's share of the batch (their units run
    in many CTAs' ranges, the decode result waits for all of them), next to
    tiny and empty ones, with in_off[0] > 0; errors in the first, a middle
    and the last unit of the large messages."""
    lens = np.array([5, 0, 40_000_003, 3, 1, 0, 7_000_000, 2, 9_999_999, 0], dtype=np.int64)
    raw, off = _batch_case(lens, 118, start=7)
    text, toff = check_encode_batch(raw, off)
    toff = toff.astype(np.int64)
    check_decode_batch(text, toff)
    bad = text.copy()
    for i, frac in ((2, 0.0), (2, 0.5), (2, 0.9999999), (6, 0.999), (8, 0.3)):
        a, b = int(toff[i]), int(toff[i + 1])
        bad[a + int((b - a - 1) * frac)] = ord("*")
    check_decode_batch(bad, toff)
    # one message only: every CTA works on it, the owner finishes it
    raw1, off1 = _batch_case(np.array([64 << 20], dtype=np.int64), 119)
    t1, to1 = check_encode_batch(raw1, off1)
    t1 = t1.copy()
    t1[-5] = ord("#")
    check_decode_batch(t1, to1.astype(np.int64))


def test_batch_empty_and_zero_messages():
    raw, off = _batch_case(np.array([0, 0, 5, 0], dtype=np.int64), 116)
    check_encode_batch(raw, off)
    check_decode_batch(np.frombuffer(b"QUJDQUJD", dtype=np.uint8).copy(), np.array([0, 0, 8, 8], dtype=np.int64))
    # k = 0
    d = to_dev(np.zeros(4, dtype=np.uint8))
    out, out_off = b64.b64_encode_batch(d, torch.zeros(1, dtype=torch.int64, device=DEV))
    assert host(out_off).tolist() == [0]


def test_host_buffer_api():
    x = splitmix_bytes(117, 0, 123457)
    hx = torch.from_numpy(x).pin_memory()
    ht = torch.empty(b64.b64_encoded_len(x.size), dtype=torch.uint8).pin_memory()
    si = torch.empty(ht.numel(), dtype=torch.uint8, device=DEV)
    so = torch.empty(ht.numel(), dtype=torch.uint8, device=DEV)
    n = b64.b64_encode_host(hx, ht, si, so)
    assert n == ht.numel() and np.array_equal(ht.numpy(), oracle.encode(x))
    hy = torch.empty(b64.b64_decoded_max_len(n), dtype=torch.uint8).pin_memory()
    st, ol, ep = b64.b64_decode_host(ht, hy, so, si)
    assert (st, ep, ol) == (0, -1, x.size) and np.array_equal(hy.numpy()[:ol], x)


def test_host_buffer_api_multichunk():
    """Host pipeline over several 24 MiB / 32 MiB chunks: round trip, an
    error in a middle chunk, '=' at a chunk seam, LENGTH on the last chunk."""
    from tests import oracle_par

    n = 150_000_001
    x = splitmix_bytes(118, 0, n)
    hx = torch.from_numpy(x).pin_memory()
    m = b64.b64_encoded_len(n)
    ht = torch.empty(m, dtype=torch.uint8).pin_memory()
    si = torch.empty(m, dtype=torch.uint8, device=DEV)
    so = torch.empty(m, dtype=torch.uint8, device=DEV)
    assert b64.b64_encode_host(hx, ht, si, so) == m
    ref = oracle_par.encode(x)
    assert np.array_equal(ht.numpy(), ref)
    hy = torch.empty(b64.b64_decoded_max_len(m), dtype=torch.uint8).pin_memory()
    st, ol, ep = b64.b64_decode_host(ht, hy, si, so)
    assert (st, ol, ep) == (0, n, -1) and np.array_equal(hy.numpy()[:n], x)
    for pos, byte, cut in [(70_000_123, 0x21, 0), ((64 << 20) - 1, ord("="), 0), (0, None, 3)]:
        t = ref.copy()
        if byte is not None:
            t[pos] = byte
        if cut:
            t = t[:-cut]
        ht2 = torch.from_numpy(t).pin_memory()
        st, ol, ep = b64.b64_decode_host(ht2, hy, si, so)
        rst, rep, rout = oracle_par.decode(t)
        assert (st, ep, ol) == (rst, rep, rout.size), (pos, st, ep, ol, rst, rep)
        assert np.array_equal(hy.numpy()[:ol], rout)


def test_host_api_respects_stream_order():
    """the host-buffer pipeline's internal copy streams wait for
    the work already queued on the caller's stream.  An async encode that
    reads X, queued behind a long sleep, must not see the host call's H2D
    copy overwrite X (X is reused as the host call's d_scratch_in)."""
    s = torch.cuda.Stream()
    x1 = splitmix_bytes(119, 0, 3 << 20)
    x2 = splitmix_bytes(120, 0, 3 << 20)
    X = torch.from_numpy(x1).to(DEV)
    out1 = torch.empty(b64.b64_encoded_len(x1.size), dtype=torch.uint8, device=DEV)
    so = torch.empty_like(out1)
    hx = torch.from_numpy(x2).pin_memory()
    ht = torch.empty(out1.numel(), dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)                    # ~25 ms of GPU time
        b64.b64_encode(X, out=out1, stream=s)            # reads X (x1)
        b64.b64_encode_host(hx, ht, X, so, stream=s)     # overwrites X with x2
    torch.cuda.synchronize()
    assert np.array_equal(host(out1), oracle.encode(x1))
    assert np.array_equal(ht.numpy(), oracle.encode(x2))


def test_host_api_flags_roundtrip():
    """b64_encode_host_ex / b64_decode_host_ex: every flag set, multichunk
    sizes, against oracle.encode_ex / decode_ex."""
    for flags in range(8):
        for n in (0, 1, 2, 100, 25_165_826):
            x = splitmix_bytes(121 + flags, 0, n)
            m = b64.b64_encoded_len_ex(n, flags)
            hx = torch.from_numpy(x).pin_memory()
            ht = torch.empty(max(m, 1), dtype=torch.uint8).pin_memory()
            si = torch.empty(max(m, 1), dtype=torch.uint8, device=DEV)
            so = torch.empty(max(m, 1), dtype=torch.uint8, device=DEV)
            assert b64.b64_encode_host(hx, ht[:m], si, so, flags=flags) == m
            ref = oracle.encode_ex(x, flags)
            assert np.array_equal(ht[:m].numpy(), ref), (flags, n)
            for c in (ref, ref[:-1]):
                hc = torch.from_numpy(c.copy()).pin_memory()
                hy = torch.empty(max(b64.b64_decoded_max_len_ex(c.size, flags), 1), dtype=torch.uint8).pin_memory()
                st, ol, ep = b64.b64_decode_host(hc, hy, si, so, flags=flags)
                rst, rep, rout = oracle.decode_ex(c, flags)
                assert (st, ep, ol) == (rst, rep, rout.size), (flags, n, c.size)
                assert np.array_equal(hy.numpy()[:ol], rout)
