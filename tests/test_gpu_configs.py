"""Config-size parity (BASELINE.json configs C1-C5) at full size, in the
launch configuration bench.py times: GPU output bytes, lengths, status and
first-error offset equal the CPU oracle's on the same seeded inputs.  C5
(32 GiB) is checked on sampled windows the oracle can compute one by one plus
properties that hold at any size (round trip, shard emulation)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs import workloads as W
from inputs.gen import splitmix_bytes
from tests import oracle_par
from tests.gpu_util import DEV, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def dev(x):
    return torch.from_numpy(x).to(DEV)


def test_c1_roundtrip_and_corrupted_copy():
    x = splitmix_bytes(W.C1_SEED, 0, W.C1_N)
    ref = oracle.encode(x)
    assert ref.size == 1_398_104 and bytes(ref[-2:]) == b"=="
    t = b64.b64_encode(dev(x))
    assert np.array_equal(host(t), ref)
    y, st, ep = b64.b64_decode(dev(ref))
    assert (st, ep) == (b64.B64_OK, -1) and np.array_equal(host(y), x)
    pos, byte = W.c1_corruption(ref.size)
    u = ref.copy()
    u[pos] = byte
    y, st, ep = b64.b64_decode(dev(u))
    rst, rep, rout = oracle.decode(u)
    assert (st, ep) == (rst, rep) == (b64.B64_ERR_INVALID_CHAR, pos)
    assert np.array_equal(host(y), rout)


def _c2():
    lens, rng = W.c2_lengths()
    off = W.offsets_from_lengths(lens)
    raw = splitmix_bytes(W.C2_SEED, 0, int(off[-1]))
    return lens, rng, off, raw


def test_c2_batched_encode_decode():
    lens, rng, off, raw = _c2()
    out, out_off = b64.b64_encode_batch(dev(raw), dev(off))
    o, oo = host(out), host(out_off)
    texts = [oracle.encode(raw[off[i]: off[i + 1]]) for i in range(lens.size)]
    tl = np.array([t.size for t in texts], dtype=np.int64)
    assert np.array_equal(np.diff(oo), tl)
    ref_all = np.concatenate(texts)
    assert np.array_equal(o[: oo[-1]], ref_all)
    toff = W.offsets_from_lengths(tl)
    y, y_off, y_len, y_err, y_st = b64.b64_decode_batch(dev(ref_all), dev(toff))
    assert (host(y_st) == 0).all() and (host(y_err) == -1).all()
    assert np.array_equal(host(y_len), lens)
    assert np.array_equal(host(y_off), off - off[0])
    assert np.array_equal(host(y)[: off[-1]], raw)

    # extra (not a config): 1% of messages carry one NA191 byte
    inj = W.c2_injections(tl, rng)
    dirty = ref_all.copy()
    for i, p, b in inj:
        dirty[toff[i] + p] = b
    y, y_off, y_len, y_err, y_st = b64.b64_decode_batch(dev(dirty), dev(toff))
    st, ep, ol, oo, yo = host(y_st), host(y_err), host(y_len), host(y_off), host(y)
    bad = {i for i, _, _ in inj}
    for i in range(lens.size):
        if i in bad or i % 50 == 0:
            rst, rep, rout = oracle.decode(dirty[toff[i]: toff[i + 1]])
            assert (st[i], ep[i], ol[i]) == (rst, rep, rout.size), i
            assert np.array_equal(yo[oo[i]: oo[i] + ol[i]], rout)
        else:
            assert st[i] == 0 and ol[i] == lens[i]
    assert sorted(int(i) for i in np.nonzero(st)[0]) == sorted(bad)


def test_c3_large_buffer_both_directions():
    x = splitmix_bytes(W.C3_SEED, 0, W.C3_N)
    ref = oracle_par.encode(x)
    assert ref.size == 1_431_655_768
    dx = dev(x)
    t = b64.b64_encode(dx)
    assert torch.equal(t.cpu(), torch.from_numpy(ref))
    del dx
    y, st, ep = b64.b64_decode(t)
    rst, rep, rout = oracle_par.decode(ref)
    assert (st, ep) == (rst, rep) == (b64.B64_OK, -1)
    assert torch.equal(y.cpu(), torch.from_numpy(rout))
    assert np.array_equal(rout, x)


def test_c4_decode_validation_stress():
    x = splitmix_bytes(W.C4_SEED, 0, W.C4_RAW)
    text = oracle_par.encode(x)
    assert text.size == W.C4_M
    y, st, ep = b64.b64_decode(dev(text))
    assert (st, ep) == (b64.B64_OK, -1) and torch.equal(y.cpu(), torch.from_numpy(x))
    pos, byt = W.c4_corruptions()
    dirty = text.copy()
    dirty[pos] = byt
    y, st, ep = b64.b64_decode(dev(dirty))
    rst, rep, rout = oracle_par.decode(dirty)
    assert (st, ep) == (rst, rep) == (b64.B64_ERR_INVALID_CHAR, int(pos.min()))
    assert np.array_equal(host(y), rout)


CHUNK = 3 * (256 << 20)   # 768 MiB of raw bytes (1 GiB of text) per oracle chunk


@pytest.mark.slow
def test_c5_32gib_full_oracle_parity_and_sharded():
    """32 GiB on one GPU (the G=1 point of config 5), compared with the CPU
    oracle IN FULL: the GPU encoding of all 2^35 bytes and the GPU decoding
    of all 45.8 G characters are streamed back in 768 MiB / 1 GiB chunks and
    compared with the oracle (Alg 1 / Alg 2) run on all host
    cores on the same seeded bytes.  Then the 8-way shard emulation with the
    exchange records, clean and with one corruption in the last shard."""
    from inputs.gpu_gen import fill

    free, _ = torch.cuda.mem_get_info()
    n = W.C5_N
    m = b64.b64_encoded_len(n)
    if free < n + m + n + (2 << 30):
        pytest.skip(f"needs {(2 * n + m) / 2**30:.0f} GiB of device memory")
    x = torch.empty(n, dtype=torch.uint8, device=DEV)
    fill(x, W.C5_SEED)
    t = torch.empty(m, dtype=torch.uint8, device=DEV)
    b64.b64_encode(x, out=t)
    y = torch.empty(b64.b64_decoded_max_len(m), dtype=torch.uint8, device=DEV)
    yv, st, ep = b64.b64_decode(t, out=y)
    assert (st, ep, yv.numel()) == (b64.B64_OK, -1, n)
    # whole-buffer oracle parity, chunk by chunk (chunks of whole groups /
    # quads; only the last chunk holds the '=' tail: n mod 3 = 2)
    pinned_t = torch.empty(4 * CHUNK // 3, dtype=torch.uint8).pin_memory()
    pinned_y = torch.empty(CHUNK, dtype=torch.uint8).pin_memory()
    checked_in = checked_out = 0
    for o in range(0, n, CHUNK):
        L = min(CHUNK, n - o)
        xs = oracle_par.gen(W.C5_SEED, o, o + L)
        ref = oracle_par.encode(xs)                       # Alg 1 on the chunk
        tv = pinned_t[: ref.size]
        tv.copy_(t[4 * (o // 3): 4 * (o // 3) + ref.size])
        assert np.array_equal(tv.numpy(), ref), ("encode chunk", o)
        rst, rep, rout = oracle_par.decode(ref)          # Alg 2 on the same text
        assert (rst, rep) == (oracle.OK, -1) and rout.size == L
        yh = pinned_y[:L]
        yh.copy_(y[o: o + L])
        assert np.array_equal(yh.numpy(), rout), ("decode chunk", o)
        checked_in += L
        checked_out += ref.size
    assert (checked_in, checked_out) == (n, m)
    assert bytes(pinned_t[ref.size - 2: ref.size].numpy()) != b"==" and pinned_t[ref.size - 1] == ord("=")
    # the CUDA generator equals the numpy twin (incl. offsets > 2^32)
    for o in (0, (1 << 32) + 5, n - 1000):
        assert np.array_equal(host(x[o: o + 1000]), splitmix_bytes(W.C5_SEED, o, o + 1000))
    del x
    # 8-way shard emulation (sequential on one GPU; no collectives): each
    # shard decode writes its exchange record, combined on the device
    for dirty_at in (None, m - 12345):
        if dirty_at is not None:
            t[dirty_at] = 0x21
        keys = torch.empty(8, 2, dtype=torch.int64, device=DEV)
        for r in range(8):
            bgn, end = b64.b64_shard(m, 4, 8, r)
            res = b64.result_tensor(DEV)
            b64.b64_decode_shard_ex_async(t[bgn:end], y[3 * (bgn // 4):], res, bgn, final_shard=(r == 7),
                                          key=keys[r])
        kmin = keys[:, 0].min().reshape(1).contiguous()
        out = b64.result_tensor(DEV)
        b64.b64_combine_shards_async(kmin, keys[:, 1].contiguous(), m, out)
        ol, ep, st, _ = b64.unpack_result(out)
        if dirty_at is None:
            assert (st, ep, ol) == (b64.B64_OK, -1, n)
        else:
            # the oracle on the dirty last quads: the error is the only one
            tail = host(t[dirty_at - 4 * 1000: m])
            rst, rep, _ = oracle.decode(tail)
            assert (st, ep, ol) == (rst, dirty_at - 4 * 1000 + rep, 3 * (dirty_at // 4))
            assert st == b64.B64_ERR_INVALID_CHAR and ep == dirty_at
