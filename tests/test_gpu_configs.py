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


@pytest.mark.slow
def test_c5_32gib_sampled_and_sharded():
    """32 GiB on one GPU (the G=1 point of config 5): sampled windows vs the
    oracle, GPU round trip, 8-way shard emulation, one corruption in the last
    shard."""
    from inputs.gpu_gen import fill
    from paper_1704_00605_b200.dist import INT64_MAX, global_decode_result

    free, _ = torch.cuda.mem_get_info()
    n = W.C5_N
    m = b64.b64_encoded_len(n)
    if free < n + m + n + (2 << 30):
        pytest.skip(f"needs {(2 * n + m) / 2**30:.0f} GiB of device memory")
    x = torch.empty(n, dtype=torch.uint8, device=DEV)
    fill(x, W.C5_SEED)
    # the CUDA generator equals the numpy twin on samples (incl. offsets > 2^32)
    for o in (0, (1 << 32) + 5, n - 1000):
        assert np.array_equal(host(x[o: o + 1000]), splitmix_bytes(W.C5_SEED, o, o + 1000))
    t = torch.empty(m, dtype=torch.uint8, device=DEV)
    b64.b64_encode(x, out=t)
    rng = np.random.default_rng(55)
    groups = n // 3
    windows = [0, groups - 100_000] + [int(g) for g in rng.integers(0, groups - 100_000, 24)]
    for g in windows:
        o = 3 * g
        L = min(3 * 100_000, n - o)
        exp = oracle.encode(splitmix_bytes(W.C5_SEED, o, o + L))
        assert np.array_equal(host(t[4 * g: 4 * g + exp.size]), exp), g
    # tail: n mod 3 = 2 -> one '='
    tail = oracle.encode(splitmix_bytes(W.C5_SEED, n - 5, n))
    assert np.array_equal(host(t[m - 8:]), tail[-8:])
    y = torch.empty(b64.b64_decoded_max_len(m), dtype=torch.uint8, device=DEV)
    yv, st, ep = b64.b64_decode(t, out=y)
    assert (st, ep, yv.numel()) == (b64.B64_OK, -1, n)
    assert torch.equal(yv, x)
    # 8-way shard emulation (sequential on one GPU; no collectives)
    for dirty_at in (None, m - 12345):
        if dirty_at is not None:
            t[dirty_at] = 0x21
        errs, lens = [], []
        for r in range(8):
            bgn, end = b64.b64_shard(m, 4, 8, r)
            res = b64.result_tensor(DEV)
            b64.b64_decode_shard_async(t[bgn:end], y[3 * (bgn // 4):], res, final_shard=(r == 7))
            ol, e, s, _ = b64.unpack_result(res)
            errs.append(bgn + e if e >= 0 else INT64_MAX)
            lens.append(ol)
        st, ep, ol = global_decode_result(min(errs), m, lens)
        if dirty_at is None:
            assert (st, ep, ol) == (b64.B64_OK, -1, n)
            assert torch.equal(y[:n], x)
        else:
            assert (st, ep, ol) == (b64.B64_ERR_INVALID_CHAR, dirty_at, 3 * (dirty_at // 4))
