"""GPU parity of the variant flags: base64url,
unpadded / optional padding, Appendix A strict -- single buffer (every length,
alignments, errors, every final quad) and batched, against oracle.*_ex."""
import itertools
import string

import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, empty_dev, host, to_dev

pytestmark = pytest.mark.gpu

U, NP, ST = b64.B64_FLAG_URL, b64.B64_FLAG_NOPAD, b64.B64_FLAG_STRICT
FLAGS = [U, NP, ST, U | NP, NP | ST, U | NP | ST]
STD = (string.ascii_uppercase + string.ascii_lowercase + string.digits + "+/").encode()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def gpu_dec(t, fl, mis=0):
    d = to_dev(t, mis)
    cap = b64.b64_decoded_max_len_ex(t.size, fl)
    base, out = empty_dev(cap, 0)
    view, st, ep = b64.b64_decode_ex(d, out=out, flags=fl)
    g = host(base)
    assert (g[cap:] == 0xCC).all()
    return st, ep, host(view)


def check(t, fl, mis=0):
    st, ep, out = gpu_dec(t, fl, mis)
    rst, rep, rout = oracle.decode_ex(t, fl)
    assert (st, ep) == (rst, rep), (t.size, fl, st, ep, rst, rep)
    assert np.array_equal(out, rout)


def test_encode_variants_every_length():
    x = splitmix_bytes(201, 0, 40000)
    for fl in (U, NP, U | NP):
        for n in list(range(0, 200)) + [12287, 12288, 12289, 36865, 40000]:
            for om in ((0, 3) if n % 97 == 5 else (0,)):
                base, out = empty_dev(b64.b64_encoded_len_ex(n, fl), om)
                res = b64.b64_encode_ex(to_dev(x[:n]), out=out, flags=fl)
                torch.cuda.synchronize()
                assert np.array_equal(host(res), oracle.encode_ex(x[:n], fl)), (fl, n)
                g = host(base)
                assert (g[:om] == 0xCC).all() and (g[om + out.numel():] == 0xCC).all()


def test_decode_variants_roundtrip_and_errors():
    rng = np.random.default_rng(202)
    x = splitmix_bytes(202, 0, 30000)
    for fl in FLAGS + [0]:
        for n in list(range(0, 120)) + [12288, 12289, 12290, 24577, 30000]:
            t = oracle.encode_ex(x[:n], fl)
            check(t, fl)
            if t.size:
                u = t.copy()
                u[int(rng.integers(0, u.size))] = int(rng.choice([0x21, ord("="), ord("+"), ord("-"), ord("_")]))
                check(u, fl)
                check(t[:-1], fl)
        # padded input in NOPAD mode, url chars in std mode and vice versa
        t = oracle.encode(x[:1001])
        check(t, fl, 5)


def test_decode_variants_all_final_quads():
    """Every 'xx==' / 'xxx=' quad and every 2/3-character tail after a
    prefix, under strict and optional-padding modes."""
    prefix = np.frombuffer(b"QUJD", dtype=np.uint8)
    cases = []
    for a, b in itertools.product(STD[::3], STD):
        cases.append(bytes([a, b]) + b"==")
        cases.append(bytes([a, b]))
        cases.append(bytes([a, b, b]) + b"=")
        cases.append(bytes([a, b, a]))
        cases.append(bytes([a, b]) + b"=")
    for fl in (ST, NP | ST, NP, U | NP | ST):
        for c in cases:
            c = np.frombuffer(c, dtype=np.uint8)
            check(np.concatenate([prefix, c]), fl)


def test_batch_variants():
    rng = np.random.default_rng(203)
    lens = np.concatenate([np.arange(0, 40), rng.integers(0, 9000, 150)])
    off = np.zeros(lens.size + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    raw = splitmix_bytes(203, 0, int(off[-1]))
    for fl in (U, NP, U | NP | ST, ST):
        out, oo = b64.b64_encode_batch(to_dev(raw, 1), torch.from_numpy(off).to(DEV), flags=fl)
        o, oo = host(out), host(oo)
        texts = [oracle.encode_ex(raw[off[i]: off[i + 1]], fl) for i in range(lens.size)]
        for i, t in enumerate(texts):
            assert np.array_equal(o[oo[i]: oo[i + 1]], t), (fl, i)
        for i in range(0, lens.size, 5):
            if texts[i].size:
                texts[i] = texts[i].copy()
                texts[i][int(rng.integers(0, texts[i].size))] = int(rng.choice([0x21, ord("=")]))
        for i in range(2, lens.size, 9):
            texts[i] = texts[i][:-1]
        toff = np.zeros(lens.size + 1, dtype=np.int64)
        toff[1:] = np.cumsum([t.size for t in texts])
        y, yo, yl, ye, ys = b64.b64_decode_batch(to_dev(np.concatenate(texts), 3),
                                                 torch.from_numpy(toff).to(DEV), flags=fl)
        y, yo, yl, ye, ys = host(y), host(yo), host(yl), host(ye), host(ys)
        for i, t in enumerate(texts):
            rst, rep, rout = oracle.decode_ex(t, fl)
            assert (ys[i], ye[i], yl[i]) == (rst, rep, rout.size), (fl, i, ys[i], ye[i], yl[i], rst, rep)
            assert np.array_equal(y[yo[i]: yo[i] + yl[i]], rout), (fl, i)
