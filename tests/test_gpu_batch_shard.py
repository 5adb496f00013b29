"""Batch sharding by message on one GPU: each of G = 1, 2,
3, 8 emulated ranks runs the batched kernels on its b64_batch_shard slice
(the offsets passed as a view into the full offsets array), and the
per-rank results -- output placed at the rank's global output base,
per-message decode results -- reproduce the whole-batch oracle."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs import workloads as W
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def test_sharded_batches_match_whole_batch():
    lens, rng = W.c2_lengths(k=2000, seed=94)
    off = W.offsets_from_lengths(lens)
    raw = splitmix_bytes(95, 0, int(off[-1]))
    encs = [oracle.encode(raw[off[i]:off[i + 1]]) for i in range(lens.size)]
    text = np.concatenate(encs)
    toff = np.concatenate([[0], np.cumsum([e.size for e in encs])]).astype(np.int64)
    bad = rng.choice(lens.size, 20, replace=False)
    for i in bad:
        text[int(rng.integers(toff[i], toff[i + 1]))] = 0x80
    ref = [oracle.decode(text[toff[i]:toff[i + 1]]) for i in range(lens.size)]
    d_raw = torch.from_numpy(raw).to(DEV)
    d_off = torch.from_numpy(off).to(DEV)
    d_text = torch.from_numpy(text).to(DEV)
    d_toff = torch.from_numpy(toff).to(DEV)
    for G in (1, 2, 3, 8):
        enc_out = np.zeros(toff[-1], dtype=np.uint8)
        base = 0
        st_all, ep_all, ol_all = [], [], []
        for r in range(G):
            i0, i1 = b64.b64_batch_shard(off, G, r)
            if i1 > i0:
                out, oo = b64.b64_encode_batch(d_raw, d_off[i0:i1 + 1], total_in=int(off[i1] - off[i0]))
                n = int(oo[-1].item())
                enc_out[base:base + n] = host(out[:n])
                base += n
            j0, j1 = b64.b64_batch_shard(toff, G, r)
            if j1 > j0:
                _, _, ol, ep, st = b64.b64_decode_batch(d_text, d_toff[j0:j1 + 1],
                                                        total_in=int(toff[j1] - toff[j0]))
                st_all += host(st).tolist()
                ep_all += host(ep).tolist()
                ol_all += host(ol).tolist()
        assert base == toff[-1] and np.array_equal(enc_out, np.concatenate(encs)), G
        assert st_all == [x[0] for x in ref], G
        assert ep_all == [x[1] for x in ref], G
        assert ol_all == [x[2].size for x in ref], G
