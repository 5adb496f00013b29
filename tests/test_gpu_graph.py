"""The asynchronous entry points are CUDA-graph capturable (no host syncs,
no allocation, self-resetting scratch): a captured encode -> validating
decode round trip (single buffer, batched, whitespace-tolerant) replays
correctly, including after the input is rewritten in place."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from tests.gpu_util import DEV, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    b64.load_library()


def test_graph_replay_single_buffer_roundtrip():
    n = 1 << 20
    x = torch.from_numpy(splitmix_bytes(600, 0, n)).to(DEV)
    t = torch.empty(b64.b64_encoded_len(n), dtype=torch.uint8, device=DEV)
    y = torch.empty(b64.b64_decoded_max_len(t.numel()), dtype=torch.uint8, device=DEV)
    res = b64.result_tensor(DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm-up (kernel attributes, per-stream scratch)
        b64.b64_encode(x, out=t, stream=s)
        b64.b64_decode_async(t, y, res, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        b64.b64_encode(x, out=t, stream=s)
        b64.b64_decode_async(t, y, res, stream=s)
    for seed in (601, 602, 603):
        x.copy_(torch.from_numpy(splitmix_bytes(seed, 0, n)))
        g.replay()
        torch.cuda.synchronize()
        xs = splitmix_bytes(seed, 0, n)
        assert np.array_equal(host(t), oracle.encode(xs))
        ol, ep, st, _ = b64.unpack_result(res)
        assert (ol, ep, st) == (n, -1, 0) and torch.equal(y[:n], x)


def test_graph_replay_ws_decode_and_batch():
    x = splitmix_bytes(604, 0, 200_000)
    w = torch.from_numpy(oracle.encode_wrapped(x, 76, crlf=True)).to(DEV)
    y = torch.empty(b64.b64_decoded_max_len(w.numel()), dtype=torch.uint8, device=DEV)
    res = b64.result_tensor(DEV)
    ws = torch.empty(b64.b64_decode_ws_workspace_bytes(w.numel()), dtype=torch.uint8, device=DEV)
    lens = np.array([5, 1000, 0, 77777, 3], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    raw = torch.from_numpy(splitmix_bytes(605, 0, int(off[-1]))).to(DEV)
    doff = torch.from_numpy(off).to(DEV)
    bout = torch.empty(4 * int(off[-1]) // 3 + 64, dtype=torch.uint8, device=DEV)
    boff = torch.empty(lens.size + 1, dtype=torch.int64, device=DEV)
    bws = torch.empty(b64.b64_batch_workspace_bytes(lens.size, int(off[-1]), 0) + 256, dtype=torch.uint8,
                      device=DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b64.b64_decode_ws_async(w, y, res, ws=ws, stream=s)
        b64.b64_encode_batch(raw, doff, out=bout, out_off=boff, ws=bws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        b64.b64_decode_ws_async(w, y, res, ws=ws, stream=s)
        b64.b64_encode_batch(raw, doff, out=bout, out_off=boff, ws=bws, stream=s)
    for _ in range(3):
        y.zero_()
        bout.zero_()
        g.replay()
        torch.cuda.synchronize()
        ol, ep, st, _ = b64.unpack_result(res)
        assert (ol, ep, st) == (x.size, -1, 0) and np.array_equal(host(y[:x.size]), x)
        o, oo = host(bout), host(boff)
        rr = host(raw)
        for i in range(lens.size):
            assert np.array_equal(o[oo[i]:oo[i + 1]], oracle.encode(rr[off[i]:off[i + 1]])), i


def test_graphs_with_own_scratch_replay_concurrently():
    """two decode graphs captured on the SAME stream, each with its
    own caller-owned scratch record (b64_decode_scratch_async), replayed at
    the same time on two streams -- one on clean text, one on text with an
    error: each result record is its own input's (the library's per-stream
    scratch would be shared between them)."""
    n = 3 << 20
    x = torch.from_numpy(splitmix_bytes(601, 0, n)).to(DEV)
    t = b64.b64_encode(x)
    td = t.clone()
    td[123_457] = ord("!")
    ya = torch.empty(b64.b64_decoded_max_len(t.numel()), dtype=torch.uint8, device=DEV)
    yb = torch.empty_like(ya)
    ra, rb = b64.result_tensor(DEV), b64.result_tensor(DEV)
    sa, sb = b64.scratch_tensor(DEV), b64.scratch_tensor(DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b64.b64_decode_scratch_async(t, ya, ra, sa, stream=s)
        b64.b64_decode_scratch_async(td, yb, rb, sb, stream=s)
    torch.cuda.synchronize()
    ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(ga, stream=s):
        b64.b64_decode_scratch_async(t, ya, ra, sa, stream=s)
    with torch.cuda.graph(gb, stream=s):
        b64.b64_decode_scratch_async(td, yb, rb, sb, stream=s)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(20):
        ra.zero_()
        rb.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            ga.replay()
        with torch.cuda.stream(s2):
            gb.replay()
        torch.cuda.synchronize()
        assert b64.unpack_result(ra)[:3] == (n, -1, 0)
        assert b64.unpack_result(rb)[:3] == (3 * (123_457 // 4), 123_457, b64.B64_ERR_INVALID_CHAR)
    assert torch.equal(ya[:n], x)
    assert int(sa.abs().sum().item()) == 0 and int(sb.abs().sum().item()) == 0  # left zero
