"""f3 / f4 at sizes past 2^32 (64-bit offsets in every index path): 3.8 GB of
seeded bytes -> line-wrapped encode (76 + CRLF, 5.2 GB of text) ->
whitespace-tolerant decode back, and despace of the same text -- each
compared in full with the CPU oracle (streamed in chunks of whole lines);
despace's general path on the same text made irregular; error offsets
beyond 2^32 are exact."""
import numpy as np
import pytest
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes
from inputs.gpu_gen import fill
from tests import oracle_par
from tests.gpu_util import DEV, host

pytestmark = pytest.mark.gpu
SEED = 96
LINES = 1 << 26          # 67,108,864 lines of 76 chars
N = 57 * LINES - 2        # raw bytes (n mod 3 = 1: the last line ends "==")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    free, _ = torch.cuda.mem_get_info()
    if free < 30 << 30:
        pytest.skip("needs ~30 GB of free device memory")
    b64.load_library()


CH_LINES = 1 << 23        # lines per oracle chunk (478 MB raw, 654 MB of text)


def test_mime_past_4gib():
    """Full-length oracle parity past 2^32: the wrapped encoding, the
    whitespace-tolerant decoding and the despaced text are each streamed back
    in chunks of whole lines and compared with the oracle (R-wrap,
    R-ws-decode, App. B) run on all host cores on the same seeded bytes."""
    raw = torch.empty(N, dtype=torch.uint8, device=DEV)
    fill(raw, SEED)
    m = b64.b64_encoded_len_wrapped(N, 76, True)
    assert m > 1 << 32
    w = b64.b64_encode_wrapped(raw, line_chars=76, crlf=True)
    assert w.numel() == m
    y, st, ep = b64.b64_decode_ws(w)
    assert (st, ep) == (b64.B64_OK, -1) and y.numel() == N
    d, dlen = b64.b64_despace(w)
    dl = int(dlen.item())
    pw = torch.empty(78 * CH_LINES, dtype=torch.uint8).pin_memory()
    py = torch.empty(57 * CH_LINES, dtype=torch.uint8).pin_memory()
    pd = torch.empty(76 * CH_LINES, dtype=torch.uint8).pin_memory()
    seen_w = seen_y = seen_d = 0
    for L0 in range(0, LINES, CH_LINES):
        L1 = min(L0 + CH_LINES, LINES)
        b0, b1 = 57 * L0, min(57 * L1, N)
        xs = oracle_par.gen(SEED, b0, b1)
        ref_w = oracle_par.encode_wrapped(xs, 76, True)
        pw[: ref_w.size].copy_(w[78 * L0: 78 * L0 + ref_w.size])
        assert np.array_equal(pw[: ref_w.size].numpy(), ref_w), ("wrapped", L0)
        rst, rep, ref_y = oracle_par.decode_ws_lines(ref_w, 78)
        assert (rst, rep) == (oracle.OK, -1) and ref_y.size == b1 - b0
        py[: ref_y.size].copy_(y[b0: b1])
        assert np.array_equal(py[: ref_y.size].numpy(), ref_y), ("decode_ws", L0)
        ref_d = oracle_par.despace(ref_w)
        pd[: ref_d.size].copy_(d[76 * L0: 76 * L0 + ref_d.size])
        assert np.array_equal(pd[: ref_d.size].numpy(), ref_d), ("despace", L0)
        seen_w += ref_w.size
        seen_y += ref_y.size
        seen_d += ref_d.size
    assert (seen_w, seen_y, seen_d) == (m, N, dl)
    # the same text with one CR past 2^32 turned into ' ' (still App. B
    # white space, so the despaced text is unchanged) is no longer line-
    # structured: despace takes its general two-pass path, whose result must
    # equal the (oracle-checked) fast-path result
    del y
    cr = 78 * ((1 << 32) // 78 + 7) + 76
    assert int(w[cr].item()) == 13
    w[cr] = ord(" ")
    ws = torch.empty(b64.load_library().b64_despace_workspace_bytes(m), dtype=torch.uint8, device=DEV)
    d2 = torch.empty(m, dtype=torch.uint8, device=DEV)
    _, dlen2 = b64.b64_despace(w, out=d2, ws=ws)
    assert int(ws[:4].view(torch.int32).item()) == 0  # WlState.verdict: general path
    assert int(dlen2.item()) == dl and torch.equal(d2[:dl], d[:dl])
    w[cr] = 13
    del d, d2, ws
    # exact first-error offsets past 2^32 (line structure: byte 78k+j, j < 76),
    # against the oracle on the text from a line boundary before the error
    for pos in [(1 << 32) + 78 * 5 + 3, m - 200]:
        old = int(w[pos].item())
        w[pos] = ord("!")
        _, st, ep = b64.b64_decode_ws(w)
        a = 78 * (pos // 78 - 10)
        rst, rep, _ = oracle_par.decode_ws_lines(host(w[a:]), 78)
        assert (st, ep) == (rst, a + rep) == (b64.B64_ERR_INVALID_CHAR, pos), pos
        w[pos] = old
