"""Multi-process (world size 2, gloo, CPU) test of the sharded-decode result
exchange in paper_1704_00605_b200/dist.py: MIN all-reduce of the shard
reduction key (b64_shard_key: global error offset + status) + all-gather of
shard output lengths, combined by the C ABI's b64_combine_shards, must
reproduce the whole-buffer oracle result under all 8 flag combinations.  Shard-local results come from the oracle
(test infrastructure); on the GPU they come from b64_decode_shard_async."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

WORLD = 2


def _collect(procs, q, timeout):
    """Results of every worker; fails fast if one of them dies."""
    import queue
    import time

    got, t0 = {}, time.time()
    while len(got) < len(procs):
        try:
            r, v = q.get(timeout=1)
            got[r] = v
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead, f"worker died: {dead}"
            assert time.time() - t0 < timeout, "workers timed out"
    return got


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_result(t_local, final, flags):
    """Shard-local (status, err_pos, out_len) with R-shard semantics, via the
    oracle: a non-final shard is decoded with a valid quad appended, so its
    last two positions are not final-quad positions."""
    import oracle

    if final:
        st, ep, out = oracle.decode_ex(t_local, flags)
        return st, ep, out.size
    st, ep, out = oracle.decode_ex(np.concatenate([t_local, np.frombuffer(b"AAAA", np.uint8)]), flags)
    if st != oracle.OK and ep < t_local.size:
        return st, ep, 3 * (ep // 4)
    return oracle.OK, -1, 3 * (t_local.size // 4)


def _worker(rank, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1704_00605_b200 import dist as b64dist
    from paper_1704_00605_b200 import b64_shard, b64_shard_key

    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    res = []
    for t, flags in cases:
        b, e = b64_shard(t.size, 4, WORLD, rank)
        st, ep, ol = _local_result(t[b:e], rank == WORLD - 1, flags)
        res.append(b64dist.combine(b64_shard_key(st, ep, b), ol, t.size, torch.device("cpu")))
    dist.destroy_process_group()
    q.put((rank, res))


def _flag_cases():
    """Whole buffers x all 8 flag combinations (URL, NOPAD, STRICT): clean,
    truncated (LENGTH / unpadded tails), corrupted in either shard, misplaced
    '=', and non-canonical trailing bits (STRICT -> NONCANONICAL)."""
    import oracle
    from inputs.gen import splitmix_bytes

    cases = []
    for flags in range(8):
        for n in (30001, 30002, 30000):
            x = splitmix_bytes(77 + n, 0, n)
            t = oracle.encode_ex(x, flags)
            cases += [(t, flags), (t[:-1], flags), (t[:-3], flags)]
        t = oracle.encode_ex(splitmix_bytes(78, 0, 30001), flags)
        m = t.size
        for pos, b in [(5, 0x21), (m // 2 + 10, 0x21), (m - 5, 0x00), (m // 2, ord("=")),
                       (m // 2 + 3, ord("=")), (m - 1, 0x80), (100, ord("-")), (200, ord("/"))]:
            u = t.copy()
            u[pos] = b
            cases.append((u, flags))
        u = t.copy()
        u[100] = 0x80
        u[m - 100] = 0x80
        cases.append((u, flags))
        # non-canonical final quad: "Zh==" / "Zm9=" tails ("Zg==" / "Zm8=" canonical)
        for tail in (b"Zh==", b"Zm9=", b"Zh", b"Zm9"):
            u = np.concatenate([t[: 4 * (m // 4) - 4], np.frombuffer(tail, np.uint8)])
            cases.append((u, flags))
    return cases


def test_sharded_decode_combine_world2():
    import oracle

    cases = _flag_cases()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, cases, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = _collect(procs, q, 240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    seen = set()
    for i, (c, flags) in enumerate(cases):
        st, ep, out = oracle.decode_ex(c, flags)
        seen.add(st)
        for r in range(WORLD):
            assert got[r][i] == (st, ep, out.size), (i, flags, r, got[r][i], (st, ep, out.size))
    assert seen == {oracle.OK, oracle.INVALID_CHAR, oracle.LENGTH, oracle.NONCANONICAL}


# ------------------------------------------------------- batches (§8(e))

def _batch_worker(rank, port, raw, off, text, toff, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1704_00605_b200 import dist as b64dist

    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    dev = torch.device("cpu")
    # encode: this rank's messages, its output total, the global output base
    i0, i1 = b64dist.shard_messages(off, WORLD, rank)
    enc = [oracle.encode(raw[off[i]:off[i + 1]]) for i in range(i0, i1)]
    base = b64dist.global_out_base(int(sum(e.size for e in enc)), dev)
    # decode: per-message results of this rank, gathered in message order
    j0, j1 = b64dist.shard_messages(toff, WORLD, rank)
    st, ep, ol = [], [], []
    for i in range(j0, j1):
        s, e, o = oracle.decode(text[toff[i]:toff[i + 1]])
        st.append(s)
        ep.append(e)
        ol.append(o.size)
    g = b64dist.gather_batch_decode(torch.tensor(st, dtype=torch.int32), torch.tensor(ep, dtype=torch.int64),
                                    torch.tensor(ol, dtype=torch.int64), dev)
    dist.destroy_process_group()
    q.put((rank, (i0, i1, base, j0, j1, [t.tolist() for t in g])))


def test_batch_shard_and_gather_world2():
    import oracle
    from inputs.gen import splitmix_bytes

    rng = np.random.default_rng(91)
    k = 300
    lens = rng.integers(0, 5000, k)
    lens[[3, 50, 51]] = 0  # empty messages
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    raw = splitmix_bytes(92, 0, int(off[-1]))
    encs = [oracle.encode(raw[off[i]:off[i + 1]]) for i in range(k)]
    text = np.concatenate(encs)
    toff = np.concatenate([[0], np.cumsum([e.size for e in encs])]).astype(np.int64)
    for i in rng.choice(k, 10, replace=False):  # corrupt some messages
        if toff[i + 1] > toff[i]:
            text[int(rng.integers(toff[i], toff[i + 1]))] = ord("!")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batch_worker, args=(r, port, raw, off, text, toff, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = _collect(procs, q, 120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # message ranges partition the batch, in rank order
    assert got[0][0] == 0 and got[WORLD - 1][1] == k
    assert all(got[r][1] == got[r + 1][0] for r in range(WORLD - 1))
    # global output base = encoded bytes of the messages before the rank's first
    for r in range(WORLD):
        assert got[r][2] == int(toff[got[r][0]])
    # gathered per-message decode results equal the whole-batch oracle
    ref = [oracle.decode(text[toff[i]:toff[i + 1]]) for i in range(k)]
    for r in range(WORLD):
        st, ep, ol = got[r][5]
        assert st == [x[0] for x in ref] and ep == [x[1] for x in ref] and ol == [x[2].size for x in ref]


def test_batch_shard_properties():
    """Equal-byte cuts moved to message boundaries: a partition of the
    messages in rank order; rank r starts at the first message starting at or
    after byte floor(T*r/G) (brute-force definition)."""
    from paper_1704_00605_b200 import b64_batch_shard

    rng = np.random.default_rng(93)
    for trial in range(200):
        k = int(rng.integers(0, 40))
        lens = rng.integers(0, 100, k) * (rng.random(k) < 0.8) + (rng.random(k) < 0.05) * 10_000
        off = np.concatenate([[int(rng.integers(0, 50))], np.cumsum(lens)]).astype(np.int64)
        off[1:] += off[0]
        T = int(off[-1] - off[0])
        for G in (1, 2, 3, 8):
            prev = 0
            for r in range(G):
                b, e = b64_batch_shard(off, G, r)
                assert b == prev and b <= e
                if r == 0:
                    assert b == 0
                else:
                    tgt = off[0] + T * r // G
                    assert b == next(i for i in range(k + 1) if off[i] >= tgt)
                prev = e
            assert prev == k
