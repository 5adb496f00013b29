"""Multi-process (world size 2, gloo, CPU) test of the sharded-decode result
exchange in paper_1704_00605_b200/dist.py: MIN all-reduce of the global
error offset + all-gather of shard output lengths must reproduce the
whole-buffer oracle result.  Shard-local results come from the oracle
(test infrastructure); on the GPU they come from b64_decode_shard_async."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_result(t_local, final):
    """Shard-local (err_pos, out_len) with R-shard semantics, via the oracle."""
    import oracle

    if final:
        st, ep, out = oracle.decode(t_local)
        return ep, out.size
    st, ep, out = oracle.decode(np.concatenate([t_local, np.frombuffer(b"AAAA", np.uint8)]))
    if st != oracle.OK and ep < t_local.size:
        return ep, 3 * (ep // 4)
    return -1, 3 * (t_local.size // 4)


def _worker(rank, port, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from paper_1704_00605_b200 import dist as b64dist
    from paper_1704_00605_b200 import b64_shard

    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    res = []
    for t in cases:
        b, e = b64_shard(t.size, 4, WORLD, rank)
        ep, ol = _local_result(t[b:e], final=(rank == WORLD - 1))
        g = b + ep if ep >= 0 else b64dist.INT64_MAX
        res.append(b64dist.combine(g, ol, t.size, torch.device("cpu")))
    dist.destroy_process_group()
    q.put((rank, res))


def test_sharded_decode_combine_world2():
    import oracle
    from inputs.gen import splitmix_bytes

    x = splitmix_bytes(77, 0, 30001)
    t = oracle.encode(x)            # 40004 chars, ends with one '='
    cases = [t, t[:-1], t[:-3]]
    for pos, b in [(5, 0x21), (20010, 0x21), (39999, 0x00), (20000, ord("=")), (20003, ord("="))]:
        u = t.copy()
        u[pos] = b
        cases.append(u)
    u = t.copy()
    u[100] = 0x80
    u[30000] = 0x80
    cases.append(u)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, cases, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for i, c in enumerate(cases):
        st, ep, out = oracle.decode(c)
        for r in range(WORLD):
            assert got[r][i] == (st, ep, out.size), (i, r, got[r][i], (st, ep, out.size))


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
    got = dict(q.get(timeout=120) for _ in range(WORLD))
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
