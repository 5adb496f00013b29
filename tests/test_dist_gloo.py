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
