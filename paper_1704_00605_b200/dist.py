"""Multi-GPU sharding of one large buffer (BASELINE.json configs[4]).

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.
Groups (3 bytes) and quads (4 chars) are independent, so a buffer is split
on 3-byte / 4-char boundaries with ``b64_shard`` and each rank runs the
single-GPU kernels on its own shard; data never crosses GPUs.  The only
exchange is decode's result: one int64 MIN all-reduce of the shard
reduction key (the global first-error offset and its status packed by the
C ABI's ``b64_shard_key``) and one all-gather of the per-shard output
lengths (NCCL over NVLink on the GPU box, gloo in the CPU tests).  The
whole-buffer result is computed by the C ABI (``b64_combine_shards``, or
``b64_combine_shards_async`` on the device); this module is collectives and
marshalling only.

Batches (configs[1]) shard by message: ``b64_batch_shard`` cuts the batch
into equal-byte ranges on message boundaries, each rank runs the batched
kernels on its messages, and the per-message results (decode: status,
err_pos, out_len; encode: the rank's output total, from which the global
output offsets follow) are all-gathered -- again no message data crosses
GPUs.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib

INT64_MAX = _lib.INT64_MAX


def combine(local_key: int, local_out_len: int, total_m: int, device, group=None):
    """Collectives of the sharded decode, host-driven form: MIN all-reduce of
    the shard reduction key (``b64_shard_key``: global first-error offset and
    status, INT64_MAX if clean) and all-gather of the shard output lengths;
    the whole-buffer result comes from the C ABI ``b64_combine_shards``.
    Returns (status, err_pos, out_len)."""
    world = dist.get_world_size(group)
    e = torch.tensor([local_key], dtype=torch.int64, device=device)
    dist.all_reduce(e, op=dist.ReduceOp.MIN, group=group)
    lens = torch.tensor([local_out_len], dtype=torch.int64, device=device)
    parts = [torch.empty(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(parts, lens, group=group)
    st, ep, ol, _ = _lib.b64_combine_shards(int(e.item()), [int(p.item()) for p in parts], total_m)
    return st, ep, ol


class ShardedDecode:
    """Device-resident sharded decode of one buffer (BASELINE.json configs[4]):
    the rank's shard decode writes its exchange record (key, out_len) in the
    kernel finalize, NCCL reduces the key (MIN) and gathers the lengths
    in place, and ``b64_combine_shards_async`` writes the whole buffer's
    b64_result on the device -- no host synchronization in the step.

    ``text_local`` is this rank's shard [begin, end) of a buffer of
    ``total_m`` characters split with ``b64_shard(total_m, 4, world, rank)``.
    """

    def __init__(self, text_local, out_local, begin: int, total_m: int, flags: int = 0, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = text_local.device
        self.text, self.out, self.begin, self.total_m, self.flags = text_local, out_local, begin, total_m, flags
        self.local = _lib.result_tensor(dev)
        self.key = torch.empty(2, dtype=torch.int64, device=dev)
        self.lens = torch.empty(self.world, dtype=torch.int64, device=dev)
        self.result = _lib.result_tensor(dev)

    def step(self, stream=None):
        _lib.b64_decode_shard_ex_async(self.text, self.out, self.local, self.begin,
                                       final_shard=(self.rank == self.world - 1), flags=self.flags,
                                       key=self.key, stream=stream)
        dist.all_reduce(self.key[0:1], op=dist.ReduceOp.MIN, group=self.group)
        dist.all_gather_into_tensor(self.lens, self.key[1:2], group=self.group)
        _lib.b64_combine_shards_async(self.key[0:1], self.lens, self.total_m, self.result, stream=stream)

    def read(self):
        """(status, err_pos, out_len) of the whole buffer (synchronizes)."""
        ol, ep, st, _ = _lib.unpack_result(self.result)
        return st, ep, ol


def decode_shard(text_local, out_local, result, begin: int, world: int, rank: int,
                 flags: int = 0, key=None, stream=None):
    """Enqueue this rank's shard decode (final-quad rules on the last rank
    only); ``key`` (int64[2]) receives the exchange record."""
    _lib.b64_decode_shard_ex_async(text_local, out_local, result, begin,
                                   final_shard=(rank == world - 1), flags=flags, key=key,
                                   stream=stream)


def local_key(result, begin: int) -> tuple[int, int]:
    """(reduction key, local out_len) from a shard's result tensor."""
    out_len, err_pos, status, _ = _lib.unpack_result(result)
    return _lib.b64_shard_key(status, err_pos, begin), out_len


def shard_range(total: int, unit: int, world: int, rank: int) -> tuple[int, int]:
    """Unit-aligned [begin, end) of rank's shard (C ABI b64_shard)."""
    return _lib.b64_shard(total, unit, world, rank)


# --------------------------------------------------------------- batches

def shard_messages(in_off, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of this rank's messages (C ABI b64_batch_shard)."""
    return _lib.b64_batch_shard(in_off, world, rank)


def _gather_var(x, device, group=None):
    """All-gather of a 1-D tensor whose length differs between ranks (padded
    to the longest, one all_gather of the lengths + one of the data)."""
    world = dist.get_world_size(group)
    n = torch.tensor([x.numel()], dtype=torch.int64, device=device)
    ns = [torch.empty(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(v.item()) for v in ns]
    mx = max(ns) if ns else 0
    pad = torch.zeros(mx, dtype=x.dtype, device=device)
    pad[: x.numel()] = x
    parts = [torch.empty(mx, dtype=x.dtype, device=device) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:m] for p, m in zip(parts, ns)])


def gather_batch_decode(status, err_pos, out_len, device, group=None):
    """Per-message decode results of every rank, in message order (the ranks
    hold consecutive message ranges).  err_pos / out_len are message-relative,
    so no translation is needed.  Returns (status, err_pos, out_len) of the
    whole batch."""
    return (_gather_var(status.to(torch.int64), device, group), _gather_var(err_pos, device, group),
            _gather_var(out_len, device, group))


def global_out_base(local_total: int, device, group=None) -> int:
    """Offset of this rank's first output byte in the concatenated output of
    the whole batch (exclusive prefix of the ranks' output totals)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = torch.tensor([local_total], dtype=torch.int64, device=device)
    parts = [torch.empty(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return int(sum(int(p.item()) for p in parts[:rank]))
