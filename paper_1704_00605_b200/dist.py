"""Multi-GPU sharding of one large buffer (BASELINE.json configs[4]).

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.
Groups (3 bytes) and quads (4 chars) are independent, so a buffer is split
on 3-byte / 4-char boundaries with ``b64_shard`` and each rank runs the
single-GPU kernels on its own shard; data never crosses GPUs.  The only
exchange is decode's result: one int64 MIN all-reduce of the global first
error offset and one all-gather of the per-shard output lengths (NCCL over
NVLink on the GPU box, gloo in the CPU tests).  Status is a pure function of
the global error offset (reading R-length), so nothing else is
exchanged.

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

INT64_MAX = (1 << 63) - 1


def shard_range(total: int, unit: int, world: int, rank: int) -> tuple[int, int]:
    """Unit-aligned [begin, end) of rank's shard (C ABI b64_shard)."""
    return _lib.b64_shard(total, unit, world, rank)


def global_decode_result(err_global: int, total_m: int, shard_lens: list[int]):
    """(status, err_pos, out_len) of the whole buffer from the reduced error
    offset (INT64_MAX = none) and the per-shard output lengths."""
    q, r = divmod(total_m, 4)
    if err_global == INT64_MAX:
        return _lib.B64_OK, -1, int(sum(shard_lens))
    if r != 0 and err_global == 4 * q:
        return _lib.B64_ERR_LENGTH, err_global, 3 * q
    return _lib.B64_ERR_INVALID_CHAR, err_global, 3 * (err_global // 4)


def combine(local_err_global: int, local_out_len: int, total_m: int, device, group=None):
    """Collectives of the sharded decode: MIN all-reduce of the error offset
    (already translated to a global offset, INT64_MAX if none) and
    all-gather of the shard output lengths.  Returns the global
    (status, err_pos, out_len)."""
    world = dist.get_world_size(group)
    e = torch.tensor([local_err_global], dtype=torch.int64, device=device)
    dist.all_reduce(e, op=dist.ReduceOp.MIN, group=group)
    lens = torch.tensor([local_out_len], dtype=torch.int64, device=device)
    parts = [torch.empty(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(parts, lens, group=group)
    return global_decode_result(int(e.item()), total_m, [int(p.item()) for p in parts])


def decode_shard(text_local, out_local, result, begin: int, world: int, rank: int,
                 stream=None):
    """Enqueue this rank's shard decode (final-quad rules on the last rank only)."""
    _lib.b64_decode_shard_async(text_local, out_local, result, final_shard=(rank == world - 1),
                                stream=stream)


def local_error_global(result, begin: int) -> tuple[int, int]:
    """(global error offset or INT64_MAX, local out_len) from a result tensor."""
    out_len, err_pos, status, _ = _lib.unpack_result(result)
    return (begin + err_pos if err_pos >= 0 else INT64_MAX), out_len


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
