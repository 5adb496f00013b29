#!/usr/bin/env python
"""What a large-message / small-message split of C2 could gain (GPU box).

Times, on the C2 workload (10,000 messages, log-uniform 100 B - 64 KiB),
with CUDA events and an L2 flush before every call:
  * the batched encode / decode of all messages (the product path);
  * the batched encode / decode of only the messages shorter than a cut;
  * the single-buffer encode / decode of the bytes of the longer messages,
    concatenated (the single-buffer kernels' rate: what CTA-wide tiles
    would reach on the long messages if they had no per-message edges).
The sum of the last two is an optimistic estimate of a hybrid kernel
(it ignores the long messages' partial tiles and runs the two parts back
to back, not concurrently).  Prints one JSON line per cut."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1704_00605_b200 as b64  # noqa: E402
from inputs import workloads as W  # noqa: E402
from inputs.gpu_gen import fill  # noqa: E402

dev = torch.device("cuda", 0)
lens, _ = W.c2_lengths()
off = W.offsets_from_lengths(lens)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps=20, warm=3):
    ts = []
    for r in range(warm + reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)) * 1000.0  # us


def batch_times(ls):
    o = W.offsets_from_lengths(ls)
    tot = int(o[-1])
    raw = torch.empty(max(tot, 1), dtype=torch.uint8, device=dev)
    fill(raw, W.C2_SEED)
    doff = torch.from_numpy(o).to(dev)
    mt = int(sum(4 * ((int(L) + 2) // 3) for L in ls))
    out = torch.empty(mt + 16, dtype=torch.uint8, device=dev)
    oo = torch.empty(ls.size + 1, dtype=torch.int64, device=dev)
    wse = torch.empty(b64.b64_batch_workspace_bytes(ls.size, tot, 0) + 256, dtype=torch.uint8, device=dev)
    wsd = torch.empty(b64.b64_batch_workspace_bytes(ls.size, mt, 1) + 256, dtype=torch.uint8, device=dev)
    y = torch.empty(tot + 16, dtype=torch.uint8, device=dev)
    yo = torch.empty(ls.size + 1, dtype=torch.int64, device=dev)
    yl = torch.empty(ls.size, dtype=torch.int64, device=dev)
    ye = torch.empty(ls.size, dtype=torch.int64, device=dev)
    ys = torch.empty(ls.size, dtype=torch.int32, device=dev)
    b64.b64_encode_batch(raw, doff, out=out, out_off=oo, ws=wse)
    te = timed(lambda: b64.b64_encode_batch(raw, doff, out=out, out_off=oo, ws=wse))
    td = timed(lambda: b64.b64_decode_batch(out, oo, out=y, out_off=yo, out_len=yl, err_pos=ye, status=ys,
                                            ws=wsd, total_in=mt))
    return te, td, tot, mt


def single_times(n):
    x = torch.empty(n, dtype=torch.uint8, device=dev)
    fill(x, W.C2_SEED)
    t = torch.empty(b64.b64_encoded_len(n), dtype=torch.uint8, device=dev)
    y = torch.empty(n + 3, dtype=torch.uint8, device=dev)
    res = b64.result_tensor(dev)
    b64.b64_encode(x, out=t)
    te = timed(lambda: b64.b64_encode(x, out=t))
    td = timed(lambda: b64.b64_decode_async(t, y, res))
    return te, td


full_e, full_d, tot, mt = batch_times(lens)
print(json.dumps({"what": "all messages, batched", "encode_us": full_e, "decode_us": full_d,
                  "bytes": tot, "text": mt}))
for cut in (8192, 16384, 32768):
    small = lens[lens < cut]
    big = lens[lens >= cut]
    se, sd, stot, smt = batch_times(small)
    be, bd = single_times(int(big.sum()))
    print(json.dumps({"cut": cut, "small_msgs": int(small.size), "small_bytes": stot,
                      "big_msgs": int(big.size), "big_bytes": int(big.sum()),
                      "small_batched_encode_us": se, "small_batched_decode_us": sd,
                      "big_single_buffer_encode_us": be, "big_single_buffer_decode_us": bd,
                      "estimate_encode_us": se + be, "estimate_decode_us": sd + bd,
                      "product_encode_us": full_e, "product_decode_us": full_d}))
