#!/usr/bin/env python
"""Small, fast invocations of every kernel (all alignment classes, tails,
errors, padding, batched, shard) for compute-sanitizer runs:
  compute-sanitizer --tool memcheck python tools/sanitize_cases.py
Checks results against the CPU oracle as it goes (test infrastructure)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import oracle
import paper_1704_00605_b200 as b64
from inputs.gen import splitmix_bytes

dev = torch.device("cuda:0")


def to_dev(x, mis=0):
    base = torch.zeros(x.size + mis + 64, dtype=torch.uint8, device=dev)
    v = base[mis: mis + x.size]
    if x.size:
        v.copy_(torch.from_numpy(x))
    return v


def main():
    x = splitmix_bytes(5, 0, 40000)
    n_ok = 0
    for n in (0, 1, 2, 3, 47, 12288, 12289, 30001):
        for im in (0, 3, 4):
            for om in (0, 1, 8):
                d = to_dev(x[:n], im)
                base = torch.zeros(b64.b64_encoded_len(n) + om + 64, dtype=torch.uint8, device=dev)
                t = b64.b64_encode(d, out=base[om: om + b64.b64_encoded_len(n)])
                ref = oracle.encode(x[:n])
                assert np.array_equal(t.cpu().numpy(), ref)
                td = to_dev(ref, om)
                yb = torch.zeros(b64.b64_decoded_max_len(ref.size) + im + 64, dtype=torch.uint8, device=dev)
                y, st, ep = b64.b64_decode(td, out=yb[im: im + b64.b64_decoded_max_len(ref.size)])
                assert st == 0 and np.array_equal(y.cpu().numpy(), x[:n])
                n_ok += 1
    t = oracle.encode(x[:20000])
    t[777] = 0
    y, st, ep = b64.b64_decode(to_dev(t))
    assert (st, ep) == (1, 777)
    # batched
    lens = np.array([0, 5, 100, 1536, 1537, 3000, 0, 64, 7000], dtype=np.int64)
    off = np.zeros(lens.size + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    raw = splitmix_bytes(6, 0, int(off[-1]))
    out, oo = b64.b64_encode_batch(to_dev(raw, 3), torch.from_numpy(off).to(dev))
    o, oo = out.cpu().numpy(), oo.cpu().numpy()
    texts = [oracle.encode(raw[off[i]: off[i + 1]]) for i in range(lens.size)]
    for i, tt in enumerate(texts):
        assert np.array_equal(o[oo[i]: oo[i + 1]], tt)
    tall = np.concatenate(texts)
    tall[oo[3] + 10] = ord("!")
    y, yo, yl, ye, ys = b64.b64_decode_batch(to_dev(tall, 5), torch.from_numpy(oo).to(dev))
    assert ys.cpu().numpy().tolist() == [0, 0, 0, 1, 0, 0, 0, 0, 0]
    # shard
    res = b64.result_tensor(dev)
    out = torch.empty(30000, dtype=torch.uint8, device=dev)
    b64.b64_decode_shard_async(to_dev(t[:8000]), out, res, final_shard=False)
    assert b64.unpack_result(res)[1] == 777
    torch.cuda.synchronize()
    print("sanitize cases ok", n_ok)


if __name__ == "__main__":
    main()
