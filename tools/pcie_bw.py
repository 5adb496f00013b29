#!/usr/bin/env python
"""Host<->device copy ceilings on this box (pinned memory, 1 GiB): H2D alone,
D2H alone, and both directions at once on two streams -- the bound for the
e2e numbers of bench.py (b64_encode_host / b64_decode_host)."""
import json
import time

import torch

n = 1 << 30
dev = torch.device("cuda", 0)
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


h2d = n / timed(lambda: d1.copy_(h1, non_blocking=True)) / 1e9
d2h = n / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


t = timed(both)
print(json.dumps({"h2d_GBps": h2d, "d2h_GBps": d2h, "duplex_each_GBps": n / t / 1e9}))
