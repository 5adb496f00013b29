#!/usr/bin/env python
"""Per-warp timeline of the batched kernel (trace build, B64_BATCH_TRACE):
runs one C2 batched encode and decode with the variant library named by
B64GPU_LIB and prints the distribution of the globaltimer stamps (kernel
start, plan done, first unit data ready, warp done) relative to the earliest."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1704_00605_b200 as b64  # noqa: E402
from inputs import workloads as W  # noqa: E402
from inputs.gpu_gen import fill  # noqa: E402

lib = b64.load_library()
dev = torch.device("cuda", 0)
lens, _ = W.c2_lengths()
off = W.offsets_from_lengths(lens)
tot = int(off[-1])
raw = torch.empty(tot, dtype=torch.uint8, device=dev)
fill(raw, W.C2_SEED)
doff = torch.from_numpy(off).to(dev)
k = lens.size
mt = int(sum(4 * ((int(L) + 2) // 3) for L in lens))
out = torch.empty(mt + 16, dtype=torch.uint8, device=dev)
out_off = torch.empty(k + 1, dtype=torch.int64, device=dev)
wse = torch.empty(b64.b64_batch_workspace_bytes(k, tot, 0) + 256, dtype=torch.uint8, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
N = 148 * 64 * 4
buf = (ctypes.c_ulonglong * N)()
lib.b64_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
for rep in range(4):
    flush.zero_()
    torch.cuda.synchronize()
    b64.b64_encode_batch(raw, doff, out=out, out_off=out_off, ws=wse)
    torch.cuda.synchronize()
lib.b64_debug_trace(ctypes.addressof(buf), N)
a = np.frombuffer(buf, dtype=np.uint64).reshape(148, 64, 4).astype(np.int64)
nw = int(os.environ.get("B64_TRACE_WARPS", "16"))
if os.environ.get("B64_TRACE_WAIT"):  # batch_kernel trace-wait build: cycles waiting for unit data / in the unit loop
    x = a[:, 32:32 + nw, :].reshape(-1, 4)
    fr = x[:, 0] / np.maximum(x[:, 1], 1)
    print("unit-data wait / unit loop cycles: mean", round(float(fr.mean()), 3), "p10", round(float(np.percentile(fr, 10)), 3),
          "p90", round(float(np.percentile(fr, 90)), 3), " loop cycles p50", int(np.median(x[:, 1])))
if os.environ.get("B64_TRACE_EXT"):  # batch2_kernel: warps 32.. hold start / searched / issued / grid-synced
    x = a[:, 32:32 + nw, :].reshape(-1, 4)
    t0x = x[:, 0].min()
    for i, name in enumerate(["k_start", "searched", "issued", "gsynced"]):
        v = (x[:, i] - t0x) / 1000.0
        print(f"{name:10} min {v.min():7.2f} p50 {np.median(v):7.2f} max {v.max():7.2f} us")
    y = a[:, :nw, :].reshape(-1, 4)
    for i, name in ((1, "plan_done"), (2, "first_data"), (3, "done")):
        v = (y[:, i] - t0x) / 1000.0
        print(f"{name:10} min {v.min():7.2f} p50 {np.median(v):7.2f} max {v.max():7.2f} us (from kernel start)")
a = a[:, :nw, :].reshape(-1, 4)
if True:  # slot 0 holds (bytes << 20 | units) of the warp (trace builds)
    wb = a[:, 0] >> 20
    wu = a[:, 0] & 0xFFFFF
    d3 = (a[:, 3] - a[:, 1]) / 1000.0
    print("units per warp: min", wu.min(), "max", wu.max(), " bytes per warp: min", wb.min(), "max", wb.max())
    import numpy as _np
    print("corr(done-plan, bytes) =", round(float(_np.corrcoef(d3, wb)[0, 1]), 3),
          " corr(done-plan, units) =", round(float(_np.corrcoef(d3, wu)[0, 1]), 3))
    slow = _np.argsort(-d3)[:5]
    print("slowest warps (cta, warp, us after plan, bytes, units):",
          [(int(i // nw), int(i % nw), round(float(d3[i]), 1), int(wb[i]), int(wu[i])) for i in slow])
    a[:, 0] = a[:, 1] - 5000
elif os.environ.get("B64_TRACE_FM"):
    fm = a[:, 0] >> 32
    tm = a[:, 0] & 0xFFFFFFFF
    print("first_msg mismatches:", int((fm != tm).sum()))
    a[:, 0] = a[:, 1] - 5000
t0 = a[:, 0].min()
r = (a - t0) / 1000.0  # us
for i, name in enumerate(["start", "plan_done", "first_data", "done"]):
    v = r[:, i]
    print(f"{name:10} min {v.min():7.2f} p10 {np.percentile(v,10):7.2f} p50 {np.median(v):7.2f} "
          f"p90 {np.percentile(v,90):7.2f} max {v.max():7.2f} us")

d = (a[:, 3] - t0) / 1000.0
idx = np.argsort(-d)[:12]
print("slowest warps (cta, warp, done_us, first_data_us):",
      [(int(i // nw), int(i % nw), round(float(d[i]), 1), round(float(r[i, 2]), 1)) for i in idx])

per = d.reshape(148, nw)
print("mean done per warp index:", [round(float(x), 1) for x in per.mean(axis=0)])
print("mean first_data per warp index:", [round(float(x), 1) for x in r[:, 2].reshape(148, nw).mean(axis=0)])
