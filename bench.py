#!/usr/bin/env python
"""bench.py -- base64 encode + validating decode throughput on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (torchrun
for N > 1) prints ONE JSON line on rank 0.

Workload (default, BASELINE.json configs[4] = "C5"): 32 GiB of seeded
random bytes split on 3-byte boundaries over the N ranks (b64_shard).  One
step = the whole hot path over the rank's shard: encode its bytes (SURVEY.md
§8 rows a1-a5), validating decode of the produced text (rows a6-a12, the
last rank applies the final-quad rules) and -- for N > 1 -- the result
exchange (int64 MIN all-reduce of the error offset + all-gather of output
lengths over NCCL).  value = (encode input bytes + decode input chars) of all
ranks x K / max-over-ranks device time, in GB/s (1e9).  Inputs are far larger
than L2 (126 MB), so no flush is needed between steps.  ``--workload c3``
runs config 3 (1 GiB + 2 bytes on every rank) instead; ``--workload c2``
the batched 10,000-message config.

``--impl reference`` times the CPU oracle (the only "reference" this paper
has: no runnable code exists) on the host cores on bounded
samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "base64 encode/decode GB/s (input bytes) per GPU and % of HBM roofline, 1-8 B200"
FALLBACK_HBM_GBS = 6650.0


# ------------------------------------------------------------------ utils

def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def source_hash():
    """sha256 of the library's sources (csrc/*.cu[h], include/b64gpu.h): the
    stamp under which profiles/ncu_traffic.json entries were captured."""
    import hashlib

    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1704_00605_b200", "csrc")
    files = sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cu", ".cuh")))
    for f in files + [os.path.join(ROOT, "include", "b64gpu.h")]:
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode())
            h.update(fh.read())
    return h.hexdigest()[:16]


def measured_traffic(key):
    """dram bytes per launch of `key` from profiles/ncu_traffic.json, only
    if it was captured from the sources being benched (else None, reason)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
    except (OSError, ValueError):
        return None, "no profiles/ncu_traffic.json"
    ent = tr.get(key)
    if not ent:
        return None, f"no entry {key}"
    if ent.get("source_sha") != source_hash():
        return None, f"stale: captured from sources {ent.get('source_sha')}, benched {source_hash()}"
    return ent.get("dram_bytes_per_launch"), ent.get("source")


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count(), len(os.sched_getaffinity(0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw",
              "clocks_event_reasons.active", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=1)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_threads_bench(x, reps_min_s=1.0, threads=None):
    """Time the scalar CPU oracle (encode, then decode of its output) on the
    host cores; the buffer is split on 3-byte boundaries into one chunk per
    thread (ctypes releases the GIL).  Returns (GB/s of input bytes, cores,
    bytes_in, seconds)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    T = threads or len(os.sched_getaffinity(0))
    n = x.size
    q = (n + 2) // 3
    bounds = [(min(3 * (q * r // T), n), min(3 * (q * (r + 1) // T), n)) for r in range(T)]
    texts = [np.empty(4 * ((e - b + 2) // 3), dtype=np.uint8) for b, e in bounds]
    outs = [np.empty(max(3 * (t.size // 4), 1), dtype=np.uint8) for t in texts]

    def job(i):
        b, e = bounds[i]
        oracle.encode_into(x[b:e], texts[i])
        oracle.decode_into(texts[i], outs[i])

    oracle.build()
    m = sum(t.size for t in texts)
    with ThreadPoolExecutor(T) as ex:
        t0 = time.perf_counter()
        reps = 0
        while True:
            list(ex.map(job, range(T)))
            reps += 1
            el = time.perf_counter() - t0
            if el >= reps_min_s:
                break
    return (n + m) * reps / el / 1e9, T, (n + m) * reps, el


# ------------------------------------------------------------- our arm

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1704_00605_b200 as b64
    from inputs import workloads as W
    from inputs.gpu_gen import fill
    from paper_1704_00605_b200.dist import INT64_MAX

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPUs visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        # communicator evidence (stderr): one line per rank
        probe = torch.ones(1, device=dev)
        dist.all_reduce(probe)
        print(f"[bench] rank {rank}/{world} on {torch.cuda.get_device_name(dev)} cuda:{local}: NCCL "
              f"{'.'.join(map(str, torch.cuda.nccl.version()))} process group up, all_reduce(1) = "
              f"{int(probe.item())}", file=sys.stderr, flush=True)
        assert int(probe.item()) == world
    b64.load_library()
    stream = torch.cuda.current_stream(dev)

    wl = args.workload
    if wl == "c5":
        total, seed = W.C5_N, W.C5_SEED
        begin, end = b64.b64_shard(total, 3, world, rank)
        scaling = "strong"
        wdesc = "C5: 32 GiB uniform random bytes (seed 5) split on 3-byte boundaries over the ranks; encode + validating decode"
    elif wl == "c3":
        total, seed = W.C3_N, W.C3_SEED
        begin, end = 0, total
        scaling = "weak"
        wdesc = "C3: 1 GiB + 2 uniform random bytes (seed 2) per rank; encode + validating decode"
    else:
        raise SystemExit(f"unknown workload {wl}")
    n = end - begin
    m = b64.b64_encoded_len(n)
    final = rank == world - 1 or wl != "c5"

    x = torch.empty(n, dtype=torch.uint8, device=dev)
    fill(x, seed, begin)
    t = torch.empty(m, dtype=torch.uint8, device=dev)
    y = torch.empty(max(b64.b64_decoded_max_len(m), 1), dtype=torch.uint8, device=dev)
    res = b64.result_tensor(dev)
    lib = b64.load_library()
    import ctypes
    sptr = ctypes.c_void_p(stream.cuda_stream)
    xp, tp, yp, rp = x.data_ptr(), t.data_ptr(), y.data_ptr(), res.data_ptr()

    # multi-GPU exchange: the shard decode writes its
    # exchange record (reduction key, out_len) in the kernel finalize; NCCL
    # reduces the key (MIN) and gathers the lengths; b64_combine_shards_async
    # writes the whole buffer's result on the device.  No host sync.
    tbegin = 4 * (begin // 3)                    # global offset of this rank's text shard
    total_m = b64.b64_encoded_len(total) if wl == "c5" else m
    key = torch.empty(2, dtype=torch.int64, device=dev)
    lens = torch.empty(world, dtype=torch.int64, device=dev)
    gres = b64.result_tensor(dev)
    kp, lp, gp = key.data_ptr(), lens.data_ptr(), gres.data_ptr()

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        rc = lib.b64_encode(xp, n, tp, sptr)
        if rc < 0:
            raise RuntimeError(f"encode rc={rc}")
        if ev is not None:
            ev[1].record(stream)
        if world == 1:
            rc = lib.b64_decode_shard_async(tp, m, 1 if final else 0, yp, rp, sptr)
        else:
            rc = lib.b64_decode_shard_ex_async(tp, m, tbegin, 1 if final else 0, yp, 0, rp, kp, sptr)
        if rc < 0:
            raise RuntimeError(f"decode rc={rc}")
        if ev is not None:
            ev[2].record(stream)
        if world > 1:
            dist.all_reduce(key[0:1], op=dist.ReduceOp.MIN)
            dist.all_gather_into_tensor(lens, key[1:2])
            rc = lib.b64_combine_shards_async(kp, lp, world, total_m, gp, sptr)
            if rc < 0:
                raise RuntimeError(f"combine rc={rc}")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    # correctness guard of the measured configuration (cheap, outside timing)
    ol, ep, st, _ = b64.unpack_result(res)
    if os.environ.get("B64_BENCH_NOCHECK") != "1":   # skeleton variants only (tools/sweep.py)
        assert st == 0 and ep == -1 and ol == n, (st, ep, ol)
        if world > 1:
            gol, gep, gst, _ = b64.unpack_result(gres)
            assert (gst, gep, gol) == (0, -1, total), (gst, gep, gol)

    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    time.sleep(0.15)
    t_start.record(stream)
    for k in range(K):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    enc_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / K
    dec_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / K
    ms = torch.tensor([ms_total, enc_ms, dec_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_total, enc_ms, dec_ms = ms.tolist()

    tot_n = total if wl == "c5" else total * world
    tot_m = b64.b64_encoded_len(total) if wl == "c5" else b64.b64_encoded_len(total) * world
    value = (tot_n + tot_m) * K / (ms_total / 1e3) / 1e9

    hbm, hbm_src = peaks()
    enc_bytes = n + m           # algorithmic bytes per encode launch (read n, write 4*ceil(n/3))
    dec_bytes = m + n           # per decode launch (read m chars, write n bytes)
    enc_gbs = enc_bytes / (enc_ms / 1e3) / 1e9
    dec_gbs = dec_bytes / (dec_ms / 1e3) / 1e9
    dom = "decode" if dec_ms >= enc_ms else "encode"
    ach = dec_gbs if dom == "decode" else enc_gbs
    traffic, traffic_src = measured_traffic(f"{wl}:{dom}")

    # ---- e2e through the C ABI host-buffer entry points (rank-local sample)
    e2e = None
    if not args.no_e2e:
        ns = min(n, args.e2e_bytes - args.e2e_bytes % 3) if n > args.e2e_bytes else n
        ms_ = b64.b64_encoded_len(ns)
        hx = torch.empty(ns, dtype=torch.uint8).pin_memory()
        hx.copy_(x[:ns])
        ht = torch.empty(ms_, dtype=torch.uint8).pin_memory()
        hy = torch.empty(max(b64.b64_decoded_max_len(ms_), 1), dtype=torch.uint8).pin_memory()
        for _ in range(1):
            b64.b64_encode_host(hx, ht, x, t)
            b64.b64_decode_host(ht, hy, t, y)
        reps = args.e2e_steps
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            b64.b64_encode_host(hx, ht, x, t)
            st_, ol_, ep_ = b64.b64_decode_host(ht, hy, t, y)
        el = time.perf_counter() - t0
        assert st_ == 0 and ol_ == ns
        elt = torch.tensor([el], dtype=torch.float64, device=dev)
        tot = torch.tensor([float(ns + ms_)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(elt, op=dist.ReduceOp.MAX)
            dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        e2e = {"value": tot.item() * reps / elt.item() / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": ns + ms_, "d2h_bytes_per_step": ms_ + ns + 2 * 24,
               "sample": f"{ns} bytes per rank (pinned host) -> b64_encode_host -> b64_decode_host, {reps} steps"}

    # ---- CPU oracle on the host cores (rank 0; the other ranks wait)
    cpu = None
    if world > 1:
        dist.barrier()
    if rank == 0 and not args.no_cpu:
        smp = min(n, args.cpu_sample)
        smp -= smp % 3
        xs = x[:smp].cpu().numpy()
        gbs, cores, nbytes, el = oracle_threads_bench(xs, reps_min_s=args.cpu_seconds)
        # the paper's own measurements are single-threaded
        s1 = min(smp, args.cpu_sample_1core - args.cpu_sample_1core % 3)
        gbs1, _, nb1, el1 = oracle_threads_bench(xs[:s1], reps_min_s=args.cpu_seconds_1core, threads=1)
        model, ncpu, naff = cpu_info()
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle",
               "sample": f"first {smp} bytes of the rank-0 workload: oracle encode + decode of its text, "
                         f"split on 3-byte boundaries over {cores} threads, {el:.1f} s wall",
               "cpu_model": model, "cpu_count": ncpu,
               "single_core": {"value": gbs1, "unit": "GB/s", "cores": 1,
                               "sample": f"first {s1} bytes, one thread, {el1:.1f} s wall (paper: single-threaded, P:1092)"}}
    if world > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_total / K, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic: counter-based SplitMix64 bytes (inputs/gen.py), generated on device",
            "config": {"workload": wdesc, "bytes_per_rank": n, "chars_per_rank": m,
                       "total_bytes": tot_n, "total_chars": tot_m,
                       "parallelism": f"shard x{world}: no data-path collective; MIN all-reduce + length all-gather",
                       "l2": "inputs larger than L2 (126 MB): no flush"},
            "roofline": {"bound": "hbm", "kernel": f"{dom}_kernel", "achieved": ach, "peak": hbm,
                         "unit": "GB/s", "frac": ach / hbm, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": hbm_src,
                         "frac_of_nominal_8tbs": ach / 8000.0,
                         "algorithmic_bytes_per_launch": dec_bytes if dom == "decode" else enc_bytes},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": (2 if world == 1 else 3) * K,
            "gpu_launches_scope": "per rank: 1 encode_kernel + 1 decode_kernel per step" + (
                "" if world == 1 else " + 1 combine_kernel (NCCL all_reduce / all_gather kernels not counted)"),
            "clocks": clocks,
            "detail": {"encode_ms": enc_ms, "decode_ms": dec_ms,
                       "encode_GBps_input": n / (enc_ms / 1e3) / 1e9,
                       "decode_GBps_input": m / (dec_ms / 1e3) / 1e9,
                       "encode_roofline_frac": enc_gbs / hbm, "decode_roofline_frac": dec_gbs / hbm,
                       "encode_hbm_GBps": enc_gbs, "decode_hbm_GBps": dec_gbs},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------- configs C1 / C2 / C4 (1 GPU)

def run_small_configs(args):
    """Config lines for C1 (1 MiB round trip, latency), C2 (batched 10,000
    messages) and C4 (256 MiB decode, clean + 256 errors).  These are parity
    configs reported for completeness; L2 is flushed (512 MiB write + 256 MiB read) before
    every timed step and only the codec calls sit between the events."""
    import numpy as np
    import torch

    import paper_1704_00605_b200 as b64
    from inputs import workloads as W
    from inputs.gpu_gen import fill

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    # L2 flush = a 512 MiB write (evicts every input line), then a 256 MiB
    # read so that the write-back of the flush's own dirty lines happens
    # before the timed region instead of inside it (126 MB of dirty L2 would
    # otherwise drain to HBM during the first microseconds of the next step).
    flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    hbm, hbm_src = peaks()
    K, Wm = args.steps, args.warmup
    res = b64.result_tensor(dev)

    samples = {}
    clocks = ClockSampler(dev.index or 0)

    def timed(fn, name=None, flush_l2=True):
        ts = []
        for k in range(Wm + K):
            if flush_l2:
                flush.zero_()
                flush_rd.amax()
            else:
                # keep the GPU busy while the host enqueues the timed call, so
                # the events bracket device time, not host submission latency
                torch.cuda._sleep(200_000)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            if k >= Wm:
                ts.append(e0.elapsed_time(e1))
        if name:
            samples[name] = {"min_ms": min(ts), "median_ms": statistics.median(ts)}
        return sum(ts) / K  # ms per step (mean)

    wl = args.workload
    detail = {}
    kname = {}
    clocks.start()
    if wl == "c1":
        n = W.C1_N
        x = torch.empty(n, dtype=torch.uint8, device=dev)
        fill(x, W.C1_SEED)
        m = b64.b64_encoded_len(n)
        t = torch.empty(m, dtype=torch.uint8, device=dev)
        y = torch.empty(b64.b64_decoded_max_len(m), dtype=torch.uint8, device=dev)
        b64.b64_encode(x, out=t)
        pos, byte = W.c1_corruption(m)
        td = t.clone()
        td[pos] = byte
        enc_ms = timed(lambda: b64.b64_encode(x, out=t), "encode")
        dec_ms = timed(lambda: b64.b64_decode_async(t, y, res), "decode")
        dirty_ms = timed(lambda: b64.b64_decode_async(td, y, res), "dirty_decode")
        assert b64.unpack_result(res)[1] == pos
        hot_enc = timed(lambda: b64.b64_encode(x, out=t), "encode_hot_l2", flush_l2=False)
        hot_dec = timed(lambda: b64.b64_decode_async(t, y, res), "decode_hot_l2", flush_l2=False)
        assert b64.unpack_result(res)[2] == 0
        # the same three calls captured once in a CUDA graph and replayed
        gs = torch.cuda.Stream()
        res2 = b64.result_tensor(dev)
        with torch.cuda.stream(gs):
            b64.b64_encode(x, out=t, stream=gs)
            b64.b64_decode_async(t, y, res, stream=gs)
            b64.b64_decode_async(td, y, res2, stream=gs)
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            b64.b64_encode(x, out=t, stream=gs)
            b64.b64_decode_async(t, y, res, stream=gs)
            b64.b64_decode_async(td, y, res2, stream=gs)
        serial_ms = timed(graph.replay, "graph_replay_serial")
        assert b64.unpack_result(res)[2] == 0 and b64.unpack_result(res2)[1] == pos
        # the two decodes are independent once the encode is done: fork-join
        # graph, the dirty decode on a second stream (its own output buffer;
        # every stream has its own decode scratch)
        gs2 = torch.cuda.Stream()
        y2 = torch.empty_like(y)
        with torch.cuda.stream(gs2):
            b64.b64_decode_async(td, y2, res2, stream=gs2)
        torch.cuda.synchronize(dev)
        graph2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph2, stream=gs):
            b64.b64_encode(x, out=t, stream=gs)
            ev_f = torch.cuda.Event()
            ev_f.record(gs)
            gs2.wait_event(ev_f)
            b64.b64_decode_async(t, y, res, stream=gs)
            b64.b64_decode_async(td, y2, res2, stream=gs2)
            ev_j = torch.cuda.Event()
            ev_j.record(gs2)
            gs.wait_event(ev_j)
        res.zero_()
        res2.zero_()
        graph_ms = timed(graph2.replay, "graph_replay")
        assert b64.unpack_result(res)[2] == 0 and b64.unpack_result(res)[0] == n
        assert b64.unpack_result(res2)[1] == pos and torch.equal(y[:n], x)
        # end-to-end sync API latency (includes the result read-back)
        t0 = time.perf_counter()
        for _ in range(200):
            b64.b64_decode(t, out=y)
        sync_us = (time.perf_counter() - t0) / 200 * 1e6
        # one step = the three calls; replayed as one CUDA graph (the kernels
        # are the same launches, the graph removes the per-launch gaps)
        ms = graph_ms
        value = (n + 2 * m) / (ms / 1e3) / 1e9
        algo = {"encode": n + m, "decode": m + n}
        detail = {"encode_us": enc_ms * 1e3, "decode_us": dec_ms * 1e3, "dirty_decode_us": dirty_ms * 1e3,
                  "encode_hot_l2_us": hot_enc * 1e3, "decode_hot_l2_us": hot_dec * 1e3,
                  "graph_replay_all_three_us": graph_ms * 1e3,
                  "graph_replay_all_three_serial_us": serial_ms * 1e3,
                  "sync_decode_api_us": sync_us}
        dom, dom_ms = ("encode", enc_ms) if enc_ms >= dec_ms else ("decode", dec_ms)
        desc = ("C1: 2^20 random bytes (seed 0): encode, decode, decode of a copy with one NA191 byte; "
                "step = one CUDA-graph replay of the three calls (the two decodes, independent once the "
                "encode is done, on forked streams)")
        launches = 3
    elif wl == "c2":
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
        wsd = torch.empty(b64.b64_batch_workspace_bytes(k, mt, 1) + 256, dtype=torch.uint8, device=dev)
        y = torch.empty(tot + 16, dtype=torch.uint8, device=dev)
        y_off = torch.empty(k + 1, dtype=torch.int64, device=dev)
        y_len = torch.empty(k, dtype=torch.int64, device=dev)
        y_err = torch.empty(k, dtype=torch.int64, device=dev)
        y_st = torch.empty(k, dtype=torch.int32, device=dev)
        b64.b64_encode_batch(raw, doff, out=out, out_off=out_off, ws=wse)

        def enc():
            b64.b64_encode_batch(raw, doff, out=out, out_off=out_off, ws=wse)

        def dec():
            b64.b64_decode_batch(out, out_off, out=y, out_off=y_off, out_len=y_len, err_pos=y_err,
                                 status=y_st, ws=wsd, total_in=mt)

        enc_ms = timed(enc, "encode")
        dec_ms = timed(dec, "decode")
        if os.environ.get("B64_BENCH_NOCHECK") != "1":
            assert int(y_st.abs().sum().item()) == 0 and torch.equal(y[:tot], raw)
        # one step = batched encode then batched decode, replayed as one CUDA graph
        gs = torch.cuda.Stream()
        with torch.cuda.stream(gs):
            b64.b64_encode_batch(raw, doff, out=out, out_off=out_off, ws=wse, stream=gs)
            b64.b64_decode_batch(out, out_off, out=y, out_off=y_off, out_len=y_len, err_pos=y_err,
                                 status=y_st, ws=wsd, total_in=mt, stream=gs)
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            b64.b64_encode_batch(raw, doff, out=out, out_off=out_off, ws=wse, stream=gs)
            b64.b64_decode_batch(out, out_off, out=y, out_off=y_off, out_len=y_len, err_pos=y_err,
                                 status=y_st, ws=wsd, total_in=mt, stream=gs)
        y.zero_()
        graph_ms = timed(graph.replay, "graph_replay")
        if os.environ.get("B64_BENCH_NOCHECK") != "1":
            assert int(y_st.abs().sum().item()) == 0 and torch.equal(y[:tot], raw)
        ms = graph_ms
        value = (tot + mt) / (ms / 1e3) / 1e9
        algo = {"encode": tot + mt + 16 * (k + 1), "decode": mt + tot + 16 * (k + 1) + 20 * k}
        detail = {"encode_ms": enc_ms, "decode_ms": dec_ms, "graph_replay_ms": graph_ms, "messages": k,
                  "raw_bytes": tot, "text_bytes": mt,
                  "encode_GBps_input": tot / (enc_ms / 1e3) / 1e9, "decode_GBps_input": mt / (dec_ms / 1e3) / 1e9}
        dom, dom_ms = ("encode", enc_ms) if enc_ms >= dec_ms else ("decode", dec_ms)
        kname = {"encode": "batch_kernel<false>", "decode": "batch_kernel<true>"}
        desc = ("C2: 10,000 messages, log-uniform 100 B - 64 KiB (seed 1): batched encode + batched decode "
                "(incl. planner); step = one CUDA-graph replay of the two calls")
        launches = 2
    elif wl in ("despace", "despace_irregular"):
        # f3: 1.27 GB of MIME-style text (76-char lines + CRLF, 2.6 % whitespace),
        # built on the device from C3-seeded bytes with our encoder + a view.
        # despace_irregular: every 50th line ends in " \n" instead of CR LF,
        # so the line fast path gives up and the two-pass path does the work.
        nraw = 57 * (1 << 24)
        raw = torch.empty(nraw, dtype=torch.uint8, device=dev)
        fill(raw, W.C3_SEED)
        t = torch.empty(b64.b64_encoded_len(nraw), dtype=torch.uint8, device=dev)
        b64.b64_encode(raw, out=t)
        lines = t.view(-1, 76)
        w = torch.empty(lines.shape[0], 78, dtype=torch.uint8, device=dev)
        w[:, :76] = lines
        w[:, 76] = 13
        w[:, 77] = 10
        if wl == "despace_irregular":
            w[::50, 76] = ord(" ")
        w = w.view(-1)
        m = w.numel()
        out = torch.empty(m, dtype=torch.uint8, device=dev)
        ws = torch.empty(b64.load_library().b64_despace_workspace_bytes(m), dtype=torch.uint8, device=dev)
        olen_t = [None]

        def ds():
            olen_t[0] = b64.b64_despace(w, out=out, ws=ws)[1]

        ds_ms = timed(ds, "despace")
        kept = int(olen_t[0].item())
        assert kept == t.numel() and torch.equal(out[:kept], t)
        fast = int(ws[:4].view(torch.int32).item())  # WlState.verdict
        assert fast == (1 if wl == "despace" else 0)
        ms = ds_ms
        value = m / (ms / 1e3) / 1e9
        algo = {"despace": m + kept}
        detail = {"despace_ms": ds_ms, "in_bytes": m, "out_bytes": kept,
                  "despace_GBps_input": m / (ds_ms / 1e3) / 1e9,
                  "path": "line fast path" if fast else "general two-pass path (fast path gave up)"}
        dom, dom_ms = "despace", ds_ms
        kname = {"despace": "b64_despace call (all its kernels)"}
        desc = ("f3: whitespace removal of 1.27 GB MIME-style text (76-char lines + CRLF)"
                + (", irregular line ends (general path)" if wl == "despace_irregular" else ""))
        launches = 3
    elif wl == "mime":
        # f4: MIME round trip of 57 * 2^24 random bytes: line-wrapped encode
        # (76-char lines + CRLF, 1.31 GB of text) and whitespace-tolerant
        # decode of that text back to the bytes.
        nraw = 57 * (1 << 24)
        raw = torch.empty(nraw, dtype=torch.uint8, device=dev)
        fill(raw, W.C3_SEED)
        m = b64.b64_encoded_len_wrapped(nraw, 76, True)
        w = torch.empty(m, dtype=torch.uint8, device=dev)
        y = torch.empty(b64.b64_decoded_max_len(m), dtype=torch.uint8, device=dev)
        ws = torch.empty(b64.b64_decode_ws_workspace_bytes(m), dtype=torch.uint8, device=dev)
        enc_ms = timed(lambda: b64.b64_encode_wrapped(raw, out=w, line_chars=76, crlf=True), "encode_wrapped")
        dec_ms = timed(lambda: b64.b64_decode_ws_async(w, y, res, ws=ws), "decode_ws")
        ol, ep, st, _ = b64.unpack_result(res)
        assert (ol, ep, st) == (nraw, -1, 0) and torch.equal(y[:nraw], raw)
        assert int(w[76].item()) == 13 and int(w[77].item()) == 10
        ms = enc_ms + dec_ms
        value = (nraw + m) / (ms / 1e3) / 1e9
        algo = {"encode_wrapped": nraw + m, "decode_ws": m + nraw}
        detail = {"encode_wrapped_ms": enc_ms, "decode_ws_ms": dec_ms, "raw_bytes": nraw, "text_bytes": m,
                  "encode_wrapped_GBps_input": nraw / (enc_ms / 1e3) / 1e9,
                  "decode_ws_GBps_input": m / (dec_ms / 1e3) / 1e9,
                  "encode_wrapped_roofline_frac": (nraw + m) / (enc_ms / 1e3) / 1e9 / hbm,
                  "note": "decode_ws takes the verified line-structured fast path here (decode_lines_kernel; "
                          "the general mask + compaction kernels return at once); algorithmic bytes = text in + "
                          "bytes out"}
        dom, dom_ms = ("decode_ws", dec_ms) if dec_ms >= enc_ms else ("encode_wrapped", enc_ms)
        kname = {"decode_ws": "decode_lines_kernel", "encode_wrapped": "encode_wrap_kernel"}
        desc = ("f4: MIME round trip, 57*2^24 random bytes (seed 2) <-> 1.31 GB of 76-char CRLF lines: "
                "line-wrapped encode + whitespace-tolerant decode")
        launches = 4
    elif wl == "mime_irregular":
        # f4 general path: the same MIME text with every 50th line ending in
        # " \n" instead of CR LF (still valid under App. B, but not line-
        # structured): the fast path must detect it and give up, the mask
        # pass + fused compaction/decode produce the result.
        nraw = 57 * (1 << 24)
        raw = torch.empty(nraw, dtype=torch.uint8, device=dev)
        fill(raw, W.C3_SEED)
        m = b64.b64_encoded_len_wrapped(nraw, 76, True)
        w = b64.b64_encode_wrapped(raw, line_chars=76, crlf=True)
        rows = w.view(-1, 78)
        rows[::50, 76] = ord(" ")
        y = torch.empty(b64.b64_decoded_max_len(m), dtype=torch.uint8, device=dev)
        ws = torch.empty(b64.b64_decode_ws_workspace_bytes(m), dtype=torch.uint8, device=dev)
        dec_ms = timed(lambda: b64.b64_decode_ws_async(w, y, res, ws=ws), "decode_ws")
        ol, ep, st, _ = b64.unpack_result(res)
        assert (ol, ep, st) == (nraw, -1, 0) and torch.equal(y[:nraw], raw)
        assert int(ws[48:52].view(torch.int32).item()) == 0  # general path taken
        ms = dec_ms
        value = m / (ms / 1e3) / 1e9
        algo = {"decode_ws": m + nraw}
        detail = {"decode_ws_ms": dec_ms, "text_bytes": m, "raw_bytes": nraw,
                  "decode_ws_GBps_input": m / (dec_ms / 1e3) / 1e9,
                  "note": "general path: fast-path attempt (gives up), mask pass, fused compaction + decode"}
        dom, dom_ms = "decode_ws", dec_ms
        kname = {"decode_ws": "b64_decode_ws call, general path (all its kernels)"}
        desc = "f4: whitespace-tolerant decode of 1.31 GB of MIME text with irregular line ends (general path)"
        launches = 3
    elif wl == "sweep":
        # Fig. 9-shaped curve: GB/s vs input length, random
        # bytes of seed 6, n in {2^k, 4 <= k <= 30} and the Table V file
        # sizes.  Device time per call (CUDA events, mean of K
        # calls after W warm-ups); L2 is not flushed (small sizes are
        # latency-bound and L2-resident, as the paper's cache-hot loops).
        sizes = sorted({1 << e for e in range(4, 31)} | {1355, 1484, 2357, 12640, 141020, 329632})
        nmax = sizes[-1]
        raw = torch.empty(nmax, dtype=torch.uint8, device=dev)
        fill(raw, 6)
        t = torch.empty(b64.b64_encoded_len(nmax), dtype=torch.uint8, device=dev)
        y = torch.empty(nmax + 3, dtype=torch.uint8, device=dev)
        curve = []
        for n in sizes:
            xv = raw[:n]
            m = b64.b64_encoded_len(n)
            tv = t[:m]
            e_ms = timed(lambda: b64.b64_encode(xv, out=tv), flush_l2=False)
            d_ms = timed(lambda: b64.b64_decode_async(tv, y, res), flush_l2=False)
            assert b64.unpack_result(res)[2] == 0
            curve.append({"n": n, "encode_us": e_ms * 1e3, "decode_us": d_ms * 1e3,
                          "encode_GBps_input": n / (e_ms / 1e3) / 1e9,
                          "decode_GBps_input": m / (d_ms / 1e3) / 1e9})
        last = curve[-1]
        ms = last["encode_us"] / 1e3 + last["decode_us"] / 1e3
        value = (nmax + b64.b64_encoded_len(nmax)) / (ms / 1e3) / 1e9
        algo = {"encode": nmax + b64.b64_encoded_len(nmax), "decode": b64.b64_encoded_len(nmax) + nmax}
        dom, dom_ms = ("decode", last["decode_us"] / 1e3) if last["decode_us"] >= last["encode_us"] \
            else ("encode", last["encode_us"] / 1e3)
        detail = {"sweep": curve, "value_is": "encode + decode input GB/s at the largest size"}
        desc = "sweep: encode/decode GB/s vs length (2^4 .. 2^30 and Table V sizes), seed 6, L2 not flushed"
        launches = 2
    else:  # c4
        raw = torch.empty(W.C4_RAW, dtype=torch.uint8, device=dev)
        fill(raw, W.C4_SEED)
        m = W.C4_M
        t = torch.empty(m, dtype=torch.uint8, device=dev)
        b64.b64_encode(raw, out=t)
        pos, byt = W.c4_corruptions()
        td = t.clone()
        td[torch.from_numpy(pos).to(dev)] = torch.from_numpy(byt).to(dev)
        y = torch.empty(b64.b64_decoded_max_len(m), dtype=torch.uint8, device=dev)
        clean_ms = timed(lambda: b64.b64_decode_async(t, y, res), "clean")
        assert b64.unpack_result(res)[2] == 0
        dirty_ms = timed(lambda: b64.b64_decode_async(td, y, res), "dirty")
        assert b64.unpack_result(res)[1] == int(pos.min())
        ms = clean_ms + dirty_ms
        value = 2 * m / (ms / 1e3) / 1e9
        algo = {"decode": m + W.C4_RAW}
        detail = {"clean_ms": clean_ms, "dirty_ms": dirty_ms,
                  "clean_GBps_input": m / (clean_ms / 1e3) / 1e9, "dirty_GBps_input": m / (dirty_ms / 1e3) / 1e9}
        dom, dom_ms = "decode", clean_ms
        desc = "C4: 256 MiB valid text (seed 3) decoded clean and with 256 NA191 bytes (seed 4)"
        launches = 2
    clk = clocks.stop()
    ach = algo[dom] / (dom_ms / 1e3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": 1, "steps": K, "warmup": Wm,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic: counter-based SplitMix64 bytes (inputs/gen.py), generated on device",
            "config": {"workload": desc, "l2": "flushed before every step: 512 MiB write, then a 256 MiB read (drains the flush's dirty lines)"},
            "roofline": {"bound": "hbm", "kernel": kname.get(dom, f"{dom}_kernel"), "achieved": ach, "peak": hbm,
                         "unit": "GB/s", "frac": ach / hbm, "traffic": None, "peak_source": hbm_src},
            "gpu_launches": launches * K, "clocks": clk, "timing": samples, "detail": detail}
    if wl == "sweep":
        line["config"]["l2"] = "not flushed (cache-hot sweep)"
    print(json.dumps(line), flush=True)


# -------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import numpy as np

    from inputs import workloads as W
    from inputs.gen import splitmix_bytes

    seed = W.C5_SEED if args.workload == "c5" else W.C3_SEED
    smp = args.cpu_sample - args.cpu_sample % 3
    x = splitmix_bytes(seed, 0, smp)
    for _ in range(args.warmup):
        oracle_threads_bench(x, reps_min_s=0.0)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        gbs, cores, nbytes, el = oracle_threads_bench(x, reps_min_s=0.0)
        vals.append(gbs)
        secs += el
    value = statistics.mean(vals)
    model, ncpu, _ = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic: counter-based SplitMix64 bytes (inputs/gen.py)",
        "config": {"workload": f"{args.workload.upper()} sample: first {smp} bytes per step (oracle encode + decode)"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"{smp} bytes per step, split on 3-byte boundaries over {cores} threads",
                         "cpu_model": model, "cpu_count": ncpu},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`--gpus N` without a torchrun environment: launch N ranks (one per
    GPU) of this same command through torch.distributed.run on 127.0.0.1,
    so that `python bench.py --gpus 8` can never silently measure one GPU.
    Rank 0's JSON line is the only stdout line; the exit code is the
    launcher's."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c3", "c1", "c2", "c4", "despace", "despace_irregular", "mime", "mime_irregular", "sweep"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-bytes", type=int, default=3 << 28)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=48 << 20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cpu-sample-1core", type=int, default=12 << 20)
    ap.add_argument("--cpu-seconds-1core", type=float, default=5.0)
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.warmup < 3 and args.impl == "ours" and os.environ.get("B64_BENCH_ALLOW_FEW_WARMUP") != "1":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload in ("c1", "c2", "c4", "despace", "despace_irregular", "mime", "mime_irregular", "sweep"):
        if args.gpus != 1:
            raise SystemExit(f"--workload {args.workload} is a single-GPU parity config; use c5 or c3 for --gpus > 1")
        run_small_configs(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
