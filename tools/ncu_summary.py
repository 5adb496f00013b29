#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) into a JSON + text block for
profiles/: DRAM bytes and throughput, issue / pipe utilisation, shared-memory
wavefronts and conflicts, warp-stall reasons and per-opcode instruction mix of
the hot loop.  Usage: tools/ncu_summary.py REPORT [ALGO_BYTES] > out.txt"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    algo = float(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    outs = [summarize(rep, hdr, units, vals, algo) for vals in rows[2:]]
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    # the source page holds one table per profiled kernel, in launch order
    tables, cur = [], None
    for r in src:
        if r and r[0] == "Kernel Name":
            cur = {"rows": []}
            tables.append(cur)
        elif r and r[0] == "Address" and cur is not None:
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur:
            cur["rows"].append(r)
    for out, t in zip(outs, tables):
        add_mix(out, t)
    json.dump(outs if len(outs) > 1 else outs[0], sys.stdout, indent=1)
    print()


def add_mix(out, t):
    ix = {k: i for i, k in enumerate(t["hdr"])}
    mix = Counter()
    total = 0
    for r in t["rows"]:
        try:
            ie = int(r[ix["Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        total += ie
        toks = r[ix["Source"]].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        mix[op.split(".")[0]] += ie
    out["warp_instructions"] = total
    out["opcode_mix_top"] = dict(mix.most_common(16))


def summarize(rep, hdr, units, vals, algo):
    kernel = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    out = {"report": rep, "kernel": kernel}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out[k] = {"value": vals[i], "unit": units[i]}
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h] = float(vals[i])
            except ValueError:
                pass
    out["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    try:
        rd = float(out["dram__bytes_read.sum"]["value"]) * (1e9 if out["dram__bytes_read.sum"]["unit"] == "Gbyte" else 1e6 if out["dram__bytes_read.sum"]["unit"] == "Mbyte" else 1)
        wr = float(out["dram__bytes_write.sum"]["value"]) * (1e9 if out["dram__bytes_write.sum"]["unit"] == "Gbyte" else 1e6 if out["dram__bytes_write.sum"]["unit"] == "Mbyte" else 1)
        out["dram_bytes_per_launch"] = rd + wr
        if algo:
            out["algorithmic_bytes_per_launch"] = algo
            out["traffic_over_algorithmic"] = (rd + wr) / algo
    except (KeyError, ValueError):
        pass
    return out


if __name__ == "__main__":
    main()
