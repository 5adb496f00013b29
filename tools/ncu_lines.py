#!/usr/bin/env python
"""Per-CUDA-source-line totals of an ncu report (instructions executed, stall
samples), for one kernel: tools/ncu_lines.py REPORT KERNEL_SUBSTR [N]."""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
path = fn = None
hdr = None
rows = []
take = False
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        take = pat in fn
        continue
    if r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if take and hdr and r[0] and r[0] != "":
        try:
            ln = int(r[0])
        except ValueError:
            continue
        def num(k):
            v = r[hdr[k]]
            return int(v) if v.isdigit() else 0
        ex = num("Instructions Executed")
        st = num("Warp Stall Sampling (All Samples)")
        if ex or st:
            rows.append((path, ln, ex, st, r[1].strip()[:90]))
tot = sum(x[2] for x in rows)
tst = sum(x[3] for x in rows)
print(f"{tot} warp instructions, {tst} stall samples")
for p, ln, ex, st, src in sorted(rows, key=lambda x: -x[2])[:top]:
    print(f"{p}:{ln:<5} {ex:>10} {100*ex/tot:5.1f}%  st={st:>6}  {src}")
