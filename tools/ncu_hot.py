#!/usr/bin/env python
"""Per-instruction view of an ncu report's source page: the SASS lines with
their executed-instruction counts, stall samples and excess shared-memory
wavefronts (bank conflicts).  Usage: tools/ncu_hot.py REPORT [KERNEL_SUBSTR] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, cur, hdr, take = [], None, None, False
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        take = pat in r[1] and cur is None
        cur = r[1] if take else cur
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if take and hdr:
        rows.append(r)
ix = hdr
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in rows)
stall = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows)
print(f"{cur}\n{len(rows)} SASS lines, {tot} warp instructions, {stall} stall samples")
for n, r in enumerate(rows):
    r.append(n)
rows.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
for r in rows[:top]:
    print(f'{r[-1]:5d} {int(r[ix["Instructions Executed"]] or 0):>11} '
          f'st={int(r[ix["Warp Stall Sampling (All Samples)"]] or 0):>6} '
          f'xs={r[ix["L1 Wavefronts Shared Excessive"]]:>8}  {r[ix["Source"]].strip()[:70]}')
