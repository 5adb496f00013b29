#!/usr/bin/env python
"""profiles/ncu_traffic.json from an ncu metrics CSV of the C5 bench step
(dram__bytes_read.sum + dram__bytes_write.sum per launch of encode_kernel /
decode_kernel), stamped with the sha of the library sources it was captured
from (bench.source_hash): bench.py reports roofline.traffic only when the
stamp matches the sources it runs.

  python tools/traffic_json.py CSV [TAG]     # run on the GPU box after the capture
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from inputs import workloads as W  # noqa: E402


def main():
    path = sys.argv[1]
    tag = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(path)
    lines = [ln for ln in open(path) if ln.startswith('"')]
    per = {}
    for r in csv.DictReader(io.StringIO("".join(lines))):
        k = r["Kernel Name"]
        kind = "encode" if "encode_kernel" in k else "decode" if "decode_kernel" in k else None
        if kind is None:
            continue
        d = per.setdefault((r["ID"], kind), {})
        d[r["Metric Name"]] = float(r["Metric Value"])
    n = W.C5_N
    m = 4 * ((n + 2) // 3)
    algo = n + m
    out = {}
    for kind in ("encode", "decode"):
        rows = [v for (i, k), v in sorted(per.items()) if k == kind]
        if not rows:
            continue
        v = rows[-1]
        tot = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
        out[f"c5:{kind}"] = {
            "dram_bytes_per_launch": tot, "dram_read": v["dram__bytes_read.sum"],
            "dram_write": v["dram__bytes_write.sum"], "algorithmic_bytes_per_launch": algo,
            "ratio": tot / algo, "ncu_duration_ns": v.get("gpu__time_duration.sum"),
            "source_sha": bench.source_hash(),
            "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                      f"(single pass) on `python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu`, {tag}",
        }
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
