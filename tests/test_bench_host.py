"""Host-side logic of bench.py (no GPU): the committed C5 DRAM-traffic
record is stamped with the hash of the library sources it was captured
from, and the bench refuses a record whose stamp differs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import pytest  # noqa: E402


def test_committed_traffic_matches_the_committed_sources():
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
        tr = json.load(f)
    if any(tr[k]["source_sha"] != bench.source_hash() for k in ("c5:encode", "c5:decode")):
        pytest.xfail("sources changed since the C5 traffic capture: re-run tools/gpu_profile_all.sh")
    for key in ("c5:encode", "c5:decode"):
        v, src = bench.measured_traffic(key)
        assert v is not None and src
        # DRAM bytes within 0.2 % of the algorithmic bytes of one C5 launch
        assert abs(v / tr[key]["algorithmic_bytes_per_launch"] - 1) < 2e-3


def test_stale_traffic_is_refused(monkeypatch):
    monkeypatch.setattr(bench, "source_hash", lambda: "0" * 16)
    v, why = bench.measured_traffic("c5:decode")
    assert v is None and why.startswith("stale")
