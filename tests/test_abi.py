"""C ABI checks that need no GPU: the library loads, exports every symbol
include/b64gpu.h declares, and its pure-host entry points behave."""
import ctypes
import os
import re

import pytest

import paper_1704_00605_b200 as b64

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "b64gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(b64_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_binding_exports():
    assert sorted(b64.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(b64.lib_path())
    for name in _declared():
        assert hasattr(lib, name), name


def test_library_targets_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {b64.lib_path()} 2>&1").read()
    assert "sm_100a" in out


def test_sizes():
    for n in range(0, 50):
        assert b64.b64_encoded_len(n) == 4 * ((n + 2) // 3)
        assert b64.b64_decoded_max_len(n) == 3 * (n // 4)
    assert b64.b64_encoded_len(-1) == -1
    assert b64.b64_encoded_len(1 << 35) == 45_812_984_492  # config 5 text length


def test_status_strings():
    for c in (0, 1, 2, -1, -2, -3):
        assert b64.b64_status_str(c)
    assert b64.b64_status_str(99) == "unknown status"


def test_argument_errors_launch_nothing():
    lib = b64.load_library()
    assert lib.b64_encode(None, -1, None, None) == b64.B64_ERR_ARG
    assert lib.b64_encode(None, 5, None, None) == b64.B64_ERR_ARG
    assert lib.b64_decode(None, -1, None, None, None, None) == b64.B64_ERR_ARG
    assert lib.b64_decode_shard_async(None, 5, 0, None, None, None) == b64.B64_ERR_ARG
    assert lib.b64_encode_batch(None, None, 1, 0, None, None, None, 0, None) == b64.B64_ERR_ARG
    assert lib.b64_encode(None, 0, None, None) == 0  # empty input: nothing to do


@pytest.mark.parametrize("total", [0, 1, 2, 3, 4, 5, 100, 1001, (1 << 35), (1 << 35) + 7, 45_812_984_492])
@pytest.mark.parametrize("unit", [3, 4])
def test_shard_partition(total, unit):
    """Shards tile [0, total) in order, start on unit boundaries, and only the
    last one may hold a partial unit."""
    for world in (1, 2, 3, 4, 7, 8):
        prev = 0
        for r in range(world):
            b, e = b64.b64_shard(total, unit, world, r)
            assert b == prev and b <= e <= total
            assert b % unit == 0
            if r < world - 1:
                assert e % unit == 0 or e == total
            prev = e
        assert prev == total


def test_shard_config5_balance():
    # 2^35 bytes = 11,453,246,123 groups over 8 ranks: 1,431,655,765 or ...766 groups each
    sizes = []
    for r in range(8):
        b, e = b64.b64_shard(1 << 35, 3, 8, r)
        sizes.append((e - b + 2) // 3)
    assert set(sizes) <= {1_431_655_765, 1_431_655_766}
    assert sum(sizes) == 11_453_246_123


def test_wrapped_len_matches_oracle_and_rejects_bad_lines():
    import oracle

    for n in [0, 1, 2, 3, 56, 57, 58, 1000, 1 << 30]:
        for L in (4, 64, 76, 16384):
            for crlf in (0, 1):
                for fl in (0, 2):
                    assert b64.b64_encoded_len_wrapped(n, L, bool(crlf), fl) == \
                        oracle._load().oracle_encoded_len_wrapped(n, L, crlf, fl)
    for bad in (0, 3, 6, 77, 16388):
        assert b64.b64_encoded_len_wrapped(10, bad, True, 0) == b64.B64_ERR_ARG


def test_shard_key_and_combine_host():
    """The multi-GPU exchange arithmetic of the C ABI (pure host): the key
    packs a global offset with its status, the MIN over shards picks the
    first error, and the combine follows Alg 2's output rule."""
    INT64_MAX = b64.INT64_MAX
    assert b64.b64_shard_key(0, -1, 123) == INT64_MAX
    assert b64.b64_shard_key(1, 5, 100) == (105 << 2) | 1
    assert b64.b64_shard_key(2, 8, 0) == (8 << 2) | 2
    assert b64.b64_shard_key(3, 10, 4) == (14 << 2) | 3
    # clean: lengths summed, pad count from the total length
    assert b64.b64_combine_shards(INT64_MAX, [30, 30, 28], 120) == (0, -1, 88, 2)
    assert b64.b64_combine_shards(INT64_MAX, [3], 6) == (0, -1, 3, 0)  # m % 4 != 0 (NOPAD tail)
    # errors: the MIN key wins; out_len = 3 * floor(err / 4) for every status
    keys = [b64.b64_shard_key(1, 7, 40), b64.b64_shard_key(3, 2, 80), INT64_MAX]
    assert b64.b64_combine_shards(min(keys), [30, 30, 0], 120) == (1, 47, 33, 0)
    assert b64.b64_combine_shards(b64.b64_shard_key(2, 4, 116), [87, 0], 121) == (2, 120, 90, 0)
    assert b64.b64_combine_shards(b64.b64_shard_key(3, 3, 116), [87, 0], 120) == (3, 119, 87, 0)
    lib = b64.load_library()
    assert lib.b64_combine_shards(0, None, 1, 4, None) == b64.B64_ERR_ARG
    assert lib.b64_combine_shards_async(None, None, 0, 4, None, None) == b64.B64_ERR_ARG
    assert lib.b64_decode_scratch_async(None, 4, None, 0, None, None, None) == b64.B64_ERR_ARG


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with the CUDA library absent, the binding raises on
    the first call instead of computing anything (no oracle on the product
    path)."""
    import subprocess
    import sys

    code = ("import paper_1704_00605_b200 as b\n"
            "try:\n    b.load_library()\nexcept RuntimeError as e:\n    print('RAISED', e)\n")
    env = dict(os.environ, B64GPU_LIB=str(tmp_path / "absent.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=120)
    assert r.returncode == 0 and "RAISED" in r.stdout and "absent.so" in r.stdout, r.stdout + r.stderr
    # the package never imports the oracle
    pkg = os.path.join(ROOT, "paper_1704_00605_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            with open(os.path.join(pkg, f)) as fh:
                assert "oracle" not in fh.read().replace("# oracle", ""), f
