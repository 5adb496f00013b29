"""The seeded input generator (inputs/gen.py) and the config recipes."""
import numpy as np

from inputs import gen, workloads


def test_splitmix64_reference_values():
    # SplitMix64 seeded with 0: first outputs (Steele, Lea, Flood 2014 reference stream)
    w = gen.splitmix_words(0, 0, 3)
    assert [int(x) for x in w] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_bytes_are_little_endian_words():
    w = gen.splitmix_words(5, 0, 4)
    b = gen.splitmix_bytes(5, 0, 32)
    for k in range(4):
        assert int.from_bytes(b[8 * k: 8 * k + 8].tobytes(), "little") == int(w[k])


def test_counter_based_shards_match():
    full = gen.splitmix_bytes(2, 0, 1000)
    for b, e in [(0, 1), (3, 17), (8, 16), (999, 1000), (123, 777)]:
        assert np.array_equal(gen.splitmix_bytes(2, b, e), full[b:e])
    hi = (1 << 33) + 5
    assert np.array_equal(gen.splitmix_bytes(9, hi, hi + 20)[3:], gen.splitmix_bytes(9, hi + 3, hi + 20))


def test_na191():
    assert workloads.NA191.size == 191
    assert ord("=") not in workloads.NA191.tolist()
    assert ord("A") not in workloads.NA191.tolist()


def test_c2_lengths_shape():
    lens, _ = workloads.c2_lengths()
    assert lens.size == 10_000 and lens.min() >= 100 and lens.max() <= 65536
    assert 2000 < np.median(lens) < 3200
    assert 9e7 < lens.sum() < 1.1e8


def test_c4_corruptions():
    pos, byt = workloads.c4_corruptions()
    assert pos.size == 256 and np.unique(pos).size == 256
    assert set(byt.tolist()) <= set(workloads.NA191.tolist())
