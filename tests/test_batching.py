"""CPU: batching / device-split planners."""
import pytest

from paper_1504_04343_b200 import ConfigError, ConvDesc
from paper_1504_04343_b200.batching import footprint, plan_partitions, proportional_split, shard_of


def test_plan_partitions_spec_examples():
    p = plan_partitions(256, 16, 4)
    assert p.partition_sizes == (64, 64, 64, 64) and p.threads_per_partition == (4, 4, 4, 4)
    p = plan_partitions(256, 16, 1)
    assert p.partition_sizes == (256,) and p.threads_per_partition == (16,)
    assert plan_partitions(7, 4, 2).partition_sizes == (4, 3)


def test_plan_partitions_remainders_and_errors():
    p = plan_partitions(10, 7, 3)
    assert p.partition_sizes == (4, 3, 3) and p.threads_per_partition == (3, 2, 2)
    for bad in (0, 11):
        with pytest.raises(ConfigError):
            plan_partitions(10, 16, bad)


def test_proportional_split():
    s = proportional_split([1.0, 2.0], 3)              # CPU gets 1/3
    assert s.fractions[0] == pytest.approx(1 / 3) and s.counts == (1, 2)
    assert proportional_split([5.0], 9).counts == (9,)
    assert proportional_split([2.0, 2.0], 7).counts == (4, 3)
    s = proportional_split([1.0] * 8, 2048)
    assert s.counts == (256,) * 8 and sum(s.counts) == 2048
    assert proportional_split([3.0, 1.0, 1.0], 10).counts == (6, 2, 2)
    assert proportional_split([10.0, 20.0], 30).fractions == proportional_split([1.0, 2.0], 30).fractions
    with pytest.raises(ConfigError):
        proportional_split([], 4)


def test_shards_cover_batch():
    for world in (1, 2, 3, 4, 8):
        cover = []
        for r in range(world):
            f, c = shard_of(2048 + 5, world, r)
            cover.extend(range(f, f + c))
        assert cover == list(range(2053))


def test_footprint_linear_and_ordered():
    d = ConvDesc(27, 5, 96, 256, 1, 1, 2)
    for t in (1, 2, 3):
        assert footprint(d, t, 256) == 256 * footprint(d, t, 1)
    assert footprint(d, 3, 8) < footprint(d, 2, 8) < footprint(d, 1, 8)
    d1 = ConvDesc(13, 1, 64, 64, 1)
    assert len({footprint(d1, t, 4) for t in (1, 2, 3)}) == 1     # k = 1
