"""Batch partitioning and device split (host-side mirror of the SPEC's batching
and scheduler modules; on B200 the partitions are per-GPU batch shards).

* ``plan_partitions`` -- SPEC.md:304-312 (PartitionPlan):
  p near-equal partitions of b images, threads divided among partitions with
  remainders to the lowest indices.
* ``proportional_split`` -- SPEC.md:366-374: each device takes a fraction of
  the batch proportional to its FLOPS, counts rounded by largest remainder.
  On one 8xB200 box every device has the same FLOPS, so this is the equal
  split used by the data-parallel driver (``stack.py``).
* ``footprint`` -- SPEC.md:322-330: exact lowered-matrix bytes, linear in the
  partition size.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from . import ConfigError, ConvDesc

__all__ = ["PartitionPlan", "plan_partitions", "SplitPlan", "proportional_split", "footprint",
           "shard_of"]


@dataclass(frozen=True)
class PartitionPlan:
    partitions: int
    partition_sizes: tuple[int, ...]
    threads_per_partition: tuple[int, ...]


def plan_partitions(b: int, total_threads: int, p: int) -> PartitionPlan:
    """1 <= p <= min(b, total_threads), sizes differ by <= 1."""
    if p < 1 or p > min(b, total_threads):
        raise ConfigError(f"partition count {p} out of range [1, min(b={b}, threads={total_threads})]")
    base, rem = divmod(b, p)
    sizes = tuple(base + (1 if i < rem else 0) for i in range(p))
    tb, tr = divmod(total_threads, p)
    threads = tuple(tb + (1 if i < tr else 0) for i in range(p))
    return PartitionPlan(p, sizes, threads)


@dataclass(frozen=True)
class SplitPlan:
    fractions: tuple[float, ...]
    counts: tuple[int, ...]


def proportional_split(flops: list[float], b: int) -> SplitPlan:
    """fraction_i = flops_i / sum(flops); largest-remainder rounding."""
    if not flops:
        raise ConfigError("proportional_split needs at least one device")
    if any(f <= 0 for f in flops):
        raise ConfigError("device flops must be > 0")
    tot = float(sum(flops))
    fr = [f / tot for f in flops]
    raw = [x * b for x in fr]
    counts = [math.floor(r) for r in raw]
    left = b - sum(counts)
    order = sorted(range(len(raw)), key=lambda i: (-(raw[i] - counts[i]), i))
    for i in order[:left]:
        counts[i] += 1
    return SplitPlan(tuple(fr), tuple(counts))


def shard_of(b: int, world: int, rank: int) -> tuple[int, int]:
    """(first image, count) of rank's contiguous shard under the equal split."""
    counts = proportional_split([1.0] * world, b).counts
    first = sum(counts[:rank])
    return first, counts[rank]


def footprint(desc: ConvDesc, lowering: int, partition_size: int) -> int:
    """Exact Dhat bytes of one partition, internal layout."""
    n, k, d, s, p = desc.n, desc.k, desc.d, desc.stride, desc.pad
    m = (n + 2 * p - k) // s + 1
    R = s * (m - 1) + k
    rows = {1: m * m, 2: R * m, 3: R * R}[lowering] * partition_size
    cols = {1: k * k * d, 2: k * d, 3: d}[lowering]
    return 4 * rows * cols
