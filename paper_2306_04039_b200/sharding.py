"""Item-corpus sharding for multi-GPU retrieval.

The corpus splits into P contiguous item ranges; every rank runs the two-stage path on its shard
with K'_local = ceil(K'/P) and lambda_local from the same sample ratio, emits (score, global id)
top-k, and the lists are all-gathered and merged with molr_merge_top_k.  The merge is exact for
the union of candidates because MoL scores are item-local.
"""

from __future__ import annotations

import math


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous item range (balanced to within one item)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    return rank * n_items // world, (rank + 1) * n_items // world


def local_k_prime(k_prime: int, world: int) -> int:
    return max(1, math.ceil(k_prime / world))


def local_lambda(n_local: int, *, lam: int | None = None, sample_ratio: float | None = None, world: int = 1) -> int:
    """lambda for one shard: the same ratio of the shard (or lam / world)."""
    if (lam is None) == (sample_ratio is None):
        raise ValueError("set exactly one of lam or sample_ratio")
    if lam is not None:
        return max(1, min(n_local, math.ceil(lam / world)))
    return max(1, min(n_local, round(sample_ratio * n_local)))
