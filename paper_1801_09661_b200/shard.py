"""Row sharding over GPUs: rank r of N owns the contiguous global rows
[r n / N, (r+1) n / N); fold membership follows the global row index (R#19), so a rank passes its
first global row as `row_offset` to oem_gram_folds. Pure host arithmetic (no method math)."""
from __future__ import annotations


def row_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Global rows [r0, r1) owned by `rank` out of `world`."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * n // world, (rank + 1) * n // world


def fold_counts(n_local: int, row_offset: int, K: int) -> list[int]:
    """Rows of this shard in each fold k, fold(i) = (row_offset + i) mod K (mirrors the count
    computation in oem_gram_folds)."""
    out = []
    for k in range(K):
        first = (k - row_offset) % K
        out.append((n_local - first + K - 1) // K if n_local > first else 0)
    return out
