"""Host-side partition of the TNRD inference pass over ranks.

Pure index arithmetic, shared by bench.py and the multi-process tests.  The
C ABI's loopback slab path (tnrd_denoise_slabs_loopback) uses the same split
rule (rows [H*k/n, H*(k+1)/n)).

  * batch sharding (BASELINE.json configs[3]): independent images, no exchange;
  * row slabs (configs[4]): each stage needs u within 2r = ksize - 1 rows of the
    slab (reading C18: v = k*u reaches r rows, kbar*phi(v) another r), so every
    rank receives `halo_rows(ksize)` rows from each neighbour before each stage.
"""
from __future__ import annotations

from typing import Tuple


def batch_shard(B: int, rank: int, world: int) -> Tuple[int, int]:
    """Images [b0, b1) of `rank`; contiguous, sizes differ by at most one."""
    if not (0 <= rank < world) or B < 1:
        raise ValueError("bad shard request")
    return B * rank // world, B * (rank + 1) // world


def slab_rows(H: int, rank: int, world: int) -> Tuple[int, int]:
    """Rows [r0, r1) owned by `rank` in the row-slab partition of an H-row image."""
    if not (0 <= rank < world) or H < 1:
        raise ValueError("bad slab request")
    return H * rank // world, H * (rank + 1) // world


def halo_rows(ksize: int) -> int:
    """Rows of u a stage needs beyond a slab edge: 2r = ksize - 1."""
    if ksize < 1 or ksize % 2 == 0:
        raise ValueError("ksize must be odd")
    return ksize - 1


def neighbours(rank: int, world: int) -> Tuple[int, int]:
    """(up, down) neighbour ranks in the slab chain, -1 where the image ends."""
    return (rank - 1 if rank > 0 else -1), (rank + 1 if rank + 1 < world else -1)
