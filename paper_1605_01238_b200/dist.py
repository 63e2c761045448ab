"""Multi-GPU host logic: one process per GPU, rows split into
contiguous slabs of the slowest index i_d, each rank forms its own CSR block.

Rows are independent, so the only exchange is the all-gather of
one int64 nnz per rank; its exclusive scan is the rank's row_ptr base
(wq_pattern's nnz_base).  Integer host logic only (no arithmetic of the WQ
method): #I_i = min(n-1, i+p) - max(0, i-p) + 1.
"""
from __future__ import annotations

import numpy as np


def ni_1d(n: int, p: int) -> np.ndarray:
    i = np.arange(n)
    return np.minimum(n - 1, i + p) - np.maximum(0, i - p) + 1


def slab_cuts(n: int, p: int, world: int) -> list[int]:
    """Cut the planes [0, n) of the slowest index into `world` contiguous slabs
    with (nearly) equal nnz: plane i carries #I_i * prod_{l<d} L_l nonzeros."""
    c = np.concatenate([[0], np.cumsum(ni_1d(n, p))])
    cuts = [int(np.searchsorted(c, c[-1] * r / world)) for r in range(world + 1)]
    cuts[0], cuts[-1] = 0, n
    for r in range(1, world + 1):  # keep slabs non-empty when n >= world
        cuts[r] = max(cuts[r], min(cuts[r - 1] + 1, n))
    return cuts


def slab_nnz(ns, p: int, b: int, e: int) -> int:
    """nnz of the rows whose slowest index lies in [b, e): d = len(ns)."""
    L = [int(ni_1d(n, p).sum()) for n in ns]
    nd = ni_1d(ns[-1], p)
    per_plane = int(np.prod(L[:-1])) if len(L) > 1 else 1
    return int(nd[b:e].sum()) * per_plane


def nnz_base(nnz_local: int, dist, device=None) -> int:
    """Exclusive scan of the all-gathered per-rank nnz (the only collective)."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    mine = torch.tensor([int(nnz_local)], dtype=torch.int64, device=device)
    allv = torch.zeros(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allv, mine)
    return int(allv[:rank].sum().item())
