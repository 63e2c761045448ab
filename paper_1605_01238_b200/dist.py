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


def nq_1d(n: int, p: int) -> np.ndarray:
    """#Q_i of the point grid of Remark 1 (reading R1) for n_EL >= p + 2: 2p+1 points for a row whose
    support touches no boundary span, p+1+2i for the boundary rows i <= p (and mirrored)."""
    i = np.arange(n)
    q = np.full(n, 2 * p + 1)
    left, right = i <= p, i >= n - 1 - p
    q[left] = p + 1 + 2 * i[left]
    q[right] = p + 1 + 2 * (n - 1 - i[right])
    return np.minimum(q, 2 * p + 1 + 2 * p)


def plane_cost(n: int, p: int) -> np.ndarray:
    """Relative cost of the planes of the slowest index: #I_i (nonzeros) plus a penalty proportional to
    #Q_i for the rows outside the uniform band [2p, n-1-2p] (boundary and near-boundary rows take the
    line kernels' table paths).  The penalty is fitted to per-rank step times of equal-nnz slabs
    (tools/time_slab.py): 0.4 for the z-line degrees, 0.1 for p >= 7 (ZHP)."""
    i = np.arange(n)
    gen = (i < 2 * p) | (i > n - 1 - 2 * p)
    beta = 0.4 if p <= 6 else 0.1
    return ni_1d(n, p) + beta * nq_1d(n, p) * gen


def slab_cuts(n: int, p: int, world: int, balance: str = "cost") -> list[int]:
    """Cut the planes [0, n) of the slowest index into `world` contiguous slabs of (nearly) equal
    cost (`balance="cost"`, plane_cost) or equal nnz (`balance="nnz"`: plane i carries
    #I_i * prod_{l<d} L_l nonzeros).  Each cut is the plane boundary nearest to its target."""
    w = plane_cost(n, p) if balance == "cost" else ni_1d(n, p)
    c = np.concatenate([[0], np.cumsum(w)])
    cuts = [0] * (world + 1)
    cuts[-1] = n
    for r in range(1, world):
        t = c[-1] * r / world
        k = int(np.searchsorted(c, t))
        if k > 0 and abs(c[k - 1] - t) <= abs(c[k] - t):
            k -= 1
        cuts[r] = k
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
