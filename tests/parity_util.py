"""Parity helpers (test infrastructure): run the CUDA path through the C-ABI
binding and compare with the oracle on the same seeded inputs.

Tolerance (reading R6): per row, |gpu - oracle| <= 1e-12 * max_j |A_ij|
when the row's roundoff amplification kappa_i <= 1e4; otherwise
<= 1e-12 * max_j sum_q |term_ijq| (= kappa-scaled).  Indices are bit-exact.
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-12
KAPPA_STRICT = 1e4


def sample_rows(n, d, p, k_random=64, seed=0, extra=()):
    """Rows touching every boundary situation + seeded random interior rows."""
    rng = np.random.default_rng(seed)
    idx = set()
    edge = sorted(set([0, 1, min(p, n - 1), min(p + 1, n - 1), n // 2, max(n - p - 2, 0), max(n - 2, 0), n - 1]))
    grids = np.array(np.meshgrid(*([edge] * d), indexing="ij")).reshape(d, -1).T
    for m in grids:
        idx.add(int(sum(int(m[l]) * n ** l for l in range(d))))
    for r in rng.integers(0, n ** d, size=k_random):
        idx.add(int(r))
    for r in extra:
        idx.add(int(r))
    return np.array(sorted(idx), dtype=np.int64)


def line_rows(n, pick):
    """All rows (i1, i2, i3), i3 = 0..n-1, of the lines with i1, i2 in `pick` (3D, n per direction)."""
    out = [i1 + n * (i2 + n * i3) for i1 in pick for i2 in pick for i3 in range(n)]
    return np.array(sorted(out), dtype=np.int64)


def compare_rows(rows, g_ptr, g_col, g_val, o_ptr, o_col, o_val, kappa, scale, row_offset=0, strict=False):
    """rows: global ids; g_*: CSR of those rows gathered from the GPU (same order).
    strict=True additionally asserts that every row is in the strict regime
    (kappa_i <= 1e4, reading R6), which holds for p <= 6.
    Returns dict of statistics; raises AssertionError on index mismatch or
    value tolerance violation."""
    if strict:
        assert np.all(np.asarray(kappa) <= KAPPA_STRICT), f"kappa {np.max(kappa):.3g} above the strict regime"
    assert np.array_equal(np.diff(g_ptr), np.diff(o_ptr)), "row lengths differ"
    assert np.array_equal(g_col, o_col), "column indices differ"
    worst = 0.0
    worst_row = -1
    n_strict = 0
    for k in range(len(rows)):
        s = slice(o_ptr[k], o_ptr[k + 1])
        err = np.abs(g_val[s] - o_val[s]).max() if o_ptr[k + 1] > o_ptr[k] else 0.0
        if kappa[k] <= KAPPA_STRICT:
            ref = np.abs(o_val[s]).max()
            n_strict += 1
        else:
            ref = scale[k]
        rel = err / ref if ref > 0 else err
        if rel > worst:
            worst, worst_row = rel, int(rows[k])
        assert err <= RTOL * ref, f"row {rows[k]}: err {err:.3e} > {RTOL:g} * {ref:.3e} (kappa {kappa[k]:.3g})"
    return dict(worst_rel=worst, worst_row=worst_row, rows=len(rows), strict_rows=n_strict,
                max_kappa=float(np.max(kappa)) if len(kappa) else 0.0)


def gather_rows_device(rp, col, val, local_rows):
    """Gather CSR segments of local rows from device tensors (torch indexing, test side)."""
    import torch
    rp_h = rp.cpu().numpy() if hasattr(rp, "cpu") else rp
    base = rp_h[0]
    starts = rp_h[local_rows] - base
    ends = rp_h[local_rows + 1] - base
    lens = ends - starts
    ptr = np.zeros(len(local_rows) + 1, np.int64)
    np.cumsum(lens, out=ptr[1:])
    idx = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)]) if len(local_rows) else np.zeros(0, np.int64)
    it = torch.from_numpy(idx).to(val.device)
    gv = val.index_select(0, it).cpu().numpy()
    gc = col.index_select(0, it).cpu().numpy() if col is not None else None
    return ptr, gc, gv


_ORC_CACHE = {}


def oracle_rows_cached(key, make_oracle, mat, rows):
    """Oracle rows memoised per (case key, matrix) across the kernels a test is parametrised over."""
    k = (key, mat, len(rows), int(rows[0]) if len(rows) else -1, int(rows[-1]) if len(rows) else -1)
    if k not in _ORC_CACHE:
        if len(_ORC_CACHE) > 16:
            _ORC_CACHE.clear()
        _ORC_CACHE[k] = make_oracle().rows(mat, rows)
    return _ORC_CACHE[k]
