"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (one plan, AUTO kernel; C5 as the 8 slabs of the multi-GPU split run one
after the other on one GPU):
  - index arrays (row_ptr, col) compared IN FULL, streamed in plane chunks
    against the oracle's pattern generator (orc_pattern_rows, by definition of
    I_i), bit-exact;
  - stiffness values on EVERY row through the zero-row-sum invariant of the WQ
    stiffness matrix (pin P5; a property that holds at any size);
  - values on sampled rows (every boundary situation + seeded random rows; for
    C5 the corner blocks and rows on both sides of every slab seam) against the
    oracle's direct sums, per-row tolerance of reading R6.
"""
import numpy as np
import pytest

import paper_1605_01238_b200 as wq
from oracle import MASS, STIFFNESS, Oracle
from parity_util import compare_rows, gather_rows_device, sample_rows
from wqinputs import baseline_config

pytestmark = pytest.mark.gpu

CHUNK_NNZ = 1 << 28  # entries per streamed comparison chunk (1 GiB of int32 columns)


def _torch():
    import torch
    return torch


def check_pattern_in_full(o, rp_dev, col_dev, row_begin, n_rows):
    """Stream the device row_ptr / col of the global rows [row_begin, row_begin + n_rows) (row_ptr
    holding global offsets) against the oracle's pattern of the same rows, in chunks of whole
    planes; bit-exact.  Returns the number of columns compared."""
    torch = _torch()
    rp = rp_dev.cpu().numpy()
    assert rp.size == n_rows + 1
    n1n2 = o.n[0] * (o.n[1] if o.d > 1 else 1)
    r, checked = 0, 0
    while r < n_rows:
        r_hi = min(r + n1n2, n_rows)
        while r_hi < n_rows and rp[min(r_hi + n1n2, n_rows)] - rp[r] <= CHUNK_NNZ:
            r_hi = min(r_hi + n1n2, n_rows)
        orp, ocol = o.pattern_rows(row_begin + r, row_begin + r_hi)
        assert np.array_equal(rp[r:r_hi + 1], orp), f"row_ptr differs in rows [{row_begin + r}, {row_begin + r_hi})"
        lo, hi = int(rp[r] - rp[0]), int(rp[r_hi] - rp[0])
        ref = torch.from_numpy(ocol).to(col_dev.device)
        assert torch.equal(col_dev[lo:hi], ref), f"columns differ in rows [{row_begin + r}, {row_begin + r_hi})"
        checked += hi - lo
        r = r_hi
    return checked


def stiffness_row_sums_every_row(rp_dev, val_dev, factor):
    """Invariant of the WQ stiffness matrix that holds at any size and for any geometry (pin P5,
    tests/test_oracle_pins.py::test_stiffness_row_sums_zero): sum_{j in I_i} D^b B_j = [b = 0] at
    every point of Q_i, so every row of S~ sums to zero up to rounding.  Checked on EVERY row of the
    device CSR: |sum_j s_ij| <= factor * #I_i * max_j |s_ij| (each entry carries at most the parity
    tolerance of reading R6 relative to the row's largest entry; the callers pass 2e-14 for p <= 6
    and 1e-12 for p >= 8, 35-75x above the worst ratios measured on the BASELINE configs:
    3e-17 .. 3e-16 for p <= 6, 1.9e-15 at p = 8, 1.3e-14 at p = 10, profiles/r02_rowsum_every_row.log).
    Returns the worst ratio |sum| / (#I_i max|s_ij|)."""
    torch = _torch()
    n_rows = rp_dev.numel() - 1
    rp = rp_dev - rp_dev[0]
    worst, r = 0.0, 0
    budget = 1 << 27
    rp_h = rp.cpu().numpy()
    while r < n_rows:
        r_hi = int(np.searchsorted(rp_h, rp_h[r] + budget, side="right")) - 1
        r_hi = min(max(r_hi, r + 1), n_rows)
        lens = rp[r + 1:r_hi + 1] - rp[r:r_hi]
        idx = torch.repeat_interleave(torch.arange(r_hi - r, device=val_dev.device), lens)
        v = val_dev[int(rp_h[r]):int(rp_h[r_hi])]
        ssum = torch.zeros(r_hi - r, dtype=torch.float64, device=v.device).index_add_(0, idx, v)
        smax = torch.zeros(r_hi - r, dtype=torch.float64, device=v.device).scatter_reduce_(0, idx, v.abs(), "amax")
        assert bool((smax > 0).all()), "a row of zeros"
        ratio = ssum.abs() / (lens.double() * smax)
        w = float(ratio.max())
        bad = int((ratio > factor).sum())
        assert bad == 0, f"{bad} rows in [{r}, {r_hi}) break the zero row sum (worst ratio {w:.3e}, row {r + int(ratio.argmax())})"
        worst = max(worst, w)
        del idx, v, ssum, smax, ratio
        r = r_hi
    return worst


@pytest.mark.parametrize("name,p,k_random", [("C2", None, 96), ("C3", None, 24), ("C4", 2, 48), ("C4", 3, 48),
                                             ("C4", 4, 32), ("C4", 6, 12), ("C4", 8, 4), ("C4", 10, 2)])
def test_baseline_full_size(name, p, k_random):
    """BASELINE configs at full size, AUTO kernel (the bench path): row_ptr and col in full,
    sampled rows' values vs the oracle (strict regime asserted for p <= 6)."""
    torch = _torch()
    cfg = baseline_config(name, p)
    ks, ctrl = cfg.knots(), cfg.ctrl()
    mats = (STIFFNESS, MASS) if "mass" in cfg.matrices else (STIFFNESS,)
    n = cfg.n_el + cfg.p
    rows = sample_rows(n, 3, cfg.p, k_random=k_random, seed=1)
    if cfg.p >= 8:
        rows = rows[:: max(1, len(rows) // 24)]
    o = Oracle(cfg.p, ks, ctrl)
    plan = wq.Plan(cfg.p, ks, ctrl=ctrl, need_mass="mass" in cfg.matrices, need_stiffness=True)
    info = plan.info
    assert info["nnz_local"] == cfg.exact_nnz()
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp)
    for mat in mats:
        wq.wq_assemble(plan.h, mat, val, col)
        wq.wq_check(plan.h)
        torch.cuda.synchronize()
        assert int(rp[-1]) == cfg.exact_nnz()
        if mat == STIFFNESS:
            assert check_pattern_in_full(o, rp, col, 0, info["n_rows_local"]) == cfg.exact_nnz()
            print(name, p, "worst |row sum| / (#I max|s|) over every row:",
                  stiffness_row_sums_every_row(rp, val, 2e-14 if cfg.p <= 6 else 1e-12))
        if mat == MASS and cfg.d == 3 and info["nnz_local"] <= (1 << 28):
            # every row of the mass matrix through its row sum against the oracle's tables
            lens = rp[1:] - rp[:-1]
            idx = torch.repeat_interleave(torch.arange(lens.numel(), device=val.device), lens)
            ssum = torch.zeros(lens.numel(), dtype=torch.float64, device=val.device).index_add_(0, idx, val)
            smax = torch.zeros(lens.numel(), dtype=torch.float64, device=val.device).scatter_reduce_(0, idx, val.abs(), "amax")
            want = mass_row_sums_oracle(o).astype(np.float64)
            ratio = np.abs(ssum.cpu().numpy() - want) / (lens.cpu().numpy() * smax.cpu().numpy())
            print(name, p, "mass worst |row sum - oracle| / (#I max|m|) over every row:", float(ratio.max()))
            assert float(ratio.max()) <= 2e-13
            del idx
        ptr, oc, ov, kappa, scale = o.rows(mat, rows)
        gptr, gc, gv = gather_rows_device(rp, col, val, rows)
        st = compare_rows(rows, gptr, gc, gv, ptr, oc, ov, kappa, scale, strict=cfg.p <= 6)
        print(name, p, mat, wq.KERNEL_NAMES[info["kernel"][mat]], st)
    plan.close()
    del rp, col, val
    torch.cuda.empty_cache()


def test_C5_slabs():
    """BASELINE configs[4] (C5: 3D p=4, 256^3 elements, quarter annulus, 12.49e9 nnz) as the 8
    x_3-slabs of the multi-GPU run, one after the other on one GPU: every slab plan
    takes the z-line kernel; the per-slab blocks chain through nnz_base to the whole matrix
    (row_ptr / col in full against the oracle pattern); values of the 8 corner blocks ((p+2)^3 rows
    each) and of rows on both planes of every seam against the oracle."""
    torch = _torch()
    from paper_1605_01238_b200.dist import slab_cuts
    cfg = baseline_config("C5")
    ks, ctrl = cfg.knots(), cfg.ctrl()
    p, n = cfg.p, cfg.n_el + cfg.p
    o = Oracle(p, ks, ctrl)
    cuts = slab_cuts(n, p, 8)
    rng = np.random.default_rng(5)
    corner = [a for a in range(p + 2)] + [n - 1 - a for a in range(p + 2)]
    crow = {i1 + n * (i2 + n * i3) for i1 in corner for i2 in corner for i3 in corner}
    seam = set()
    for c in cuts[1:-1]:
        for i3 in (c - 1, c):
            for i1, i2 in rng.integers(0, n, size=(48, 2)):
                seam.add(int(i1) + n * (int(i2) + n * i3))
    want = np.array(sorted(crow | seam), dtype=np.int64)
    base = 0
    total_checked = 0
    for s in range(8):
        plan = wq.Plan(p, ks, ctrl=ctrl, slab=(cuts[s], cuts[s + 1]), need_mass=False, need_stiffness=True)
        info = plan.info
        assert info["kernel"][1] == wq.WQ_KERNEL_ZLINE
        rp, col, val = plan.form(STIFFNESS, nnz_base=base)
        torch.cuda.synchronize()
        r0, nr = info["row_begin"], info["n_rows_local"]
        total_checked += check_pattern_in_full(o, rp, col, r0, nr)
        print("C5 slab", s, "worst |row sum| / (#I max|s|) over every row:", stiffness_row_sums_every_row(rp, val, 2e-14))
        mine = want[(want >= r0) & (want < r0 + nr)]
        ptr, oc, ov, kappa, scale = o.rows(STIFFNESS, mine)
        gptr, gc, gv = gather_rows_device(rp - base, col, val, mine - r0)
        compare_rows(mine, gptr, gc, gv, ptr, oc, ov, kappa, scale, strict=True)
        assert int(rp[0]) == base
        base += info["nnz_local"]
        assert int(rp[-1]) == base
        plan.close()
        del rp, col, val
        torch.cuda.empty_cache()
    assert base == cfg.exact_nnz() == total_checked


def mass_row_sums_oracle(o):
    """sum_{j in I_i} m~_ij for every row i from the oracle's own tables, by the partition of unity
    on Q_i (sum_{j in I_i} B_j = 1 at every point of Q_i; Eq. massquadrature):
    sum_q w^(0,0)_{1,i1,q1} w^(0,0)_{2,i2,q2} w^(0,0)_{3,i3,q3} c(x_q), in long double.
    Returns [n_3][n_2][n_1] flattened (row index i_1 fastest)."""
    Wd = []
    for l in range(3):
        D = o.direction(l)
        W = np.zeros((o.n[l], o.nq[l]), dtype=np.longdouble)
        for i in range(o.n[l]):
            lo, ln = int(D["qlo"][i]), int(D["qlen"][i])
            W[i, lo:lo + ln] = D["w"][i, 0, :ln]
        Wd.append(W)
    ref, det, st = o.coef_box([0, 0, 0], list(o.nq))
    assert st == 0
    c = ref[:, 0].reshape(o.nq[2], o.nq[1], o.nq[0]).astype(np.longdouble)   # [q3][q2][q1]
    t = np.einsum("ia,cba->cbi", Wd[0], c)
    t = np.einsum("jb,cbi->cji", Wd[1], t)
    t = np.einsum("kc,cji->kji", Wd[2], t)
    return t.reshape(-1)


@pytest.mark.parametrize("n_el,p", [(20, p) for p in range(1, 11)] + [(40, 3), (40, 6), (40, 10)])
def test_mass_shapes_every_row(n_el, p):
    """the paper's timing shapes (3D mass, 20^3 and 40^3 elements, Fig. 3),
    AUTO kernel (tile for p <= 3, ZHP above): index arrays in full against the oracle pattern;
    values of sampled rows against the oracle's direct sums; and the values of EVERY row through
    their row sum against the oracle's weights and coefficient field (mass_row_sums_oracle)."""
    torch = _torch()
    from wqinputs import Config
    cfg = Config(f"M{n_el}p{p}", 3, p, n_el, "grid", 0.1, ("mass",))
    ks, ctrl = cfg.knots(), cfg.ctrl()
    o = Oracle(p, ks, ctrl)
    plan = wq.Plan(p, ks, ctrl=ctrl, need_mass=True, need_stiffness=False)
    info = plan.info
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp)
    wq.wq_assemble(plan.h, MASS, val, col)
    wq.wq_check(plan.h)
    torch.cuda.synchronize()
    assert int(rp[-1]) == cfg.exact_nnz()
    assert check_pattern_in_full(o, rp, col, 0, info["n_rows_local"]) == cfg.exact_nnz()
    # every row: row sums
    n_rows = info["n_rows_local"]
    lens = rp[1:] - rp[:-1]
    idx = torch.repeat_interleave(torch.arange(n_rows, device=val.device), lens)
    ssum = torch.zeros(n_rows, dtype=torch.float64, device=val.device).index_add_(0, idx, val)
    smax = torch.zeros(n_rows, dtype=torch.float64, device=val.device).scatter_reduce_(0, idx, val.abs(), "amax")
    del idx
    want = mass_row_sums_oracle(o)
    got = ssum.cpu().numpy().astype(np.longdouble)
    ratio = np.abs(got - want) / (lens.cpu().numpy() * smax.cpu().numpy())
    # measured worst ratios (profiles/r02_mass_shapes.log): <= 1.9e-14 for p <= 6; 1.3e-13, 2.9e-13, 2.2e-12,
    # 1.4e-11 at p = 7..10 (boundary rows, kappa_i up to 3e7: the weights alternate in sign)
    factor = 2e-13 if p <= 6 else 2e-10
    print(f"mass {n_el}^3 p={p}", wq.KERNEL_NAMES[info["kernel"][0]], "worst |row sum - oracle| / (#I max|m|):",
          float(ratio.max()), "row", int(ratio.argmax()))
    assert float(ratio.max()) <= factor
    # sampled rows, entry by entry
    n = n_el + p
    rows = sample_rows(n, 3, p, k_random=8, seed=2)
    if p >= 5:
        rows = rows[:: max(1, len(rows) // (40 if p <= 7 else 16))]
    ptr, oc, ov, kappa, scale = o.rows(MASS, rows)
    gptr, gc, gv = gather_rows_device(rp, col, val, rows)
    # these small shapes reach kappa_i ~ 1e4 on corner rows at p = 6 (R6): strict regime for p <= 5
    st = compare_rows(rows, gptr, gc, gv, ptr, oc, ov, kappa, scale, strict=p <= 5)
    print(f"mass {n_el}^3 p={p}", st)
    plan.close()


@pytest.mark.parametrize("p", [2, 4, 6])
def test_2d_1000_every_row(p):
    """The d = 2 entries of the bench sweep (1000^2 elements, k_sf2l), both matrices: indices in
    full; stiffness of EVERY row through the zero row sum; mass of EVERY row through its row sum
    against the oracle's weights and coefficient field; sampled rows entry by entry."""
    torch = _torch()
    from wqinputs import Config
    cfg = Config(f"2D1000p{p}", 2, p, 1000, "grid", 0.1, ("stiffness", "mass"))
    ks, ctrl = cfg.knots(), cfg.ctrl()
    o = Oracle(p, ks, ctrl)
    plan = wq.Plan(p, ks, ctrl=ctrl, need_mass=True, need_stiffness=True)
    info = plan.info
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp)
    n = cfg.n_el + p
    rows = sample_rows(n, 2, p, k_random=64, seed=3)
    for mat in (STIFFNESS, MASS):
        wq.wq_assemble(plan.h, mat, val, col)
        wq.wq_check(plan.h)
        torch.cuda.synchronize()
        assert int(rp[-1]) == cfg.exact_nnz()
        if mat == STIFFNESS:
            assert check_pattern_in_full(o, rp, col, 0, info["n_rows_local"]) == cfg.exact_nnz()
            print("2D 1000^2 p =", p, "stiffness worst |row sum| / (#I max|s|):", stiffness_row_sums_every_row(rp, val, 2e-14))
        else:
            Wd = []
            for l in range(2):
                D = o.direction(l)
                W = np.zeros((o.n[l], o.nq[l]))
                for i in range(o.n[l]):
                    lo, ln = int(D["qlo"][i]), int(D["qlen"][i])
                    W[i, lo:lo + ln] = D["w"][i, 0, :ln]
                Wd.append(W)
            ref, det, st = o.coef_box([0, 0], list(o.nq))
            assert st == 0
            c = ref[:, 0].reshape(o.nq[1], o.nq[0])          # [q2][q1]
            want = (Wd[1] @ c @ Wd[0].T).reshape(-1)          # [i2][i1]
            lens = rp[1:] - rp[:-1]
            idx = torch.repeat_interleave(torch.arange(lens.numel(), device=val.device), lens)
            ssum = torch.zeros(lens.numel(), dtype=torch.float64, device=val.device).index_add_(0, idx, val)
            smax = torch.zeros(lens.numel(), dtype=torch.float64, device=val.device).scatter_reduce_(0, idx, val.abs(), "amax")
            ratio = np.abs(ssum.cpu().numpy() - want) / (lens.cpu().numpy() * smax.cpu().numpy())
            print("2D 1000^2 p =", p, "mass worst |row sum - oracle| / (#I max|m|):", float(ratio.max()))
            assert float(ratio.max()) <= 2e-13
        ptr, oc, ov, kappa, scale = o.rows(mat, rows)
        gptr, gc, gv = gather_rows_device(rp, col, val, rows)
        st = compare_rows(rows, gptr, gc, gv, ptr, oc, ov, kappa, scale, strict=p <= 5)
        print("2D 1000^2 p =", p, mat, wq.KERNEL_NAMES[info["kernel"][mat]], st)
    plan.close()
