"""GPU parity: the CUDA path (through the C-ABI binding) against the CPU oracle
on the same seeded inputs.  Indices bit-exact; values within the per-row
tolerance of tests/parity_util.py (reading R6)."""
import numpy as np
import pytest

import paper_1605_01238_b200 as wq
from oracle import MASS, STIFFNESS, Oracle
from parity_util import compare_rows, gather_rows_device, line_rows, oracle_rows_cached, sample_rows
from wqinputs import control_net, graded_open_knots, greville, uniform_open_knots

pytestmark = pytest.mark.gpu

KERNELS = [wq.WQ_KERNEL_AUTO, wq.WQ_KERNEL_DIRECT, wq.WQ_KERNEL_TILE, wq.WQ_KERNEL_ZLINE, wq.WQ_KERNEL_ZHP,
           wq.WQ_KERNEL_SF2]


def _torch():
    import torch
    return torch


def make_case(d, p, E, geometry="grid", amp=0.1, knots="uniform", seed=0):
    ks = [(uniform_open_knots if knots == "uniform" else graded_open_knots)(p, E + (l if knots != "uniform" else 0))
          for l in range(d)]
    ctrl = control_net(geometry, p, ks, amp, seed=seed)
    return ks, ctrl


class Unavailable(Exception):
    pass


def run_full(ks, ctrl, p, matrix, kernel=wq.WQ_KERNEL_AUTO, slab=(0, -1), fused_col=True, kappa=None, gamma=None,
             need=(True, True)):
    """Whole device path through the C-ABI for one matrix; raises Unavailable when the requested
    kernel does not serve (matrix, d, p) (a loud WQ_EINVAL from the library, never a fallback)."""
    torch = _torch()
    plan = wq.Plan(p, ks, ctrl=ctrl, kappa=kappa, gamma=gamma, slab=slab, need_mass=need[0], need_stiffness=need[1])
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp, None if fused_col else col)
    try:
        wq.wq_assemble(plan.h, matrix, val, col if fused_col else None, kernel=kernel)
    except wq.WQError as e:
        plan.close()
        if e.status == wq.WQ_EINVAL and kernel != wq.WQ_KERNEL_AUTO:
            raise Unavailable(str(e))
        raise
    wq.wq_check(plan.h)
    torch.cuda.synchronize()
    info = plan.info
    plan.close()
    return rp, col, val, info


def check_every_row(o, mat, rp, col, val, key=None, strict=False):
    orp, ocol = o.pattern()
    assert np.array_equal(rp.cpu().numpy(), orp)
    assert np.array_equal(col.cpu().numpy(), ocol)
    rows = np.arange(o.ndof)
    if key is None:
        ptr, oc, ov, kappa, scale = o.rows(mat, rows)
    else:
        ptr, oc, ov, kappa, scale = oracle_rows_cached(key, lambda: o, mat, rows)
    return compare_rows(rows, ptr, col.cpu().numpy(), val.cpu().numpy(), ptr, oc, ov, kappa, scale, strict=strict)


def refusal_expected(kernel, ks, p, mat):
    """The documented contract of the explicit kernels (include/wq.h wq_kernel): ZLINE serves
    stiffness, d = 3, 2 <= p <= 6, n_EL >= p+2 in every direction; TILE and ZHP serve d = 3, SF2 d <= 2; none of them serves a direction with
    one DOF row pair or a support that holds both boundary spans (#Q > 3p+1, reading R15).  AUTO and
    DIRECT serve every plan.  Used to turn a refusal into a check instead of a skip."""
    if kernel in (wq.WQ_KERNEL_AUTO, wq.WQ_KERNEL_DIRECT):
        return False
    d = len(ks)
    if kernel == wq.WQ_KERNEL_SF2:  # d <= 2, any p (the row tables of these tests fit in shared memory)
        return d == 3
    if d != 3:
        return True
    if kernel == wq.WQ_KERNEL_ZLINE and (mat != STIFFNESS or p < 2 or p > 6):
        return True
    for k in ks:
        D = Oracle(p, [k]).direction(0)
        n = len(D["qlen"])
        if int(np.max(D["qlen"])) > 3 * p + 1 or n < 2:
            return True
        # the z-line kernel compiles the 2p+3 row types of a direction with n_EL >= p+2 (ZTy)
        if kernel == wq.WQ_KERNEL_ZLINE and n - p < p + 2:
            return True
    return False


def run_matrices(ks, ctrl, p, kernel, mats, check):
    """Run each matrix with `kernel`.  A matrix the kernel refuses (loud WQ_EINVAL) must be one
    the documented contract excludes (refusal_expected); every other one is compared."""
    for mat in mats:
        try:
            rp, col, val, info = run_full(ks, ctrl, p, mat, kernel)
        except Unavailable as e:
            assert refusal_expected(kernel, ks, p, mat), f"kernel {kernel} refused a plan it serves: {e}"
            continue
        assert not refusal_expected(kernel, ks, p, mat), "kernel served a plan outside its documented contract"
        check(mat, rp, col, val, info)


# ------------------------------------------------------------------ rules
@pytest.mark.parametrize("p,E,knots", [(1, 1, "uniform"), (1, 6, "uniform"), (2, 2, "graded"), (3, 9, "uniform"),
                                       (4, 12, "graded"), (6, 16, "uniform"), (8, 20, "graded"), (10, 24, "uniform"),
                                       (10, 3, "graded")])
def test_rules_match_oracle(p, E, knots):
    """Points bit-exact (reading R1 formulas); Q ranges exact; basis tables and
    weights agree with the binary128 oracle to a few ulp (both are rounded
    from >=106-bit computations: Alg. 1 lines 3-4, Alg. 2)."""
    k = uniform_open_knots(p, E) if knots == "uniform" else graded_open_knots(p, E)
    o = Oracle(p, [k])
    D = o.direction(0)
    plan = wq.Plan(p, [k], need_mass=True, need_stiffness=False)
    R = wq.wq_export_rules(plan.h, 0, p)
    plan.close()
    assert np.array_equal(R["points"], D["points"])
    assert np.array_equal(R["qlo"], D["qlo"]) and np.array_equal(R["qlen"], D["qlen"])
    # basis tables: GPU stores functions span..span+p; oracle stores all n
    for q in range(o.nq[0]):
        s = R["span"][q]
        for r in range(p + 1):
            for b, tab in ((0, D["Bv"]), (1, D["Bd"])):
                ref = tab[q, s + r]
                assert abs(R["basis"][q, b, r] - ref) <= 2e-16 * max(abs(ref), 1e-300) * 4 + 1e-300
    W = R["w"]
    for i in range(o.n[0]):
        for f in range(4):
            ref = D["w"][i, f]
            sc = np.abs(ref).max()
            err = np.abs(W[i, f, :ref.size] - ref).max()
            assert err <= 8e-16 * sc, (i, f, err / sc)


def test_rules_valid_on_every_degree():
    """wq_plan_create validates the exactness systems (WQ_ESINGULAR) of every row for p = 1..10."""
    for p in range(1, 11):
        k = graded_open_knots(p, 2 * p + 3)
        plan = wq.Plan(p, [k, k], need_mass=True, need_stiffness=False)
        plan.close()


# ------------------------------------------------------------ coefficients
def _coef_ref(o, qb, nq_loc, d):
    """Oracle coefficient field on the plan's sub-grid (all q_1.., q_d in [qb, qb + nq_loc))."""
    ref, det, st = o.coef_box([0] * (d - 1) + [qb], list(o.nq[:-1]) + [qb + nq_loc])
    assert st == 0
    return ref


@pytest.mark.parametrize("d,p,E,geom", [(1, 3, 7, "grid"), (2, 2, 5, "annulus"), (2, 5, 6, "grid"),
                                        (3, 3, 4, "grid"), (3, 4, 5, "annulus"), (3, 10, 2, "grid"),
                                        (3, 1, 5, "grid"), (3, 7, 9, "annulus"), (3, 4, 14, "grid")])
def test_coef_matches_oracle(d, p, E, geom):
    """Step 5 (Alg. 1 lines 12/15): every component of c and C on the plan's sub-grid within 1e-13
    of the long-double oracle; d = 3 plans hold the z layout (k_dnet + k_coefz), incl. the
    uniform-line configuration E >= 4p+2 and p = 1, 7, 10 (generic-degree instantiation)."""
    ks, ctrl = make_case(d, p, E, geom, 0.05)
    o = Oracle(p, ks, ctrl)
    plan = wq.Plan(p, ks, ctrl=ctrl, need_mass=True, need_stiffness=True)
    G, qb = wq.wq_export_coef(plan.h)
    plan.close()
    nq_loc = G.shape[1] // int(np.prod(o.nq[:-1]))
    assert qb == 1 and nq_loc == o.nq[-1] - 2
    ref = _coef_ref(o, qb, nq_loc, d)
    comps = [(l, m) for l in range(d) for m in range(l, d)]
    for k, (l, m) in enumerate(comps):
        r = ref[:, 1 + l * d + m]
        np.testing.assert_allclose(G[k], r, rtol=0, atol=1e-13 * np.abs(r).max() + 1e-15)
    np.testing.assert_allclose(G[len(comps)], ref[:, 0], rtol=1e-13)


def test_coef_C2_zlayout_every_point():
    """BASELINE configs[1] (C2) coefficient field, every point, z layout (the z-line plan)."""
    from wqinputs import baseline_config
    cfg = baseline_config("C2")
    ks, ctrl = cfg.knots(), cfg.ctrl()
    o = Oracle(cfg.p, ks, ctrl)
    plan = wq.Plan(cfg.p, ks, ctrl=ctrl, need_mass=True, need_stiffness=True)
    assert plan.info["kernel"][1] == wq.WQ_KERNEL_ZLINE
    G, qb = wq.wq_export_coef(plan.h)
    plan.close()
    nq_loc = G.shape[1] // int(np.prod(o.nq[:-1]))
    ref = _coef_ref(o, qb, nq_loc, 3)
    for k, (l, m) in enumerate([(l, m) for l in range(3) for m in range(l, 3)]):
        r = ref[:, 1 + 3 * l + m]
        np.testing.assert_allclose(G[k], r, rtol=0, atol=1e-13 * np.abs(r).max())
    np.testing.assert_allclose(G[6], ref[:, 0], rtol=1e-13)


def test_folded_geometry_rejected_at_create():
    """Reading R7: det J changing sign on the grid -> wq_plan_create returns WQ_EGEOMETRY; the same
    control net passed to the stream-ordered wq_build_coef is reported by wq_check."""
    torch = _torch()
    p = 2
    ks = [uniform_open_knots(p, 4)] * 2
    P = control_net("grid", p, ks, 0.0)
    P[7, 0] += 0.9
    with pytest.raises(wq.WQError) as e:
        wq.Plan(p, ks, ctrl=P)
    assert e.value.status == wq.WQ_EGEOMETRY
    plan = wq.Plan(p, ks)
    plan.setup(torch.from_numpy(P).cuda())
    with pytest.raises(wq.WQError) as e:
        wq.wq_check(plan.h)
    assert e.value.status == wq.WQ_EGEOMETRY
    plan.close()


def test_assemble_without_geometry_refused():
    ks = [uniform_open_knots(2, 4)] * 3
    plan = wq.Plan(2, ks)
    rp, col, val = plan.alloc_csr()
    with pytest.raises(wq.WQError) as e:
        wq.wq_assemble(plan.h, STIFFNESS, val, col)
    assert e.value.status == wq.WQ_EINVAL
    plan.close()


# ------------------------------------------------------------- full parity
SMALL = [(1, 1, 1), (1, 2, 6), (1, 5, 3), (2, 1, 3), (2, 2, 2), (2, 3, 5), (2, 4, 1), (3, 1, 2), (3, 2, 3),
         (3, 3, 4), (3, 4, 2), (3, 5, 1), (3, 6, 2)]


@pytest.mark.parametrize("d,p,E", SMALL)
@pytest.mark.parametrize("kernel", KERNELS)
def test_full_parity_small(d, p, E, kernel):
    """Every row of small problems, both matrices, incl. n_EL = 1 and 2; each matrix runs if the
    kernel serves it (a kernel refusing one matrix does not skip the other)."""
    ks, ctrl = make_case(d, p, E, "grid", 0.08, knots="graded" if (p + E) % 2 else "uniform", seed=d + p)
    o = Oracle(p, ks, ctrl)
    key = ("small", d, p, E)
    run_matrices(ks, ctrl, p, kernel, (MASS, STIFFNESS),
                 lambda mat, rp, col, val, info: check_every_row(o, mat, rp, col, val, key))


@pytest.mark.parametrize("kernel", KERNELS)
def test_C1_full(kernel):
    """BASELINE configs[0]: 2D p=3, 16x16 elements, S and M, every row."""
    from wqinputs import baseline_config
    cfg = baseline_config("C1")
    ks, ctrl = cfg.knots(), cfg.ctrl()
    o = Oracle(cfg.p, ks, ctrl)

    def check(mat, rp, col, val, info):
        assert info["nnz_local"] == cfg.exact_nnz()
        check_every_row(o, mat, rp, col, val, "C1")
    run_matrices(ks, ctrl, cfg.p, kernel, (MASS, STIFFNESS), check)


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("kernel", [wq.WQ_KERNEL_AUTO, wq.WQ_KERNEL_ZHP])
def test_uniform_lines_every_row(p, kernel):
    """Uniform open knots with E = 4p+2 elements: the z-line plan has uniform lines (R16 tables in
    registers / kernel parameters: PU and CU classes), interior and boundary lines, every row type
    in every direction -- every row of the stiffness (and, for the kernels that serve it, the
    mass) matrix against the oracle."""
    E = 4 * p + 2
    ks, ctrl = make_case(3, p, E, "annulus", 0.05, seed=p)
    o = Oracle(p, ks, ctrl)
    plan = wq.Plan(p, ks, ctrl=ctrl)
    if kernel == wq.WQ_KERNEL_AUTO:
        assert plan.info["kernel"][1] == wq.WQ_KERNEL_ZLINE and plan.info["uniform_rules"] == 1
    plan.close()
    run_matrices(ks, ctrl, p, kernel, (STIFFNESS, MASS),
                 lambda mat, rp, col, val, info: check_every_row(o, mat, rp, col, val, ("uni", p), strict=True))


@pytest.mark.parametrize("p", [5, 6])
@pytest.mark.parametrize("kernel", [wq.WQ_KERNEL_AUTO, wq.WQ_KERNEL_ZHP])
def test_uniform_lines_all_classes(p, kernel):
    """p = 5, 6 (column-chunked z-line launches) on uniform knots, E = 4p+2: every row of the lines
    (i1, i2) with i1, i2 over one index of every row type (boundary types 0, 1, p, first interior
    p+1, first uniform 2p, the middle, and their mirrors) -- uniform, interior and boundary line
    classes, all i3 -- against the oracle."""
    torch = _torch()
    E = 4 * p + 2
    ks, ctrl = make_case(3, p, E, "annulus", 0.05, seed=p)
    n = E + p
    pick = sorted({0, 1, p, p + 1, 2 * p, n // 2, n - 1 - 2 * p, n - 2 - p, n - 1})
    rows = line_rows(n, pick)
    o = Oracle(p, ks, ctrl)
    for mat in (STIFFNESS,):
        try:
            rp, col, val, info = run_full(ks, ctrl, p, mat, kernel)
        except Unavailable as e:
            assert refusal_expected(kernel, ks, p, mat), str(e)
            continue
        ptr, oc, ov, kappa, scale = o.rows(mat, rows)
        gptr, gc, gv = gather_rows_device(rp, col, val, rows)
        compare_rows(rows, gptr, gc, gv, ptr, oc, ov, kappa, scale, strict=True)
        orp, ocol = o.pattern()
        assert np.array_equal(rp.cpu().numpy(), orp) and np.array_equal(col.cpu().numpy(), ocol)
        del rp, col, val
        torch.cuda.empty_cache()


@pytest.mark.parametrize("p,E", [(2, 7), (3, 8), (4, 9), (6, 8)])
@pytest.mark.parametrize("kernel", [wq.WQ_KERNEL_AUTO, wq.WQ_KERNEL_ZHP])
def test_graded_knots_every_row(p, E, kernel):
    """Non-uniform (graded) knots: every row's own rules (no uniform tables, reading R16
    inapplicable); every row of the stiffness matrix against the oracle."""
    ks, ctrl = make_case(3, p, E, "grid", 0.08, knots="graded", seed=3)
    o = Oracle(p, ks, ctrl)
    run_matrices(ks, ctrl, p, kernel, (STIFFNESS, MASS),
                 lambda mat, rp, col, val, info: check_every_row(o, mat, rp, col, val, ("graded", p, E)))


# ------------------------------------------------- d <= 2 sum-factorised rows
@pytest.mark.parametrize("d,p,E,knots", [(2, p, E, kn) for p, E in [(1, 9), (2, 7), (3, 11), (4, 6), (5, 8),
                                                                   (6, 5), (7, 9), (8, 3), (9, 4), (10, 12)]
                                         for kn in ("uniform", "graded")] + [(1, 10, 17, "graded"), (1, 4, 2, "uniform")])
def test_sf2_every_row(d, p, E, knots):
    """The d <= 2 product kernel (WQ_KERNEL_SF2, Eq. sumfactorization) on every row, both
    matrices, p = 1..10, uniform and graded knots, n_EL from below p+1 to several tiles of rows
    per CTA (8 rows per CTA: the last CTA ragged); AUTO must pick it."""
    ks, ctrl = make_case(d, p, E, "grid", 0.08, knots=knots, seed=5 + p)
    o = Oracle(p, ks, ctrl)
    for mat in (MASS, STIFFNESS):
        rp, col, val, info = run_full(ks, ctrl, p, mat, wq.WQ_KERNEL_SF2)
        assert info["kernel"][mat] == wq.WQ_KERNEL_SF2
        check_every_row(o, mat, rp, col, val, ("sf2", d, p, E, knots))


@pytest.mark.parametrize("p,E,knots", [(2, 7, "graded"), (4, 6, "uniform"), (9, 4, "graded")])
def test_sf2_row_variant_every_row(p, E, knots, monkeypatch):
    """The warp-per-row form of WQ_KERNEL_SF2 (d = 1, and d = 2 when the chunk tables do not fit),
    forced on d = 2 by the measurement switch WQ_SF2_ROWS: every row against the oracle."""
    monkeypatch.setenv("WQ_SF2_ROWS", "1")
    ks, ctrl = make_case(2, p, E, "grid", 0.08, knots=knots, seed=3)
    o = Oracle(p, ks, ctrl)
    for mat in (MASS, STIFFNESS):
        rp, col, val, info = run_full(ks, ctrl, p, mat, wq.WQ_KERNEL_SF2)
        check_every_row(o, mat, rp, col, val, ("sf2r", p, E, knots))


@pytest.mark.parametrize("p,E,chunk", [(3, 40, 20000), (5, 37, 9000)])
def test_sf2_plane_ranges_form_host(p, E, chunk, monkeypatch):
    """d = 2 through wq_form_host in plane chunks (the line kernel's launches then start inside the
    slab, at chunk boundaries that are not multiples of its rows per CTA) == one device call."""
    torch = _torch()
    ks, ctrl = make_case(2, p, E)
    for mat in (MASS, STIFFNESS):
        rp0, col0, val0, info = run_full(ks, ctrl, p, mat, wq.WQ_KERNEL_SF2)
        monkeypatch.setenv("WQ_FORM_CHUNK_NNZ", str(chunk))
        plan = wq.Plan(p, ks)
        n, nnz = plan.info["n_rows_local"], plan.info["nnz_local"]
        hrp = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        hcol = torch.empty(nnz, dtype=torch.int32).pin_memory()
        hval = torch.empty(nnz, dtype=torch.float64).pin_memory()
        wq.wq_form_host(plan.h, mat, torch.from_numpy(ctrl).pin_memory(), 0, hrp, hcol, hval)
        plan.close()
        monkeypatch.delenv("WQ_FORM_CHUNK_NNZ")
        assert np.array_equal(hrp.numpy(), rp0.cpu().numpy())
        assert np.array_equal(hcol.numpy(), col0.cpu().numpy())
        assert np.array_equal(hval.numpy(), val0.cpu().numpy())


# ------------------------------------------------- scalar coefficients (R17)
@pytest.mark.parametrize("d,p,E", [(1, 3, 9), (2, 3, 6), (3, 2, 6), (3, 4, 5), (3, 7, 2)])
@pytest.mark.parametrize("kernel", KERNELS)
def test_coefficients_every_row(d, p, E, kernel):
    """-div(kappa grad u) + gamma u with spline coefficient nets kappa, gamma (
    reading R17): c = gamma |det J| and C = kappa |det J| J^-1 J^-T on the GPU against the oracle,
    every row, both matrices."""
    ks, ctrl = make_case(d, p, E, "grid", 0.08, seed=11)
    rng = np.random.default_rng(7)
    n = int(np.prod([k.size - p - 1 for k in ks]))
    kap = 1.0 + 0.5 * rng.uniform(size=n)
    gam = 0.5 + rng.uniform(size=n)
    o = Oracle(p, ks, ctrl, kappa=kap, gamma=gam)
    for mat in (STIFFNESS, MASS):
        try:
            rp, col, val, info = run_full(ks, ctrl, p, mat, kernel, kappa=kap, gamma=gam)
        except Unavailable as e:
            assert refusal_expected(kernel, ks, p, mat), str(e)
            continue
        check_every_row(o, mat, rp, col, val, ("coef", d, p, E))


def test_coefficient_example_printed_gpu():
    """The paper's worked example P:391-402 through the GPU mass path: p = 3, h = 2, identity map,
    gamma(zeta) = zeta: m~_{8,9} and m~_{9,8} equal the printed sums (2.3647 / 2.3615)."""
    import json
    import os
    from fractions import Fraction as Fr
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))["asymmetry_example"]
    k = np.array([-10.0] * 4 + [float(x) for x in range(-8, 20, 2)] + [20.0] * 4)
    gv = greville(3, k)
    rp, col, val, info = run_full([k], gv.reshape(-1, 1), 3, MASS, gamma=gv, need=(True, False))
    rp, col, val = rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()
    m89 = val[rp[8]:rp[9]][list(col[rp[8]:rp[9]]).index(9)]
    m98 = val[rp[9]:rp[10]][list(col[rp[9]:rp[10]]).index(8)]
    assert abs(m89 - float(sum(Fr(*a) * b * Fr(*c) for a, b, c in g["Qi_cBj_terms"]))) < 1e-13
    assert abs(m98 - float(sum(Fr(*a) * b * Fr(*c) for a, b, c in g["Qj_cBi_terms"]))) < 1e-13


# ---------------------------------------------------------- slabs / e2e
@pytest.mark.parametrize("d,p,E,nslab", [(2, 3, 8, 3), (3, 2, 5, 2), (3, 4, 6, 4), (3, 4, 18, 3), (3, 8, 5, 2)])
def test_slabs_concatenate_bit_exact(d, p, E, nslab):
    """Multi-GPU decomposition, run sequentially on one
    GPU: per-slab CSR blocks with nnz_base from an exclusive scan concatenate
    to the single-plan CSR, bit for bit (indices and values)."""
    torch = _torch()
    from paper_1605_01238_b200.dist import slab_cuts
    ks, ctrl = make_case(d, p, E)
    rp0, col0, val0, info0 = run_full(ks, ctrl, p, STIFFNESS)
    cuts = slab_cuts(E + p, p, nslab)
    base = 0
    rps, cols, vals = [], [], []
    for s in range(nslab):
        plan = wq.Plan(p, ks, ctrl=ctrl, slab=(cuts[s], cuts[s + 1]), need_mass=False, need_stiffness=True)
        assert plan.info["kernel"][1] == info0["kernel"][1]
        rp, col, val = plan.form(STIFFNESS, nnz_base=base)
        base += plan.info["nnz_local"]
        rps.append(rp[:-1].cpu().numpy())
        cols.append(col.cpu().numpy())
        vals.append(val.cpu().numpy())
        plan.close()
    assert base == info0["nnz_total"]
    rp_cat = np.concatenate(rps + [np.array([base])])
    assert np.array_equal(rp_cat, rp0.cpu().numpy())
    assert np.array_equal(np.concatenate(cols), col0.cpu().numpy())
    assert np.array_equal(np.concatenate(vals), val0.cpu().numpy())


def test_form_host_equals_device():
    """wq_form_host (host buffers, chunked, copies overlapped) == device path, incl. coefficients."""
    torch = _torch()
    ks, ctrl = make_case(3, 3, 10)
    n = ctrl.shape[0]
    kap = np.linspace(1.0, 2.0, n)
    for mat in (MASS, STIFFNESS):
        for kk in (None, kap):
            rp0, col0, val0, info = run_full(ks, ctrl, 3, mat, kappa=kk, gamma=kk)
            plan = wq.Plan(3, ks)
            nr, nnz = plan.info["n_rows_local"], plan.info["nnz_local"]
            hrp = torch.empty(nr + 1, dtype=torch.int64).pin_memory()
            hcol = torch.empty(nnz, dtype=torch.int32).pin_memory()
            hval = torch.empty(nnz, dtype=torch.float64).pin_memory()
            hctrl = torch.from_numpy(ctrl).pin_memory()
            hk = None if kk is None else torch.from_numpy(kk).pin_memory()
            wq.wq_form_host(plan.h, mat, hctrl, 0, hrp, hcol, hval, h_kappa=hk, h_gamma=hk)
            plan.close()
            assert np.array_equal(hrp.numpy(), rp0.cpu().numpy())
            assert np.array_equal(hcol.numpy(), col0.cpu().numpy())
            assert np.array_equal(hval.numpy(), val0.cpu().numpy())


@pytest.mark.parametrize("p,E,chunk", [(2, 9, 4000), (3, 8, 9000), (4, 7, 20000)])
def test_zline_plane_ranges(p, E, chunk, monkeypatch):
    """z-line kernel over plane sub-ranges (wq_form_host chunks: odd first task
    point, few rows per line) equals the whole-plan launch bit for bit."""
    torch = _torch()
    ks, ctrl = make_case(3, p, E, "annulus", 0.05)
    rp0, col0, val0, info = run_full(ks, ctrl, p, STIFFNESS, wq.WQ_KERNEL_ZLINE)
    monkeypatch.setenv("WQ_FORM_CHUNK_NNZ", str(chunk))
    plan = wq.Plan(p, ks, need_mass=False, need_stiffness=True)
    n, nnz = plan.info["n_rows_local"], plan.info["nnz_local"]
    hrp = torch.empty(n + 1, dtype=torch.int64).pin_memory()
    hcol = torch.empty(nnz, dtype=torch.int32).pin_memory()
    hval = torch.empty(nnz, dtype=torch.float64).pin_memory()
    wq.wq_form_host(plan.h, STIFFNESS, torch.from_numpy(ctrl).pin_memory(), 0, hrp, hcol, hval)
    plan.close()
    assert np.array_equal(hrp.numpy(), rp0.cpu().numpy())
    assert np.array_equal(hcol.numpy(), col0.cpu().numpy())
    assert np.array_equal(hval.numpy(), val0.cpu().numpy())


def test_every_kernel_reads_every_plan():
    """The coefficient layout is the library's business: on a z-line plan (z layout) the direct and
    tile kernels still assemble the stiffness matrix, within the oracle tolerance (per row)."""
    p, E = 3, 6
    ks, ctrl = make_case(3, p, E)
    o = Oracle(p, ks, ctrl)
    for k in (wq.WQ_KERNEL_DIRECT, wq.WQ_KERNEL_TILE, wq.WQ_KERNEL_ZLINE):
        rp, col, val, info = run_full(ks, ctrl, p, STIFFNESS, k)
        assert info["kernel"][1] == wq.WQ_KERNEL_ZLINE
        check_every_row(o, STIFFNESS, rp, col, val)


@pytest.mark.parametrize("p,E,kernel,matrix", [(3, 14, "ZLINE", STIFFNESS), (4, 18, "ZLINE", STIFFNESS),
                                               (4, 18, "ZHP", STIFFNESS), (8, 20, "ZHP", STIFFNESS),
                                               (6, 16, "ZHP", MASS)])
def test_zline_repeatable_bit_exact(p, E, kernel, matrix):
    """Stress check of the producer/consumer hand-offs (ADVICE: ring slots are returned with relaxed
    mbarrier arrives, z-line and ZHP): 20 back-to-back assemblies of the same plan give bit-identical
    values."""
    torch = _torch()
    ks, ctrl = make_case(3, p, E, "annulus", 0.05)
    plan = wq.Plan(p, ks, ctrl=ctrl, need_mass=matrix == MASS, need_stiffness=matrix == STIFFNESS)
    k = getattr(wq, "WQ_KERNEL_" + kernel)
    rp, col, val = plan.alloc_csr()
    wq.wq_assemble(plan.h, matrix, val, col, kernel=k)
    ref = val.clone()
    for _ in range(20):
        val.zero_()
        wq.wq_assemble(plan.h, matrix, val, col, kernel=k)
        torch.cuda.synchronize()
        assert torch.equal(val, ref)
    plan.close()


def test_stream_ordered_calls_capture_in_cuda_graph():
    """wq_build_rules / wq_build_coef / wq_pattern / wq_assemble never synchronise the host (wq.h):
    they are captured into a CUDA graph (a synchronising call would invalidate the capture), and
    the replayed graph reproduces the eager result bit for bit."""
    torch = _torch()
    p, E = 4, 10
    ks, ctrl = make_case(3, p, E)
    plan = wq.Plan(p, ks, ctrl=ctrl)
    d_ctrl = torch.from_numpy(ctrl).cuda()
    rp, col, val = plan.alloc_csr()
    rp2, col2, val2 = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp)
    wq.wq_assemble(plan.h, STIFFNESS, val, col)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        st = torch.cuda.current_stream()
        wq.wq_build_rules(plan.h, st)
        wq.wq_build_coef(plan.h, d_ctrl, stream=st)
        wq.wq_pattern(plan.h, 0, rp2, None, st)
        wq.wq_assemble(plan.h, STIFFNESS, val2, col2, st)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(rp, rp2) and torch.equal(col, col2) and torch.equal(val, val2)
    plan.close()
