"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Every test names the passage of /root/reference/PAPER.md ("P:<line>") or the
mathematical fact it uses.  None of these re-types the oracle's formulas: they
use printed values (tests/golden/paper_values.json), closed forms (cardinal
B-splines, Marsden's identity, affine maps), invariants and brute force.
"""
import json
import math
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
from oracle import MASS, STIFFNESS, Oracle
from wqinputs import control_net, greville, uniform_open_knots, graded_open_knots

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def frac(v):
    return float(Fr(v[0], v[1]))


# ---------------------------------------------------------------- closed forms
def cardinal(p, x):
    """Cardinal B-spline of degree p on [0, p+1] (closed form, truncated powers)."""
    s = 0.0
    for k in range(p + 2):
        t = x - k
        if t > 0:
            s += (-1) ** k * math.comb(p + 1, k) * t ** p
    return s / math.factorial(p) if 0 < x < p + 1 else 0.0


def cardinal_d(p, x):
    return cardinal(p - 1, x) - cardinal(p - 1, x - 1) if p >= 1 else 0.0


def interior_row(p, E):
    """0-based interior row whose support touches no boundary span (reading R14)."""
    return p + 1 + (E - 2 * p - 3) // 2


# ------------------------------------------------------------------ P1 / P2
@pytest.mark.parametrize("p", [1, 2, 3])
def test_interior_w00_printed(p):
    """P1: w^(0,0) = printed closed forms."""
    E = 4 * p + 6
    h = 1.0 / E
    o = Oracle(p, [uniform_open_knots(p, E)])
    D = o.direction(0)
    ref = np.array([frac(v) for v in GOLD["interior_weights_w00_over_h"][str(p)]])
    for i in range(p + 1, o.n[0] - p - 1):
        got = D["w"][i, 0, : D["qlen"][i]] / h
        assert D["qlen"][i] == 2 * p + 1
        np.testing.assert_allclose(got, ref, rtol=2e-14, atol=0)


@pytest.mark.parametrize("p", [1, 2])
def test_interior_integrals_printed(p):
    """P2: I^(0,0) interior entries = printed values."""
    E = 10
    h = 1.0 / E
    o = Oracle(p, [uniform_open_knots(p, E)])
    D = o.direction(0)
    ref = np.array([frac(v) for v in GOLD["interior_integrals_I00_over_h"][str(p)]])
    i = interior_row(p, E)
    np.testing.assert_allclose(D["I4"][i, : 2 * p + 1, 0] / h, ref, rtol=1e-14)


def test_bspline_printed_values():
    """B-spline values quoted in Eq. int_1d_5 and P:397-401."""
    g = GOLD["bspline_values"]
    p, E = 2, 12
    k = uniform_open_knots(p, E)
    h = 1.0 / E
    i = interior_row(p, E)  # support (xi_i, xi_{i+3}) = ((i-2)h, (i+1)h)
    a = (i - p) * h
    for x_h, ref in zip(g["p2_points_over_h"], g["p2_B_im1"]):
        v, _ = oracle.basis_all(p, k, a + x_h * h)
        assert abs(v[i - 1] - frac(ref)) < 1e-15
    # p = 3, h = 2 on [-10, 20]: B_j with support (2, 10), j = i+1
    k3 = np.array([-10.0] * 4 + [float(x) for x in range(-8, 20, 2)] + [20.0] * 4)
    for x, ref in zip(g["p3_h2_points"], g["p3_B_jplus1_rel"]):
        v, _ = oracle.basis_all(3, k3, float(x))
        j = 9  # xi_9 = chi_6 = 2
        assert abs(v[j] - frac(ref)) < 1e-15


@pytest.mark.parametrize("p", [1, 2, 3, 5, 8])
def test_bspline_partition_and_derivative(p):
    """Partition of unity, sum of derivatives 0, central-difference derivative check."""
    k = graded_open_knots(p, 9)
    rng = np.random.default_rng(p)
    for x in rng.uniform(0, 1, 40):
        v, dv = oracle.basis_all(p, k, x)
        assert abs(v.sum() - 1) < 1e-14
        assert abs(dv.sum()) < 1e-11 * max(1, np.abs(dv).max())
        e = 1e-6
        vp, _ = oracle.basis_all(p, k, x + e)
        vm, _ = oracle.basis_all(p, k, x - e)
        if not np.any((k > x - e) & (k < x + e)):
            np.testing.assert_allclose((vp - vm) / (2 * e), dv, atol=1e-5 * max(1, np.abs(dv).max()))


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_bspline_vs_cardinal(p):
    """Interior functions on uniform knots equal the closed-form cardinal B-spline."""
    E = 3 * p + 6
    h = 1.0 / E
    k = uniform_open_knots(p, E)
    i = interior_row(p, E)
    a = (i - p) * h
    for t in np.linspace(0.05, p + 0.95, 23) + 0.0137:  # avoid knots (derivative jumps at p=1)
        v, dv = oracle.basis_all(p, k, a + t * h)
        assert abs(v[i] - cardinal(p, t)) < 1e-14
        assert abs(dv[i] * h - cardinal_d(p, t)) < 1e-12


@pytest.mark.parametrize("n", [1, 2, 5, 11, 16])
def test_gauss_legendre(n):
    """n-point Gauss-Legendre integrates x^k exactly for k <= 2n-1."""
    t, w = oracle.gauss(n)
    for kk in range(2 * n):
        exact = 0.0 if kk % 2 else 2.0 / (kk + 1)
        assert abs(np.sum(w * t ** kk) - exact) < 1e-15


# ------------------------------------------------------------- weights, P1'
@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_interior_all_families_vs_cardinal_minnorm(p):
    """All four families on interior rows equal the min-norm solution built from
    closed-form cardinal B-splines, integrals by mpmath quadrature and a
    40-digit SVD pseudo-inverse (h = 1): Eq. integrals/quadrule/exact
    (P:588-633), Remark 2.  Independent of the oracle's QR."""
    import mpmath as mp
    mp.mp.dps = 40

    def card(q, x):
        if not (0 < x < q + 1):
            return mp.mpf(0)
        s = mp.mpf(0)
        for k in range(q + 2):
            t = x - k
            if t > 0:
                s += (-1) ** k * mp.binomial(q + 1, k) * t ** q
        return s / mp.factorial(q)

    def card_d(q, x):
        return card(q - 1, x) - card(q - 1, x - 1)

    E = 4 * p + 6
    o = Oracle(p, [uniform_open_knots(p, E)])
    D = o.direction(0)
    h = 1.0 / E
    i = interior_row(p, E)
    xs = [mp.mpf(k + 1) / 2 for k in range(2 * p + 1)]  # midpoints and knots inside (0, p+1)
    scale = {0: h, 1: 1.0, 2: h, 3: 1.0}  # w^(a,b) scaling with h (P10)
    for f, (a, b) in enumerate(oracle.FAMILIES):
        fb = card_d if b else card
        fa = card_d if a else card
        M = mp.matrix([[fb(p, x - s) for x in xs] for s in range(-p, p + 1)])
        I = mp.matrix([sum(mp.quad(lambda x: fa(p, x) * fb(p, x - s), [e, e + 1]) for e in range(p + 1))
                       for s in range(-p, p + 1)])
        U, S, V = mp.svd_r(M)
        tol = mp.mpf(10) ** -25 * max(S)
        Sp = mp.diag([1 / sv if sv > tol else 0 for sv in S])
        w = V.T * Sp * U.T * I
        w = np.array([float(v) for v in w])
        got = D["w"][i, f, : 2 * p + 1] / scale[f]
        np.testing.assert_allclose(got, w, rtol=0, atol=5e-15 * np.abs(w).max())


@pytest.mark.parametrize("p", [1, 2, 3, 4, 6, 8, 10])
@pytest.mark.parametrize("knots", ["uniform", "graded"])
def test_exactness_all_rows(p, knots):
    """P7: Eq. exact for all four families on every row, including
    boundary rows, checked in float64 from the exported tables (no solver)."""
    E = max(2 * p + 4, 12)
    k = uniform_open_knots(p, E) if knots == "uniform" else graded_open_knots(p, E)
    o = Oracle(p, [k])
    D = o.direction(0)
    for i in range(o.n[0]):
        q0, nq, j0, ni = D["qlo"][i], D["qlen"][i], D["jlo"][i], D["jlen"][i]
        for f, (a, b) in enumerate(oracle.FAMILIES):
            B = D["Bd"] if b else D["Bv"]
            w = D["w"][i, f, :nq]
            T = w[None, :] * B[q0:q0 + nq, j0:j0 + ni].T
            res = T.sum(axis=1) - D["I4"][i, :ni, f]
            tol = 1e-12 * (np.abs(T).sum(axis=1) + np.abs(D["I4"][i, :ni, f])) + 1e-300
            assert np.all(np.abs(res) <= tol), (i, f, res)
            assert np.all(D["w"][i, f, nq:] == 0)


@pytest.mark.parametrize("p", [2, 3, 5, 8, 10])
def test_w00_positive_interior(p):
    """P11: interior w^(0,0) > 0 (Fig. 2 caption)."""
    E = 2 * p + 8
    o = Oracle(p, [uniform_open_knots(p, E)])
    D = o.direction(0)
    for i in range(p + 1, o.n[0] - p - 1):
        assert np.all(D["w"][i, 0, : D["qlen"][i]] > 0)


@pytest.mark.parametrize("p", [2, 4, 7])
def test_translation_and_scaling(p):
    """P10: interior rows on uniform knots are translates of each other; under
    zeta -> s*zeta the families scale as (s, 1, s, 1)."""
    E = 3 * p + 8
    o1 = Oracle(p, [uniform_open_knots(p, E)])
    s = 3.5
    o2 = Oracle(p, [uniform_open_knots(p, E) * s])
    D1, D2 = o1.direction(0), o2.direction(0)
    rows = list(range(p + 1, o1.n[0] - p - 1))
    ref = D1["w"][rows[0]]
    for i in rows[1:]:
        np.testing.assert_allclose(D1["w"][i], ref, rtol=0, atol=1e-13 * np.abs(ref).max())
    fac = np.array([s, 1.0, s, 1.0])[:, None]
    for i in range(o1.n[0]):
        np.testing.assert_allclose(D2["w"][i], D1["w"][i] * fac, rtol=0,
                                   atol=1e-13 * max(1.0, np.abs(D1["w"][i] * fac).max()))


def test_asymmetry_example_printed():
    """P3: the worked example P:391-402 (p=3, h=2, c(zeta)=zeta, j=i+1).
    The oracle's weights/points/basis reproduce the paper's printed sums."""
    g = GOLD["asymmetry_example"]
    k = np.array([-10.0] * 4 + [float(x) for x in range(-8, 20, 2)] + [20.0] * 4)
    o = Oracle(3, [k])
    D = o.direction(0)
    i, j = 8, 9  # supports (0, 8) and (2, 10)

    def Q(row, other):
        q0, nq = D["qlo"][row], D["qlen"][row]
        x = D["points"][q0:q0 + nq]
        return float(np.sum(D["w"][row, 0, :nq] * x * D["Bv"][q0:q0 + nq, other]))

    exact_i = sum(Fr(*a) * b * Fr(*c) for a, b, c in g["Qi_cBj_terms"])
    exact_j = sum(Fr(*a) * b * Fr(*c) for a, b, c in g["Qj_cBi_terms"])
    assert abs(Q(i, j) - float(exact_i)) < 1e-13
    assert abs(Q(j, i) - float(exact_j)) < 1e-13
    assert abs(Q(i, j) - g["Qi_cBj_printed"]) < 0.5e-4
    assert abs(Q(j, i) - g["Qj_cBi_printed"]) < 0.5e-4
    assert np.allclose(D["points"][D["qlo"][i]:D["qlo"][i] + 7], np.arange(1, 8))


# --------------------------------------------------------------- grid, P8/P9
@pytest.mark.parametrize("p,E", [(1, 1), (1, 2), (2, 1), (2, 3), (3, 7), (5, 5), (10, 12)])
def test_point_grid(p, E):
    """P9: n_QP = 2E+2p+1 (E >= 2); knots + internal midpoints + p+1 points inside each
    boundary span (Remark 1, reading R1); #Q_i >= #I_i (Eq. numb_nodes)."""
    k = graded_open_knots(p, E)
    x = oracle.points(p, k)
    assert x.size == (2 * E + 2 * p + 1 if E >= 2 else p + 3)  # E = 1: one span, p+1 inner points
    assert np.all(np.diff(x) > 0)
    chi = k[p:p + E + 1]
    assert set(chi).issubset(set(x))
    o = Oracle(p, [k])
    D = o.direction(0)
    assert np.all(D["qlen"] >= D["jlen"])
    for e in range(E):
        inside = np.sum((x > chi[e]) & (x < chi[e + 1]))
        assert inside == (p + 1 if e in (0, E - 1) else 1)


@pytest.mark.parametrize("d,p,E", [(1, 3, 9), (2, 2, 5), (3, 2, 3), (3, 1, 4)])
def test_pattern(d, p, E):
    """P8: 1D nnz = (2p+1)n - p(p+1); nD nnz = product; cols = prod_l I_{l,i_l},
    ascending (i_1 fastest)."""
    o = Oracle(p, [uniform_open_knots(p, E)] * d)
    rp, col = o.pattern()
    n = E + p
    assert rp[-1] == ((2 * p + 1) * n - p * (p + 1)) ** d
    for r in range(o.ndof):
        c = col[rp[r]:rp[r + 1]]
        assert np.all(np.diff(c) > 0)
        ii = np.unravel_index(r, [n] * d, order="F")
        jj = np.array(np.unravel_index(c, [n] * d, order="F"))
        for l in range(d):
            assert set(jj[l]) == set(range(max(0, ii[l] - p), min(n - 1, ii[l] + p) + 1))


def test_bad_knots():
    assert oracle.check_knots(2, [0, 0, 0, 0.5, 0.5, 1, 1, 1]) == 2  # repeated interior knot
    assert oracle.check_knots(2, [0, 0, 0.5, 1, 1, 1]) == 2           # not open
    assert oracle.check_knots(2, [0, 0, 0, 0.7, 0.3, 1, 1, 1]) == 2   # decreasing
    assert oracle.check_knots(2, [0, 0, 0, 1, 1, 1]) == 0


# ------------------------------------------------------------ coefficients
def test_coef_affine():
    """Affine F(zeta) = A zeta (Greville control points, linear precision):
    c = |det A|, C = |det A| A^{-1} A^{-T} at every grid point (Eq. coef_stiff)."""
    A = np.array([[2.0, 0.5, 0.1], [0.3, 1.5, -0.2], [0.0, 0.4, 1.2]])
    p = 3
    ks = [uniform_open_knots(p, 4), graded_open_knots(p, 3), uniform_open_knots(p, 2)]
    ctrl = control_net("affine:" + ",".join(map(str, A.ravel())), p, ks, 0.0)
    o = Oracle(p, ks, ctrl)
    out, det, st = o.coef_box([0, 0, 0], o.nq)
    assert st == 0
    Ai = np.linalg.inv(A)
    np.testing.assert_allclose(out[:, 0], abs(np.linalg.det(A)), rtol=1e-13)
    Cref = abs(np.linalg.det(A)) * Ai @ Ai.T
    np.testing.assert_allclose(out[:, 1:], np.tile(Cref.ravel(), (out.shape[0], 1)), rtol=1e-12, atol=1e-14)


def test_coef_marsden_quadratic():
    """Non-affine map F = (z1 + 0.3 z2^2, z2 + 0.2 z1 z3, z3) built exactly with
    Marsden's identity (zeta^2 = sum_k sym2(xi_{k+1..k+p})/C(p,2) B_k);
    J is known in closed form."""
    p, E = 3, 4
    ks = [graded_open_knots(p, E), uniform_open_knots(p, E + 1), uniform_open_knots(p, E - 1)]
    gs = [greville(p, k) for k in ks]

    def sym2(k):
        n = k.size - p - 1
        out = np.empty(n)
        for i in range(n):
            t = k[i + 1:i + p + 1]
            out[i] = (t.sum() ** 2 - (t ** 2).sum()) / 2 / math.comb(p, 2)
        return out
    s2 = sym2(ks[1])
    n = [g.size for g in gs]
    P = np.zeros((np.prod(n), 3))
    r = 0
    for k3 in range(n[2]):
        for k2 in range(n[1]):
            for k1 in range(n[0]):
                z1, z2, z3 = gs[0][k1], gs[1][k2], gs[2][k3]
                P[r] = (z1 + 0.3 * s2[k2], z2 + 0.2 * z1 * z3, z3)  # bilinear z1*z3 is exact on products of Greville
                r += 1
    o = Oracle(p, ks, P)
    out, det, st = o.coef_box([0, 0, 0], o.nq)
    assert st == 0
    x = [o.direction(l)["points"] for l in range(3)]
    r = 0
    for q3 in range(o.nq[2]):
        for q2 in range(o.nq[1]):
            for q1 in range(o.nq[0]):
                z1, z2, z3 = x[0][q1], x[1][q2], x[2][q3]
                J = np.array([[1, 0.6 * z2, 0], [0.2 * z3, 1, 0.2 * z1], [0, 0, 1.0]])
                dJ = np.linalg.det(J)
                Ji = np.linalg.inv(J)
                assert abs(det[r] - dJ) < 1e-13
                np.testing.assert_allclose(out[r, 1:], (abs(dJ) * Ji @ Ji.T).ravel(), atol=1e-13)
                r += 1


def test_coef_folded_map_rejected():
    """Reading R7: det J changing sign -> EGEOMETRY."""
    p = 2
    ks = [uniform_open_knots(p, 4)] * 2
    P = control_net("grid", p, ks, 0.0)
    P[7, 0] += 0.9  # fold
    o = Oracle(p, ks, P)
    _, det, st = o.coef_box([0, 0], o.nq)
    assert st == oracle.ORC_EGEOMETRY
    assert det.min() < 0 < det.max()


# ------------------------------------------------------------- whole rows
@pytest.mark.parametrize("d,p,E", [(1, 3, 7), (2, 2, 4), (2, 3, 5), (3, 2, 3)])
def test_affine_wq_equals_galerkin(d, p, E):
    """P4: for affine F and constant coefficients WQ is exact:
    oracle WQ rows == element-loop Gauss brute force (SGQ), every row."""
    A = np.array([[1.7, 0.4, 0.2], [-0.3, 1.1, 0.25], [0.1, -0.2, 0.9]])[:d, :d]
    ks = [graded_open_knots(p, E + l) for l in range(d)]
    ctrl = control_net("affine:" + ",".join(map(str, A.ravel())), p, ks, 0.0)
    o = Oracle(p, ks, ctrl)
    for mat in (MASS, STIFFNESS):
        W = o.dense(mat)
        G = o.sgq_dense(mat)
        for r in range(o.ndof):
            sc = np.abs(G[r]).max()
            assert np.abs(W[r] - G[r]).max() <= 1e-13 * sc, (mat, r)


def test_affine_kronecker_1d():
    """P4 (second form): diagonal affine map in 2D -> M = a1 a2 (M1 (x) M2), S = a2/a1 K1 (x) M2 + a1/a2 M1 (x) K2
    with the 1D Galerkin matrices (interior entries pinned by P2)."""
    p, E = 2, 6
    ks = [uniform_open_knots(p, E), uniform_open_knots(p, E + 1)]
    a1, a2 = 2.0, 0.5
    ctrl = control_net(f"affine:{a1},0,0,{a2}", p, ks, 0.0)
    o = Oracle(p, ks, ctrl)
    mats = []
    for l in range(2):
        D = o.direction(l)
        n = o.n[l]
        M1 = np.zeros((n, n)); K1 = np.zeros((n, n))
        for i in range(n):
            j0, ni = D["jlo"][i], D["jlen"][i]
            M1[i, j0:j0 + ni] = D["I4"][i, :ni, 0]
            K1[i, j0:j0 + ni] = D["I4"][i, :ni, 3]
        mats.append((M1, K1))
    (M1, K1), (M2, K2) = mats
    Mref = a1 * a2 * np.kron(M2, M1)
    Sref = (a2 / a1) * np.kron(M2, K1) + (a1 / a2) * np.kron(K2, M1)
    np.testing.assert_allclose(o.dense(MASS), Mref, atol=1e-14 * np.abs(Mref).max())
    np.testing.assert_allclose(o.dense(STIFFNESS), Sref, atol=1e-13 * np.abs(Sref).max())


@pytest.mark.parametrize("d,p,E", [(2, 3, 6), (3, 2, 4), (3, 4, 3)])
def test_stiffness_row_sums_zero(d, p, E):
    """P5: sum_j s~_ij = 0 for any geometry: sum_{j in I_i} D^b B_j = [b=0] on Q_i."""
    ks = [uniform_open_knots(p, E)] * d
    ctrl = control_net("grid", p, ks, 0.1, seed=3)
    o = Oracle(p, ks, ctrl)
    ptr, col, val, kappa, scale = o.rows(STIFFNESS, np.arange(o.ndof))
    for r in range(o.ndof):
        s = val[ptr[r]:ptr[r + 1]].sum()
        assert abs(s) <= 1e-14 * scale[r] * (ptr[r + 1] - ptr[r])


def test_mass_row_sums_affine():
    """P6: affine F with |det J| = c0: sum_j m~_ij = c0 prod_l (xi_{i+p+1}-xi_i)/(p+1)."""
    p, E = 3, 5
    A = np.array([[1.2, 0.3, 0.0], [0.0, 0.8, 0.1], [0.2, 0.0, 1.1]])
    ks = [graded_open_knots(p, E), uniform_open_knots(p, E), graded_open_knots(p, E + 1)]
    ctrl = control_net("affine:" + ",".join(map(str, A.ravel())), p, ks, 0.0)
    o = Oracle(p, ks, ctrl)
    c0 = abs(np.linalg.det(A))
    ptr, col, val, _, _ = o.rows(MASS, np.arange(o.ndof))
    for r in range(o.ndof):
        ii = np.unravel_index(r, o.n, order="F")
        ref = c0 * np.prod([(ks[l][ii[l] + p + 1] - ks[l][ii[l]]) / (p + 1) for l in range(3)])
        assert abs(val[ptr[r]:ptr[r + 1]].sum() - ref) <= 1e-15 * max(ref, 1e-300) * 50


def test_nonaffine_asymmetric():
    """P12: for non-affine F the WQ matrices are not symmetric (Remark P:919-921)."""
    p, E = 2, 5
    ks = [uniform_open_knots(p, E)] * 2
    o = Oracle(p, ks, control_net("annulus", p, ks, 0.0))
    for mat in (MASS, STIFFNESS):
        A = o.dense(mat)
        asym = np.abs(A - A.T).max() / np.abs(A).max()
        assert asym > 1e-6


def test_kappa_interior_small():
    """kappa_i ~ 1 for interior rows (no cancellation), larger near the boundary."""
    p, E = 4, 12
    ks = [uniform_open_knots(p, E)] * 3
    o = Oracle(p, ks, control_net("grid", p, ks, 0.1))
    n = o.n[0]
    mid = n // 2
    rows = [mid + n * (mid + n * mid), 0]
    _, _, _, kappa, _ = o.rows(STIFFNESS, rows)
    assert kappa[0] < 20 and kappa[1] > kappa[0]
