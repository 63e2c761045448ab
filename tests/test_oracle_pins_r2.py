"""Round-2 pins of the CPU oracle (no GPU): scalar PDE coefficients (reading
R17), boundary-row minimum-norm weights, and the roundoff amplification
kappa_i used by the parity tolerance (reading R6).

As in test_oracle_pins.py, every test names the passage of PAPER.md ("P:<line>")
or the mathematical fact it uses; none re-types the oracle's formulas.
"""
import json
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
from oracle import MASS, STIFFNESS, Oracle
from wqinputs import control_net, graded_open_knots, greville, uniform_open_knots

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _tensor_greville(p, ks):
    """[N_DOF][d] Greville abscissae of the tensor basis (k_1 fastest)."""
    gs = [greville(p, k) for k in ks]
    mesh = np.meshgrid(*gs, indexing="ij")
    return np.stack([m.reshape(-1, order="F") for m in mesh], axis=1)


def _int_B(k, p, i):
    """int B_i = (xi_{i+p+1} - xi_i) / (p+1) (standard B-spline identity)."""
    return (k[i + p + 1] - k[i]) / (p + 1)


def _centroid(k, p, i):
    """int zeta B_i / int B_i = (xi_i + ... + xi_{i+p+1}) / (p+2) (standard identity)."""
    return sum(k[i:i + p + 2]) / (p + 2)


# ------------------------------------------------------ coefficients (R17)
def test_coefficient_example_printed_whole_pipeline():
    """P3 through the whole mass pipeline: P:391-402 apply the p = 3 rule of an
    interior row (h = 2, points x = 1..7) to c(zeta) = zeta.  With the identity
    geometry (control points = Greville abscissae, Marsden's identity) and the
    reaction coefficient gamma(zeta) = zeta (coefficients = Greville abscissae),
    the WQ mass entries m~_{i,i+1} and m~_{i+1,i} are exactly the paper's two
    printed sums (rational terms in tests/golden, 2.3647 / 2.3615)."""
    g = GOLD["asymmetry_example"]
    k = np.array([-10.0] * 4 + [float(x) for x in range(-8, 20, 2)] + [20.0] * 4)
    gv = greville(3, k)
    o = Oracle(3, [k], gv.reshape(-1, 1), gamma=gv)
    i, j = 8, 9  # supports (0, 8) and (2, 10)
    ptr, col, val, _, _ = o.rows(MASS, np.array([i, j]))
    m_ij = val[ptr[0]:ptr[1]][list(col[ptr[0]:ptr[1]]).index(j)]
    m_ji = val[ptr[1]:ptr[2]][list(col[ptr[1]:ptr[2]]).index(i)]
    exact_i = float(sum(Fr(*a) * b * Fr(*c) for a, b, c in g["Qi_cBj_terms"]))
    exact_j = float(sum(Fr(*a) * b * Fr(*c) for a, b, c in g["Qj_cBi_terms"]))
    assert abs(m_ij - exact_i) < 1e-13 and abs(m_ji - exact_j) < 1e-13
    assert abs(m_ij - g["Qi_cBj_printed"]) < 0.5e-4 and abs(m_ji - g["Qj_cBi_printed"]) < 0.5e-4


@pytest.mark.parametrize("d,p,E", [(2, 2, 5), (3, 3, 3)])
def test_constant_coefficients_scale(d, p, E):
    """Constant coefficient nets reproduce the constants (partition of unity,
    P:359): kappa = 2.5 scales S~ by 2.5, gamma = 0.75 scales M~ by 0.75."""
    ks = [uniform_open_knots(p, E)] * d
    ctrl = control_net("grid", p, ks, 0.1, seed=5)
    n = int(np.prod([len(k) - p - 1 for k in ks]))
    o1 = Oracle(p, ks, ctrl)
    o2 = Oracle(p, ks, ctrl, kappa=np.full(n, 2.5), gamma=np.full(n, 0.75))
    rows = np.arange(n)
    for mat, fac in ((STIFFNESS, 2.5), (MASS, 0.75)):
        _, _, v1, _, _ = o1.rows(mat, rows)
        _, _, v2, _, _ = o2.rows(mat, rows)
        np.testing.assert_allclose(v2, fac * v1, rtol=0, atol=1e-14 * np.abs(v1).max())


def test_mass_row_sums_affine_coefficient():
    """Affine F (|det J| = c0) and gamma affine in zeta: the WQ rows of each
    test function integrate every spline of the trial space exactly (Eq. exact,
    P:613-620), and 1, zeta_l are such splines, so
      sum_j m~_ij = c0 gamma(centroid_i) prod_l int B_{i_l}
    with centroid_l = (xi_{i_l} + .. + xi_{i_l+p+1})/(p+2) -- every row, incl.
    boundary rows, graded knots."""
    p, E = 3, 4
    A = np.array([[1.1, 0.2, 0.0], [0.1, 0.9, 0.0], [0.0, 0.3, 1.3]])
    ks = [graded_open_knots(p, E), uniform_open_knots(p, E), graded_open_knots(p, E + 1)]
    ctrl = control_net("affine:" + ",".join(map(str, A.ravel())), p, ks, 0.0)
    G = _tensor_greville(p, ks)
    a = np.array([0.7, 0.4, -0.3, 0.25])
    gam = a[0] + G @ a[1:]
    o = Oracle(p, ks, ctrl, gamma=gam)
    c0 = abs(np.linalg.det(A))
    ptr, col, val, _, _ = o.rows(MASS, np.arange(o.ndof))
    for r in range(o.ndof):
        ii = np.unravel_index(r, o.n, order="F")
        cen = np.array([_centroid(ks[l], p, ii[l]) for l in range(3)])
        ref = c0 * (a[0] + cen @ a[1:]) * np.prod([_int_B(ks[l], p, ii[l]) for l in range(3)])
        assert abs(val[ptr[r]:ptr[r + 1]].sum() - ref) <= 1e-14 * abs(ref) * 20, r


def test_stiffness_kappa_linear_moment():
    """Identity geometry (C = kappa I) and kappa affine: applying S~ to the
    coefficients of u = zeta_1 (Greville abscissae, Marsden) leaves only the
    direction-1 term, whose family (1,1) integrates the degree p-1 spline
    kappa against B_i' exactly (Eq. exact), so for rows with 1 <= i_1 <= n-2
      sum_j s~_ij gamma_{j,1} = int kappa dB_i/dzeta_1 = -g_1 prod_l int B_{i_l}
    (integration by parts, B_i = 0 at zeta_1 = 0, 1).  Also sum_j s~_ij = 0."""
    p, E = 3, 4
    ks = [uniform_open_knots(p, E), graded_open_knots(p, E), uniform_open_knots(p, E + 1)]
    G = _tensor_greville(p, ks)
    g = np.array([1.3, 0.45, -0.2, 0.35])
    kap = g[0] + G @ g[1:]
    o = Oracle(p, ks, G, kappa=kap)
    ptr, col, val, kappa_i, scale = o.rows(STIFFNESS, np.arange(o.ndof))
    u = G[:, 0]
    n1 = o.n[0]
    for r in range(o.ndof):
        ii = np.unravel_index(r, o.n, order="F")
        s = val[ptr[r]:ptr[r + 1]]
        assert abs(s.sum()) <= 1e-14 * scale[r] * len(s)
        if 1 <= ii[0] <= n1 - 2:
            ref = -g[1] * np.prod([_int_B(ks[l], p, ii[l]) for l in range(3)])
            got = float(s @ u[col[ptr[r]:ptr[r + 1]]])
            assert abs(got - ref) <= 1e-13 * scale[r], (r, got, ref)


# -------------------------------------------- boundary-row minimum norm
@pytest.mark.parametrize("p", [2, 3, 4, 5, 6])
def test_boundary_rows_minnorm_mpmath(p):
    """Rows 0..p (boundary rows: #Q_i = p+1+2i > #I_i, so the exact rule is
    not unique and the min-norm member is the paper's choice, Remark 2
    P:675-679; for b = 1 the system has rank #I-1, reading R4) of all four
    families equal a 40-digit pseudo-inverse solution built from an
    independent mpmath Cox-de Boor recursion on the same knots and the same
    (FP64) points, with integrals by a 40-digit (p+1)-point Gauss rule span by span."""
    import mpmath as mp
    mp.mp.dps = 40
    E = 3 * p + 4
    k = uniform_open_knots(p, E)
    K = [mp.mpf(float(x)) for x in k]
    n = len(k) - p - 1

    def bspl(i, q, x):  # degree q B-spline i on K, right-continuous, x inside (0, 1)
        if q == 0:
            return mp.mpf(1) if K[i] <= x < K[i + 1] else mp.mpf(0)
        v = mp.mpf(0)
        if K[i + q] > K[i]:
            v += (x - K[i]) / (K[i + q] - K[i]) * bspl(i, q - 1, x)
        if K[i + q + 1] > K[i + 1]:
            v += (K[i + q + 1] - x) / (K[i + q + 1] - K[i + 1]) * bspl(i + 1, q - 1, x)
        return v

    def dbspl(i, x):
        v = mp.mpf(0)
        if K[i + p] > K[i]:
            v += p / (K[i + p] - K[i]) * bspl(i, p - 1, x)
        if K[i + p + 1] > K[i + 1]:
            v -= p / (K[i + p + 1] - K[i + 1]) * bspl(i + 1, p - 1, x)
        return v

    # (p+1)-point Gauss-Legendre rule in 40 digits (Newton on P_{p+1} from the float64 nodes): exact
    # for the degree-2p integrands on every span
    m = p + 1
    gx, gw = [], []
    for x0 in np.polynomial.legendre.leggauss(m)[0]:
        x = mp.mpf(float(x0))
        for _ in range(8):
            Pm, Pm1 = mp.legendre(m, x), mp.legendre(m - 1, x)
            dP = m * (x * Pm - Pm1) / (x * x - 1)
            x -= Pm / dP
        gx.append(x)
        gw.append(2 / ((1 - x * x) * dP * dP))

    def quad(fn, lo, hi):
        return (hi - lo) / 2 * sum(wg * fn((lo + hi) / 2 + (hi - lo) / 2 * xg) for xg, wg in zip(gx, gw))

    o = Oracle(p, [k])
    D = o.direction(0)
    for i in range(p + 1):
        q0, nq = int(D["qlo"][i]), int(D["qlen"][i])
        xs = [mp.mpf(float(x)) for x in D["points"][q0:q0 + nq]]
        js = list(range(max(0, i - p), min(n - 1, i + p) + 1))
        spans = [(K[e], K[e + 1]) for e in range(len(K) - 1) if K[e + 1] > K[e]]
        for f, (a, b) in enumerate(oracle.FAMILIES):
            fa = (lambda x: dbspl(i, x)) if a else (lambda x: bspl(i, p, x))
            M = mp.matrix([[dbspl(j, x) if b else bspl(j, p, x) for x in xs] for j in js])
            rhs = []
            for j in js:
                fb = (lambda x, j=j: dbspl(j, x)) if b else (lambda x, j=j: bspl(j, p, x))
                rhs.append(sum(quad(lambda x: fa(x) * fb(x), lo, hi) for lo, hi in spans
                               if lo < K[i + p + 1] and hi > K[i]))
            U, S, V = mp.svd_r(M)
            tol = mp.mpf(10) ** -25 * max(S)
            Sp = mp.diag([1 / sv if sv > tol else 0 for sv in S])
            w = V.T * Sp * U.T * mp.matrix(rhs)
            w = np.array([float(v) for v in w])
            got = D["w"][i, f, :nq]
            np.testing.assert_allclose(got, w, rtol=0, atol=2e-14 * np.abs(w).max(), err_msg=f"row {i} fam {f}")


# ---------------------------------------------------------------- kappa_i
@pytest.mark.parametrize("mat", [MASS, STIFFNESS])
def test_kappa_recomputed_from_tables(mat):
    """kappa_i = max_j sum_q |term_ijq| / max_j |sum_q term_ijq| (reading R6)
    and the row values, recomputed in numpy from the oracle's exported rules
    (weights, basis tables) and coefficient field for rows in every boundary
    situation of a 3D p = 3 problem."""
    p, E = 3, 5
    ks = [uniform_open_knots(p, E)] * 3
    ctrl = control_net("annulus", p, ks, 0.05, seed=2)
    o = Oracle(p, ks, ctrl)
    Ds = [o.direction(l) for l in range(3)]
    n = o.n[0]
    rows = [0, 1 + n * 2, n // 2 * (1 + n + n * n), (n - 1) + n * (n - 2), n * n * (n - 1) + 3]
    ptr, col, val, kappa, scale = o.rows(mat, np.array(rows))
    for k, r in enumerate(rows):
        ii = np.unravel_index(r, o.n, order="F")
        q0 = [int(Ds[l]["qlo"][ii[l]]) for l in range(3)]
        nq = [int(Ds[l]["qlen"][ii[l]]) for l in range(3)]
        j0 = [int(Ds[l]["jlo"][ii[l]]) for l in range(3)]
        nj = [int(Ds[l]["jlen"][ii[l]]) for l in range(3)]
        cb, _, st = o.coef_box(q0, [q0[l] + nq[l] for l in range(3)])
        cb = cb.reshape(nq[2], nq[1], nq[0], 10)  # q_3 slowest
        pairs = [(None, None)] if mat == MASS else [(l, m) for l in range(3) for m in range(3)]
        tot = np.zeros((nj[2], nj[1], nj[0]))
        abs_sum = np.zeros((nj[2], nj[1], nj[0]))
        for (lt, mt) in pairs:
            fac = []
            for l in range(3):
                a = 0 if mat == MASS else int(l == lt)
                b = 0 if mat == MASS else int(l == mt)
                w = Ds[l]["w"][ii[l], a + 2 * b, :nq[l]]
                B = (Ds[l]["Bd"] if b else Ds[l]["Bv"])[q0[l]:q0[l] + nq[l], j0[l]:j0[l] + nj[l]]
                fac.append((w[:, None] * B).T)  # [j, q] = w_q D^b B_j(x_q)
            cf = cb[..., 0] if mat == MASS else cb[..., 1 + 3 * lt + mt]
            t = np.einsum("aq,br,cs,srq->cbasrq", fac[0], fac[1], fac[2], cf)  # [j3, j2, j1, q3, q2, q1]
            tot += t.sum(axis=(3, 4, 5))
            abs_sum += np.abs(t).sum(axis=(3, 4, 5))
        vals = tot.reshape(-1)  # column order: t_1 fastest
        got = val[ptr[k]:ptr[k + 1]]
        np.testing.assert_allclose(got, vals, rtol=0, atol=1e-14 * np.abs(vals).max())
        kap = abs_sum.max() / np.abs(vals).max()
        assert abs(kappa[k] - kap) <= 1e-10 * kap, (r, kappa[k], kap)
        assert abs(scale[k] - abs_sum.max()) <= 1e-12 * abs_sum.max()


@pytest.mark.parametrize("p,E", [(2, 4), (3, 3)])
def test_mass_row_sum_identity_used_by_gpu_tests(p, E):
    """The every-row mass check of tests/test_gpu_zfullsize.py compares device row sums with
    sum_q w1 w2 w3 c(x_q) built from the oracle's weights and coefficient field (partition of unity
    on Q_i, Eq. massquadrature).  Here that helper is checked against the row sums of the
    oracle's dense mass matrix on a perturbed 3D geometry (index order, family, point ranges)."""
    from test_gpu_zfullsize import mass_row_sums_oracle
    ks = [uniform_open_knots(p, E)] * 3
    ctrl = control_net("grid", p, ks, 0.1, seed=0)
    o = Oracle(p, ks, ctrl)
    M = o.dense(MASS)
    w = mass_row_sums_oracle(o).astype(np.float64)
    assert np.abs(M.sum(axis=1) - w).max() <= 1e-13 * np.abs(M).max()
