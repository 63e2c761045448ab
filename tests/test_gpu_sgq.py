"""GPU element-loop standard Gauss quadrature (SGQ, the paper's comparison method, P:109-116;
SURVEY f2) against the oracle's element-loop Gauss brute force (orc_sgq_dense), every entry, and
the textbook fact that both WQ and SGQ reproduce the exact Galerkin matrices for affine maps
(P:396)."""
import numpy as np
import pytest

import paper_1605_01238_b200 as wq
from oracle import MASS, STIFFNESS, Oracle
from wqinputs import control_net, graded_open_knots, uniform_open_knots

pytestmark = pytest.mark.gpu


def _dense_from_csr(rp, col, val, n):
    A = np.zeros((n, n))
    for r in range(n):
        A[r, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
    return A


def run_sgq(p, ks, ctrl, mat, kappa=None, gamma=None, slab=(0, -1)):
    import torch
    plan = wq.Plan(p, ks, slab=slab, need_mass=True, need_stiffness=True)
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp)
    dk = None if kappa is None else torch.from_numpy(kappa).cuda()
    dg = None if gamma is None else torch.from_numpy(gamma).cuda()
    wq.wq_assemble_sgq(plan.h, mat, torch.from_numpy(ctrl).cuda(), val, col, d_kappa=dk, d_gamma=dg)
    torch.cuda.synchronize()
    info = plan.info
    plan.close()
    return rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy(), info


@pytest.mark.parametrize("d,p,E,geom", [(1, 1, 5, "grid"), (1, 4, 6, "grid"), (2, 2, 4, "annulus"),
                                        (2, 3, 5, "grid"), (3, 2, 3, "grid"), (3, 3, 3, "annulus"),
                                        (3, 1, 4, "grid"), (3, 5, 1, "grid")])
@pytest.mark.parametrize("mat", [MASS, STIFFNESS])
def test_sgq_matches_oracle(d, p, E, geom, mat):
    ks = [(graded_open_knots if l % 2 else uniform_open_knots)(p, E + l) for l in range(d)]
    ctrl = control_net(geom, p, ks, 0.05, seed=4)
    n = ctrl.shape[0]
    rng = np.random.default_rng(1)
    kap = 1.0 + rng.uniform(size=n) if d == 3 else None
    gam = 0.5 + rng.uniform(size=n) if d == 3 else None
    o = Oracle(p, ks, ctrl, kappa=kap, gamma=gam)
    ref = o.sgq_dense(mat)
    rp, col, val, info = run_sgq(p, ks, ctrl, mat, kap, gam)
    orp, ocol = o.pattern()
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol)
    A = _dense_from_csr(rp, col, val, n)
    scale = np.abs(ref).max(axis=1, keepdims=True)
    assert np.all(np.abs(A - ref) <= 1e-12 * scale)
    # nothing outside the pattern in the oracle either
    mask = np.zeros_like(ref, dtype=bool)
    for r in range(n):
        mask[r, col[rp[r]:rp[r + 1]]] = True
    assert np.all(ref[~mask] == 0)


@pytest.mark.parametrize("mat", [MASS, STIFFNESS])
def test_sgq_equals_wq_affine(mat):
    """For an affine map both quadratures are exact: SGQ == WQ to roundoff."""
    import torch
    p, E = 3, 4
    A = [[1.2, 0.3, 0.0], [0.0, 0.8, 0.1], [0.2, 0.0, 1.1]]
    ks = [uniform_open_knots(p, E), graded_open_knots(p, E + 1), uniform_open_knots(p, E + 2)]
    ctrl = control_net("affine:" + ",".join(str(x) for r in A for x in r), p, ks, 0.0)
    rp, col, val, info = run_sgq(p, ks, ctrl, mat)
    plan = wq.Plan(p, ks, ctrl=ctrl)
    rp2, col2, val2 = plan.form(mat)
    torch.cuda.synchronize()
    plan.close()
    v2 = val2.cpu().numpy()
    for r in range(len(rp) - 1):
        s = slice(rp[r], rp[r + 1])
        assert np.abs(val[s] - v2[s]).max() <= 1e-13 * np.abs(v2[s]).max()


def test_sgq_slabs():
    """SGQ on slab plans (rows of the slab only; elements that straddle the seam contribute to both)
    concatenates to the single-plan result (up to atomic summation order)."""
    p, E = 2, 5
    ks = [uniform_open_knots(p, E)] * 3
    ctrl = control_net("grid", p, ks, 0.1, seed=2)
    rp0, col0, val0, _ = run_sgq(p, ks, ctrl, STIFFNESS)
    vals = []
    for sl in ((0, 3), (3, 7)):
        rp, col, val, info = run_sgq(p, ks, ctrl, STIFFNESS, slab=sl)
        vals.append(val)
    v = np.concatenate(vals)
    assert np.abs(v - val0).max() <= 1e-14 * np.abs(val0).max()
