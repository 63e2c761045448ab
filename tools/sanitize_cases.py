"""Small cases through every product kernel path, for compute-sanitizer (memcheck / initcheck /
racecheck / synccheck):

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_cases.py

Each case runs the whole hot path (rules, coefficient field, pattern, values) through the C-ABI and
reads one checksum back, so that every launch of the case has completed before the next one starts.
No oracle here: parity is the tests' job; this script only gives the sanitizer the launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import control_net, graded_open_knots, uniform_open_knots  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--only", default="", help="comma-separated case names (default: all)")
a = ap.parse_args()
only = set(x for x in a.only.split(",") if x)

M, S = wq.WQ_MASS, wq.WQ_STIFFNESS
# name, d, p, E, knots, matrices, slab, coefficient fields
CASES = [
    ("z3p2", 3, 2, 12, "uniform", (S, M), (0, -1), False),   # z-line (uniform / interior / boundary lines), tile
    ("z3p3", 3, 3, 14, "uniform", (S, M), (0, -1), False),
    ("z3p4", 3, 4, 18, "uniform", (S, M), (0, -1), True),    # z-line, ZHP mass, kappa / gamma folded in
    ("z3p5", 3, 5, 12, "uniform", (S, M), (0, -1), False),   # ZHP stiffness
    ("z3p6", 3, 6, 26, "uniform", (S,), (3, 9), False),      # z-line at p = 6 on a slab
    ("h3p7", 3, 7, 9, "uniform", (S, M), (0, -1), False),    # ZHP, high degree
    ("h3p10", 3, 10, 6, "uniform", (S,), (0, -1), False),
    ("g3p3", 3, 3, 10, "graded", (S, M), (2, 9), False),     # graded knots (table paths), slab
    ("s2p3", 2, 3, 40, "uniform", (S, M), (0, -1), True),    # d = 2 chunked-line kernel
    ("s2p9", 2, 9, 14, "graded", (S, M), (0, -1), False),    # d = 2, one entry per lane
    ("s1p4", 1, 4, 64, "uniform", (S, M), (0, -1), False),
]


def run_case(name, d, p, E, kn, mats, slab, coef):
    k1 = uniform_open_knots(p, E) if kn == "uniform" else graded_open_knots(p, E)
    knots = [k1] * d
    ctrl = control_net("grid", p, knots, 0.1, seed=1)
    n = ctrl.shape[0]
    rng = np.random.default_rng(7)
    kap = torch.from_numpy(1.0 + 0.5 * rng.random(n)).cuda() if coef else None
    gam = torch.from_numpy(1.0 + 0.5 * rng.random(n)).cuda() if coef else None
    d_ctrl = torch.from_numpy(ctrl).cuda()
    plan = wq.Plan(p, knots, slab=slab, need_mass=M in mats, need_stiffness=S in mats)
    out = []
    for mat in mats:
        rp, col, val = plan.form(mat, d_ctrl, d_kappa=kap, d_gamma=gam)
        torch.cuda.synchronize()
        out.append((int(rp[-1] - rp[0]), float(val.abs().sum())))
        assert torch.isfinite(val).all(), f"{name}: non-finite value"
    # standalone column pattern
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp, col)
    torch.cuda.synchronize()
    plan.close()
    return out


def run_sgq():
    p, E, d = 2, 4, 3
    knots = [uniform_open_knots(p, E)] * d
    ctrl = control_net("grid", p, knots, 0.1, seed=2)
    plan = wq.Plan(p, knots)
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp, None)
    for mat in (M, S):
        wq.wq_assemble_sgq(plan.h, mat, torch.from_numpy(ctrl).cuda(), val, col)
        torch.cuda.synchronize()
    plan.close()
    return float(val.abs().sum())


def run_form_host():
    p, E, d = 3, 12, 3
    knots = [uniform_open_knots(p, E)] * d
    ctrl = control_net("grid", p, knots, 0.1, seed=3)
    plan = wq.Plan(p, knots, need_mass=False)
    info = plan.info
    h_rp = torch.empty(info["n_rows_local"] + 1, dtype=torch.int64).pin_memory()
    h_col = torch.empty(info["nnz_local"], dtype=torch.int32).pin_memory()
    h_val = torch.empty(info["nnz_local"], dtype=torch.float64).pin_memory()
    wq.wq_form_host(plan.h, S, np.ascontiguousarray(ctrl), 0, h_rp, h_col, h_val)
    plan.close()
    return float(h_val.abs().sum())


for c in CASES:
    if only and c[0] not in only:
        continue
    print(c[0], run_case(*c), flush=True)
if not only or "sgq" in only:
    print("sgq", run_sgq(), flush=True)
if not only or "form_host" in only:
    print("form_host", run_form_host(), flush=True)
print("sanitize_cases: ok")
