"""Per-rank step times of the N-GPU slab decomposition, measured on ONE GPU by running
each rank's slab plan in turn: the whole per-rank step (rules, coefficient field on the slab + halo,
pattern, values; the all-gather of one int64 is not included) with CUDA events, L2 flushed, median
of reps.  The N-GPU step time is the max over the ranks (ranks are independent: P:256-260)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from paper_1605_01238_b200.dist import slab_cuts  # noqa: E402
from wqinputs import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--config", default="C4")
ap.add_argument("--world", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--balance", default="cost", help="slab cuts: cost (default, dist.plane_cost) or nnz")
a = ap.parse_args()
cfg = baseline_config(a.config, a.p)
n = cfg.n_el + cfg.p
ctrl = cfg.ctrl()
d_ctrl = torch.from_numpy(ctrl).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for world in [int(x) for x in a.world.split(",")]:
    cuts = slab_cuts(n, cfg.p, world, a.balance)
    per = []
    for r in range(world):
        plan = wq.Plan(cfg.p, cfg.knots(), ctrl=ctrl, slab=(cuts[r], cuts[r + 1]), need_mass=False)
        rp, col, val = plan.alloc_csr()
        ts, ta = [], []
        for _ in range(a.reps + 1):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            wq.wq_build_rules(plan.h)
            wq.wq_build_coef(plan.h, d_ctrl)
            wq.wq_pattern(plan.h, 0, rp)
            e1.record()
            wq.wq_assemble(plan.h, wq.WQ_STIFFNESS, val, col)
            e2.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e2))
            ta.append(e1.elapsed_time(e2))
        ts, ta = sorted(ts[1:]), sorted(ta[1:])
        per.append((ts[len(ts) // 2], ta[len(ta) // 2], plan.info["nnz_local"]))
        plan.close()
        del rp, col, val
        torch.cuda.empty_cache()
    tmax = max(x[0] for x in per)
    nnz = sum(x[2] for x in per)
    print(json.dumps({"config": cfg.name, "world": world, "balance": a.balance, "cuts": cuts, "step_ms_max": round(tmax, 3),
                      "step_ms_per_rank": [round(x[0], 3) for x in per],
                      "assemble_ms_per_rank": [round(x[1], 3) for x in per],
                      "nnz_per_s": nnz / tmax * 1e3}), flush=True)
