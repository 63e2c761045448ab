"""Time the steps of the hot path separately (CUDA events, L2 flushed between reps, median)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--matrix", default="stiffness")
a = ap.parse_args()
cfg = baseline_config(a.config, a.p)
mat = wq.WQ_STIFFNESS if a.matrix == "stiffness" else wq.WQ_MASS
plan = wq.Plan(cfg.p, cfg.knots(), ctrl=cfg.ctrl(), need_mass=mat == 0, need_stiffness=mat == 1)
d_ctrl = torch.from_numpy(cfg.ctrl()).cuda()
rp, col, val = plan.alloc_csr()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
parts = {"rules": lambda: wq.wq_build_rules(plan.h), "coef": lambda: wq.wq_build_coef(plan.h, d_ctrl),
         "pattern": lambda: wq.wq_pattern(plan.h, 0, rp), "assemble": lambda: wq.wq_assemble(plan.h, mat, val, col)}
out = {"cfg": cfg.name}
for k, f in parts.items():
    f()
    ts = []
    for _ in range(a.reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[k] = sorted(ts)[len(ts) // 2]
print(json.dumps(out))
