"""Time wq_build_coef (CUDA events) on a BASELINE config for both coefficient layouts."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--config", default="C4")
a = ap.parse_args()
cfg = baseline_config(a.config, a.p)
ctrl = torch.from_numpy(cfg.ctrl()).cuda()
for layout in (0, 1):
    plan = wq.Plan(cfg.p, cfg.knots(), need_mass=False, need_stiffness=True, coef_layout=layout)
    wq.wq_build_rules(plan.h)
    ts = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        wq.wq_build_coef(plan.h, ctrl)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    wq.wq_build_rules(plan.h)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"layout": layout, "coef_ms": sorted(ts)[3], "rules_ms": e0.elapsed_time(e1)}))
    plan.close()
