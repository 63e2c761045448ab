"""Run a few full hot-path steps on one BASELINE config (for ncu / sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--matrix", default="stiffness")
ap.add_argument("--kernel", type=int, default=0)
a = ap.parse_args()
cfg = baseline_config(a.config, a.p)
mat = wq.WQ_STIFFNESS if a.matrix == "stiffness" else wq.WQ_MASS
plan = wq.Plan(cfg.p, cfg.knots(), ctrl=cfg.ctrl(), need_mass=mat == wq.WQ_MASS, need_stiffness=mat == wq.WQ_STIFFNESS)
ctrl = torch.from_numpy(cfg.ctrl()).cuda()
rp, col, val = plan.alloc_csr()
for _ in range(a.steps):
    plan.form(mat, ctrl, out=(rp, col, val), kernel=a.kernel)
torch.cuda.synchronize()
print("ok", cfg.name, plan.info["nnz_local"])
