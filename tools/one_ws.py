"""Run the WS kernel once on a small case (debug helper; not product code)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import baseline_config, control_net, uniform_open_knots  # noqa: E402

p, E, mat = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kernel = int(sys.argv[5]) if len(sys.argv) > 5 else wq.WQ_KERNEL_WS
if len(sys.argv) > 4 and sys.argv[4] != "-":
    cfg = baseline_config(sys.argv[4], p)
    ks, ctrl = cfg.knots(), cfg.ctrl()
else:
    ks = [uniform_open_knots(p, E)] * 3
    ctrl = control_net("grid", p, ks, 0.05, seed=0)
plan = wq.Plan(p, ks, need_mass=True, need_stiffness=True)
rp, col, val = plan.alloc_csr()
plan.setup(torch.from_numpy(ctrl).cuda())
wq.wq_pattern(plan.h, 0, rp, None)
wq.wq_assemble(plan.h, mat, val, col, kernel=kernel)
torch.cuda.synchronize()
print("ok", p, E, mat, float(val.abs().max()))
