"""Time one rank's assembly (CUDA events) for the slab decomposition of an N-GPU run, on one GPU."""
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
ap.add_argument("--layout", type=int, default=0, help="coefficient layout: 0 library choice (z-line), 1 standard")
a = ap.parse_args()
cfg = baseline_config(a.config, a.p)
ctrl = torch.from_numpy(cfg.ctrl()).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for w in [int(x) for x in a.world.split(",")]:
    cuts = slab_cuts(cfg.n_el + cfg.p, cfg.p, w)
    worst = 0.0
    for rank in sorted({0, w // 2, w - 1}):
        plan = wq.Plan(cfg.p, cfg.knots(), slab=(cuts[rank], cuts[rank + 1]), need_mass=False, need_stiffness=True,
                       coef_layout=a.layout)
        rp, col, val = plan.alloc_csr()
        plan.setup(ctrl)
        wq.wq_pattern(plan.h, 0, rp, None)
        ts = []
        for _ in range(4):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            wq.wq_assemble(plan.h, wq.WQ_STIFFNESS, val, col)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[len(ts) // 2]
        worst = max(worst, t)
        print(json.dumps({"world": w, "rank": rank, "planes": [int(cuts[rank]), int(cuts[rank + 1])],
                          "nnz_local": plan.info["nnz_local"], "asm_ms": t}))
        plan.close()
        del rp, col, val
    print(json.dumps({"world": w, "max_rank_asm_ms": worst}))
