"""Time the row-block kernels (CUDA events, L2 flushed, median of reps) on BASELINE configs."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import Config, baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", default="2,3,4")
ap.add_argument("--kernels", default="3,4")
ap.add_argument("--matrix", default="stiffness")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--config", default="C4")
ap.add_argument("--nel", type=int, default=0, help="override n_el (grid geometry)")
ap.add_argument("--d", type=int, default=3, help="dimension with --nel")
a = ap.parse_args()
mat = wq.WQ_STIFFNESS if a.matrix == "stiffness" else wq.WQ_MASS
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for p in [int(x) for x in a.p.split(",")]:
    cfg = baseline_config(a.config, p) if not a.nel else Config(f"G{a.d}d{a.nel}p{p}", a.d, p, a.nel, "grid", 0.1)
    plan = wq.Plan(cfg.p, cfg.knots(), ctrl=cfg.ctrl(), need_mass=mat == wq.WQ_MASS,
                   need_stiffness=mat == wq.WQ_STIFFNESS)
    rp, col, val = plan.alloc_csr()
    wq.wq_pattern(plan.h, 0, rp, None)
    ref = None
    for k in [int(x) for x in a.kernels.split(",")]:
        try:
            wq.wq_assemble(plan.h, mat, val, col, kernel=k)
            torch.cuda.synchronize()
        except wq.WQError as e:
            print(json.dumps({"p": p, "kernel": k, "error": str(e)[:120]}))
            continue
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            wq.wq_assemble(plan.h, mat, val, col, kernel=k)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        wq.wq_check(plan.h)
        nnz = plan.info["nnz_local"]
        ms = sorted(ts)[len(ts) // 2]
        v = val[:: max(1, nnz // 4000000)].clone()
        diff = None if ref is None else float((v - ref).abs().max() / ref.abs().max())
        if ref is None:
            ref = v
        print(json.dumps({"cfg": cfg.name, "p": p, "mat": a.matrix, "kernel": wq.KERNEL_NAMES[k] if k else "auto:" + wq.KERNEL_NAMES[plan.info["kernel"][mat]], "ms": round(ms, 3),
                          "nnz": nnz, "Gnnz_s": round(nnz / ms / 1e6, 1), "GBs": round(12 * nnz / ms / 1e6, 1),
                          "hbm_frac": round(12 * nnz / ms / 1e6 / 6552.6, 3), "rel_diff_vs_first": diff, "csum": float(v.sum())}), flush=True)
    plan.close()
    del rp, col, val
    torch.cuda.empty_cache()
