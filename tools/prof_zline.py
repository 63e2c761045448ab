"""Per-warp wait accounting of the z-line kernel (debug build with -DWQ_ZL_PROF).
Usage: nvcc ... -DWQ_ZL_PROF -o /tmp/libwq_prof.so csrc/*.cu; WQ_LIB_DEBUG_PATH=/tmp/libwq_prof.so WQ_ZL_PROF=1 python tools/prof_zline.py --p 4
Producers (warp % 4 in {0,1}): wait1 = TMA box (pfull), wait2 = free ring slot (gempty).
Consumers (warp % 4 in {2,3}): wait1 = G ready (gfull), wait2 = weight prefetch (wfull)."""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import baseline_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=4)
ap.add_argument("--config", default="C4")
ap.add_argument("--slab", default="0,-1", help="planes [b,e) of the slowest index (one rank of a multi-GPU run)")
a = ap.parse_args()
cfg = baseline_config(a.config, a.p)
plan = wq.Plan(cfg.p, cfg.knots(), slab=tuple(int(x) for x in a.slab.split(",")), need_mass=False,
               need_stiffness=True)
ctrl = torch.from_numpy(cfg.ctrl()).cuda()
rp, col, val = plan.alloc_csr()
for _ in range(2):
    plan.form(wq.WQ_STIFFNESS, ctrl, out=(rp, col, val))
torch.cuda.synchronize()
lib = wq.load_library()
n = 3 * 148 * 32 * 3
buf = (C.c_ulonglong * n)()
assert lib.wq_debug_zprof(buf, n) == 0
A = np.frombuffer(buf, dtype=np.uint64).reshape(3, 148, 32, 3).astype(np.float64)
for k, name in enumerate(("uni", "int", "bnd")):
    B = A[k]
    live = B[:, :, 0] > 0
    if not live.any():
        continue
    warps = np.arange(32)
    for role, sel in (("producer", (warps % 4) < 2), ("consumer", (warps % 4) >= 2)):
        m = live & sel[None, :]
        if not m.any():
            continue
        tot = B[:, :, 0][m].mean()
        w1 = B[:, :, 1][m].mean() / tot
        w2 = B[:, :, 2][m].mean() / tot
        print(f"{name} {role}: cycles {tot:.3g}  wait1 {w1:.1%}  wait2 {w2:.1%}")
    tot_blk = B[:, :, 0].max(axis=1)
    print(f"{name} per-CTA cycles: max {tot_blk.max():.3g} mean {tot_blk[tot_blk > 0].mean():.3g}")
