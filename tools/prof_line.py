"""Per-warp cycle accounting of the line kernel (debug helper): WQ_LINE_PROF=1."""
import ctypes as C
import os
import sys

os.environ["WQ_LINE_PROF"] = "1"
os.environ.setdefault("WQ_LINE_ONLY", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import subprocess  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1605_01238_b200 as wq  # noqa: E402
from wqinputs import baseline_config  # noqa: E402

_cs = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1605_01238_b200", "csrc")
_lib = "/tmp/libwq_linedebug.so"
if not os.path.exists(_lib):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-DWQ_LINE_DEBUG",
                    "-Xcompiler", "-fPIC", "-shared", "-diag-suppress", "177", "-o", _lib,
                    *sorted(os.path.join(_cs, f) for f in os.listdir(_cs) if f.endswith(".cu"))], check=True)
wq.load_library(_lib)

p = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = baseline_config("C4", p)
plan = wq.Plan(p, cfg.knots(), need_mass=False, need_stiffness=True)
rp, col, val = plan.alloc_csr()
plan.setup(torch.from_numpy(cfg.ctrl()).cuda())
wq.wq_pattern(plan.h, 0, rp, None)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    wq.wq_assemble(plan.h, wq.WQ_STIFFNESS, val, col, kernel=wq.WQ_KERNEL_LINE)
    e1.record()
    torch.cuda.synchronize()
print("ms", e0.elapsed_time(e1))
lib = wq.load_library()
buf = (C.c_ulonglong * (148 * 32 * 4))()
print("rc", lib.wq_debug_prof(buf, 148 * 32 * 4))
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 11
a = np.frombuffer(buf, dtype=np.uint64)[: 148 * nw * 4].reshape(148, nw, 4).astype(np.float64)
for w in range(nw):
    tot = a[:, w, 0].mean()
    print(f"warp {w:2d}: total {tot/1e6:7.3f} Mcyc  waitA {a[:, w, 1].mean()/tot*100:5.1f}%  waitB {a[:, w, 2].mean()/tot*100:5.1f}%  waitC {a[:, w, 3].mean()/tot*100:5.1f}%")
