"""Time the WS kernel under debug ablation masks (WQ_WS_DBG) on one config
(debug helper, not product code).  mask bits: 1 no TMA, 2 no bulk stores,
8 no stage 2, 16 no stage-1 compute."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import torch
    import paper_1605_01238_b200 as wq
    from wqinputs import baseline_config
    p, mat, kern = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    cfg = baseline_config("C4", p)
    plan = wq.Plan(p, cfg.knots(), need_mass=mat == 0, need_stiffness=mat == 1)
    rp, col, val = plan.alloc_csr()
    plan.setup(torch.from_numpy(cfg.ctrl()).cuda())
    wq.wq_pattern(plan.h, 0, rp, None)
    ts = []
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        wq.wq_assemble(plan.h, mat, val, col, kernel=kern)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{min(ts[1:]):.3f}")
    sys.exit(0)
p = sys.argv[1] if len(sys.argv) > 1 else "4"
mat = sys.argv[2] if len(sys.argv) > 2 else "1"
for mask in sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "2", "16", "18", "8", "24", "27"]:
    env = dict(os.environ, WQ_WS_DBG=mask)
    r = subprocess.run([sys.executable, __file__, "child", p, mat, os.environ.get("KERN", "3")], env=env, capture_output=True, text=True, timeout=120)
    print(f"p={p} mat={mat} mask={mask}: {r.stdout.strip() or r.stderr.strip()[-200:]} ms", flush=True)
