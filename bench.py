#!/usr/bin/env python
"""bench.py -- WQ formation of the IGA stiffness matrix on B200 (arXiv:1605.01238).

One step = the whole hot path over one synthetic input:
  wq_build_rules   point grid, ranges, basis tables, exact integrals, WQ weights
  wq_build_coef    coefficient field C = |det J| J^-1 J^-T on the point grid
  wq_pattern       CSR row_ptr (int64)
  wq_assemble      values (FP64) + fused int32 columns, row-block kernel
  [N>1]            NCCL all-gather of per-rank nnz -> row_ptr base (the only exchange)

Metric (BASELINE.json): CSR nonzeros assembled per second, whole job.
Default workload: BASELINE configs[3] (C4: 3D, 100^3 elements, p=4), the
sweep p = 2,3,4,6,8,10 is reported under "sweep" (--no-sweep to skip).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from wqinputs import C4_DEGREES, baseline_config  # noqa: E402

L2_BYTES = 126 * 1024 * 1024


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    return 6650.0, "fallback (B200_PROFILING.md)", {}


def fp64_peak_tflops(sm_mhz):
    # 148 SMs x 64 FP64 FMA/clk/SM x 2 FLOP; at 1965 MHz 37.2 TF, which the DMMA microbenchmark
    # reaches (37.1 TF) and DFMA nearly (34.2 TF): profiles/r01_fp64_peak.jsonl (tools/fp64_peak.cu)
    return 148 * 64 * 2 * sm_mhz * 1e6 / 1e12


def stiffness_flops(plan_h, p):
    """Algorithmic FLOPs of the stiffness row-block step: (4 S1 + 6 T1) R with
    S1 = sum_i #I_1 #Q_1, T1 = sum_i #Q_1, R = (sum_i #I_i)^2 over the other directions."""
    import paper_1605_01238_b200 as wq
    info = wq.wq_plan_info(plan_h)
    n = info["n_dof"][0]
    R1 = wq.wq_export_rules(plan_h, 0, p)
    qlen = R1["qlen"].astype(np.int64)
    ilen = np.array([min(n - 1, i + p) - max(0, i - p) + 1 for i in range(n)], dtype=np.int64)
    S1, T1 = int((ilen * qlen).sum()), int(qlen.sum())
    R = info["nnz_local"] / int(ilen.sum())
    return (4 * S1 + 6 * T1) * R


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed region.

    NVML (pynvml) polled every ~2 ms from a thread, so that even a ~100 ms timed
    region gets dozens of samples; falls back to `nvidia-smi -lms 100`."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []  # (sm_mhz, reasons_mask)
        self.max_mhz = None
        self.stop = False
        self.proc = None

    def _poll_nvml(self, nv, h):
        while not self.stop:
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.t.start()
            self.mode = "nvml"
        except Exception:
            self.mode = "nvidia-smi"
            q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
            try:
                self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read_smi, daemon=True)
                self.t.start()
            except FileNotFoundError:
                self.proc = None
        return self

    def _read_smi(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            try:
                self.max_mhz = float(f[1])
                self.samples.append((float(f[0]), int(f[2], 16)))
            except (ValueError, IndexError):
                pass

    def __exit__(self, *a):
        self.stop = True
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if hasattr(self, "t"):
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        sm = [x[0] for x in self.samples]
        reasons = sorted({nm for _, m in self.samples for nm, bit in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": self.mode}


# ------------------------------------------------------------------- ours
def run_ours(cfg, steps, warmup, rank, world, device, dist, want_e2e=True, want_roofline=True):
    import torch
    import paper_1605_01238_b200 as wq

    torch.cuda.set_device(device)
    from paper_1605_01238_b200.dist import slab_cuts
    cuts = slab_cuts(cfg.n_el + cfg.p, cfg.p, world)
    knots = cfg.knots()
    ctrl = cfg.ctrl()
    plan = wq.Plan(cfg.p, knots, slab=(cuts[rank], cuts[rank + 1]), need_mass=False, need_stiffness=True,
                   device=device)
    info = plan.info
    wq.wq_build_rules(plan.h)
    flops = stiffness_flops(plan.h, cfg.p)
    stream = torch.cuda.Stream(device)
    d_ctrl = torch.from_numpy(ctrl).to(device)
    rp, col, val = plan.alloc_csr()
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=device)
    nnz_all = torch.zeros(world, dtype=torch.int64, device=device)
    my_nnz = torch.tensor([info["nnz_local"]], dtype=torch.int64, device=device)
    matrix = wq.WQ_STIFFNESS

    def step():
        with torch.cuda.stream(stream):
            wq.wq_build_rules(plan.h, stream)
            wq.wq_build_coef(plan.h, d_ctrl, stream)
            if world > 1:  # the one exchange: all-gather of per-rank nnz -> row_ptr base
                dist.all_gather_into_tensor(nnz_all, my_nnz)
                base = int(nnz_all[:rank].sum().item()) if rank else 0
            else:
                base = 0
            wq.wq_pattern(plan.h, base, rp, None, stream)
            ev_a0.record(stream)
            wq.wq_assemble(plan.h, matrix, val, col, stream)
            ev_a1.record(stream)

    ev_a0 = torch.cuda.Event(enable_timing=True)
    ev_a1 = torch.cuda.Event(enable_timing=True)
    for _ in range(warmup):
        step()
    wq.wq_check(plan.h, stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = wq.wq_launch_count()
    t_steps, t_asm = [], []
    with ClockSampler(device) as clk:
        for _ in range(steps):
            flush.zero_()  # L2 flush between timed iterations (outside the timed interval)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            t_steps.append(e0.elapsed_time(e1) / 1e3)
            t_asm.append(ev_a0.elapsed_time(ev_a1) / 1e3)
    launches = wq.wq_launch_count() - launches0
    wq.wq_check(plan.h, stream)
    t_total = sum(t_steps)
    t_asm_mean = sum(t_asm) / len(t_asm)
    if world > 1:
        tt = torch.tensor([t_total, t_asm_mean], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total, t_asm_max = float(tt[0]), float(tt[1])
        dist.barrier()
    res = dict(nnz=info["nnz_total"], nnz_local=info["nnz_local"], rows_local=info["n_rows_local"], flops=flops,
               t_total=t_total, t_step=t_total / steps, t_asm=t_asm_mean, launches=launches // steps,
               clocks=clk.summary(), coef_points=info["coef_points"], n_dof=info["n_dof_total"])
    # end to end through the public host-buffer call (rank-local block)
    if want_e2e:
        n_rows, nnz_l = info["n_rows_local"], info["nnz_local"]
        hrp = torch.empty(n_rows + 1, dtype=torch.int64).pin_memory()
        hcol = torch.empty(nnz_l, dtype=torch.int32).pin_memory()
        hval = torch.empty(nnz_l, dtype=torch.float64).pin_memory()
        hctrl = torch.from_numpy(ctrl).pin_memory()
        del rp, col, val
        torch.cuda.empty_cache()
        base = int(nnz_all[:rank].sum().item()) if world > 1 else 0
        wq.wq_form_host(plan.h, matrix, hctrl, base, hrp, hcol, hval, stream)  # warm-up
        e_t = []
        e2e_steps = max(1, min(steps, 3))
        for _ in range(e2e_steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            wq.wq_form_host(plan.h, matrix, hctrl, base, hrp, hcol, hval, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            e_t.append(e0.elapsed_time(e1) / 1e3)
        te = sum(e_t)
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        res["e2e"] = dict(t=te / e2e_steps, steps=e2e_steps, h2d=int(hctrl.numel() * 8),
                          d2h=int(nnz_l * 12 + (n_rows + 1) * 8))
    plan.close()
    return res


# ------------------------------------------------------------------- oracle
def run_oracle_sample(cfg, budget_s=20.0, seed=0):
    """Time the CPU oracle (as it stands) on a bounded, seeded row sample."""
    from oracle import STIFFNESS, Oracle
    t0 = time.perf_counter()
    o = Oracle(cfg.p, cfg.knots(), cfg.ctrl())
    t_setup = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    n = cfg.n_el + cfg.p
    done_nnz, t_rows, nrows = 0, 0.0, 0
    batch = 8
    while t_rows < budget_s:
        rows = rng.integers(0, n ** 3, size=batch)
        t1 = time.perf_counter()
        ptr, *_ = o.rows(STIFFNESS, rows)
        dt = time.perf_counter() - t1
        t_rows += dt
        done_nnz += int(ptr[-1])
        nrows += rows.size
        if dt < 0.25 * budget_s / 4:
            batch *= 2
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return dict(value=done_nnz / t_rows, rows=nrows, nnz=done_nnz, t_rows=t_rows, t_setup=t_setup, cores=cores)


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=4, help="C4 degree of the headline line")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--oracle-seconds", type=float, default=20.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = baseline_config("C4", args.p)
    workload = f"C4: 3D Poisson stiffness, p={cfg.p}, C^{cfg.p - 1}, {cfg.n_el}^3 elements, Greville grid + 0.1 h noise"

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_oracle_sample(cfg, args.oracle_seconds)
        per_step = r["t_rows"] / max(1, args.steps)
        line = {"impl": "reference", "metric": "CSR nonzeros assembled/sec (FP64, 3D stiffness)",
                "value": r["value"], "unit": "nnz/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64 (long-double accumulation)",
                "data": "synthetic", "config": {"workload": workload, "nnz": cfg.exact_nnz()},
                "cpu_baseline": {"value": r["value"], "unit": "nnz/s", "cores": r["cores"], "kind": "oracle",
                                 "sample": f"{r['rows']} seeded random rows ({r['nnz']} nnz) of {workload}; "
                                           f"oracle setup {r['t_setup']:.1f} s excluded"},
                "e2e": {"value": r["value"], "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    device = local_rank

    res = run_ours(cfg, args.steps, args.warmup, rank, world, device, dist, want_e2e=not args.no_e2e)
    hbm_peak, peak_src, peaks_doc = peaks()
    nnz = res["nnz"]
    value = nnz * args.steps / res["t_total"]
    # roofline of the dominant kernel (row-block assembly) on this rank
    alg_bytes = 12 * res["nnz_local"] + 8 * res["coef_points"] * 6
    achieved = alg_bytes / res["t_asm"] / 1e9
    sm_mhz = res["clocks"]["sm_mhz"] or peaks_doc.get("clocks_under_load", {}).get("sm_mhz_median", 1320.0)
    fp64 = fp64_peak_tflops(sm_mhz)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(f"C4p{cfg.p}")
    fp64_max = fp64_peak_tflops(res["clocks"]["sm_max_mhz"] or 1965.0)
    t_hbm, t_fp = alg_bytes / (hbm_peak * 1e9), res["flops"] / (fp64_max * 1e12)
    roof = {"bound": "hbm" if t_hbm >= t_fp else "fp64", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
            "frac": achieved / hbm_peak, "traffic": traffic, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg_bytes,
            "algorithmic_bytes": "12 B/nnz (8 value + 4 column) + 48 B per coefficient point read",
            "kernel": "wq_assemble (z-line kernel, p <= 4: uniform / interior / boundary line launches; row-tile kernel for p > 4)",
            "kernel_ms": res["t_asm"] * 1e3, "kernel_share_of_step": res["t_asm"] / res["t_step"],
            "fp64": {"algorithmic_flops_per_launch": res["flops"], "achieved_tflops": res["flops"] / res["t_asm"] / 1e12,
                     "peak_tflops": fp64_max, "frac": res["flops"] / res["t_asm"] / 1e12 / fp64_max,
                     "peak_source": "148 SM x 64 DFMA/clk x 2 at max SM clock (DMMA microbenchmark 37.1 TF)"},
            "roofline_time_ms": max(t_hbm, t_fp) * 1e3, "frac_of_roofline": max(t_hbm, t_fp) / res["t_asm"]}
    line = {"metric": "CSR nonzeros assembled/sec (FP64, 3D, p=2..10) and % of HBM-write roofline",
            "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["t_total"] / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "nnz": nnz, "n_dof": res["n_dof"], "matrix": "stiffness",
                       "csr": "int64 row_ptr, int32 col, f64 val",
                       "parallelism": f"x{3}-slabs over {world} GPU(s)" if world > 1 else "1 GPU",
                       "l2": "256 MB buffer zeroed between timed steps; CSR output >> 126 MB L2"},
            "roofline": roof, "gpu_launches": res["launches"], "clocks": res["clocks"]}
    if "e2e" in res:
        e = res["e2e"]
        line["e2e"] = {"value": nnz / e["t"], "unit": "nnz/s", "h2d_bytes_per_step": e["h2d"],
                       "d2h_bytes_per_step": e["d2h"], "steps": e["steps"],
                       "api": "wq_form_host (pinned host buffers, chunked D2H overlapped with assembly)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        r = run_oracle_sample(cfg, args.oracle_seconds)
        line["cpu_baseline"] = {"value": r["value"], "unit": "nnz/s", "cores": r["cores"], "kind": "oracle",
                                "sample": f"{r['rows']} seeded random rows ({r['nnz']} nnz) of the same workload, "
                                          f"{r['t_rows']:.1f} s; oracle setup {r['t_setup']:.1f} s excluded"}
    if not args.no_sweep and world == 1:
        sweep = []
        for p in C4_DEGREES:
            c = baseline_config("C4", p)
            rr = run_ours(c, 3, 3, rank, world, device, dist, want_e2e=False)
            ab = 12 * rr["nnz_local"] + 8 * rr["coef_points"] * 6
            th, tf_ = ab / (hbm_peak * 1e9), rr["flops"] / (fp64_peak_tflops(1965.0) * 1e12)
            sweep.append({"p": p, "nnz": rr["nnz"], "value": rr["nnz"] / rr["t_step"], "ms_per_step": rr["t_step"] * 1e3,
                          "asm_ms": rr["t_asm"] * 1e3, "hbm_frac": ab / rr["t_asm"] / 1e9 / hbm_peak,
                          "fp64_frac": rr["flops"] / rr["t_asm"] / 1e12 / fp64_peak_tflops(1965.0),
                          "bound": "hbm" if th >= tf_ else "fp64", "frac_of_roofline": max(th, tf_) / rr["t_asm"],
                          "sm_mhz": rr["clocks"]["sm_mhz"]})
            torch.cuda.empty_cache()
        line["sweep"] = sweep
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
