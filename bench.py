#!/usr/bin/env python
"""bench.py -- WQ formation of IGA Galerkin matrices on B200 (arXiv:1605.01238).

One step = the whole hot path over one synthetic input:
  wq_build_rules   point grid, ranges, basis tables, exact integrals, WQ weights
  wq_build_coef    coefficient field C = |det J| J^-1 J^-T (and c) on the point grid
  wq_pattern       CSR row_ptr (int64)
  wq_assemble      values (FP64) + fused int32 columns, row-block kernel
  [N>1]            NCCL all-gather of per-rank nnz -> row_ptr base (the only exchange)

Metric (BASELINE.json): CSR nonzeros assembled per second, whole job.
Default workload: BASELINE configs[3] (C4: 3D, 100^3 elements) at p=4, stiffness.
`--config C1..C5 [--p P] [--matrix mass]` selects another workload; the default
run also reports a "sweep" (C4 p=2..10, C2 S+M, C3, C5, the paper's mass shapes
20^3/40^3 p=1..10, and WQ vs the standard element-loop Gauss quadrature).

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

from wqinputs import C4_DEGREES, Config, baseline_config  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
# BASELINE.json "metric", printed identically by both arms
METRIC = "CSR nonzeros assembled/sec (FP64, 3D, p=2..10) and % of HBM-write roofline"


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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def alg_flops(plan_h, p, matrix):
    """Algorithmic FLOPs of the row-block step, exact over the grid:
    stiffness (4 S1 + 6 T1) R, mass 2 S1 R, with S1 = sum_i #I_1 #Q_1, T1 = sum_i #Q_1 over
    direction 1 and R = nnz_local / sum_i #I_1."""
    import paper_1605_01238_b200 as wq
    info = wq.wq_plan_info(plan_h)
    n = info["n_dof"][0]
    R1 = wq.wq_export_rules(plan_h, 0, p)
    qlen = R1["qlen"].astype(np.int64)
    ilen = np.array([min(n - 1, i + p) - max(0, i - p) + 1 for i in range(n)], dtype=np.int64)
    S1, T1 = int((ilen * qlen).sum()), int(qlen.sum())
    R = info["nnz_local"] / int(ilen.sum())
    return ((4 * S1 + 6 * T1) if matrix == 1 else 2 * S1) * R


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
def run_ours(cfg, matrix, steps, warmup, rank, world, device, dist, want_e2e=True, sgq=False, dump=None):
    """Time `steps` whole-path steps on this rank's slab; returns per-rank timings (max over ranks
    where it matters)."""
    import torch
    import paper_1605_01238_b200 as wq

    torch.cuda.set_device(device)
    from paper_1605_01238_b200.dist import slab_cuts
    n_d = cfg.n_el + cfg.p
    cuts = slab_cuts(n_d, cfg.p, world)
    knots = cfg.knots()
    ctrl = cfg.ctrl()
    plan = wq.Plan(cfg.p, knots, ctrl=ctrl, slab=(cuts[rank], cuts[rank + 1]), need_mass=matrix == wq.WQ_MASS,
                   need_stiffness=matrix == wq.WQ_STIFFNESS, device=device)
    info = plan.info
    flops = alg_flops(plan.h, cfg.p, matrix)
    stream = torch.cuda.Stream(device)
    d_ctrl = torch.from_numpy(ctrl).to(device)
    rp, col, val = plan.alloc_csr()
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=device)
    # the exchange runs on the device with NCCL; gloo (CPU tests of the rank path) needs host tensors
    xdev = "cpu" if dist is not None and dist.get_backend() == "gloo" else device
    nnz_all = torch.zeros(world, dtype=torch.int64, device=xdev)
    my_nnz = torch.tensor([info["nnz_local"]], dtype=torch.int64, device=xdev)
    ev_a0 = torch.cuda.Event(enable_timing=True)
    ev_a1 = torch.cuda.Event(enable_timing=True)

    def step():
        with torch.cuda.stream(stream):
            wq.wq_build_rules(plan.h, stream)
            wq.wq_build_coef(plan.h, d_ctrl, stream=stream)
            if world > 1:  # the one exchange: all-gather of per-rank nnz -> row_ptr base
                dist.all_gather_into_tensor(nnz_all, my_nnz)
                base = int(nnz_all[:rank].sum().item()) if rank else 0
            else:
                base = 0
            wq.wq_pattern(plan.h, base, rp, None, stream)
            ev_a0.record(stream)
            if sgq:
                wq.wq_assemble_sgq(plan.h, matrix, d_ctrl, val, col, stream=stream)
            else:
                wq.wq_assemble(plan.h, matrix, val, col, stream)
            ev_a1.record(stream)

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
    if dump:  # rank's CSR block (tests of the multi-rank path)
        os.makedirs(dump, exist_ok=True)
        for nm, t in (("rp", rp), ("col", col), ("val", val)):
            np.save(os.path.join(dump, f"rank{rank}_{nm}.npy"), t.cpu().numpy())
    t_total = sum(t_steps)
    t_asm_mean = sum(t_asm) / len(t_asm)
    if world > 1:
        tt = torch.tensor([t_total, t_asm_mean], dtype=torch.float64, device=xdev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total, t_asm_mean = float(tt[0]), float(tt[1])
        dist.barrier()
    res = dict(nnz=info["nnz_total"], nnz_local=info["nnz_local"], rows_local=info["n_rows_local"], flops=flops,
               t_total=t_total, t_step=t_total / steps, t_asm=t_asm_mean, launches=launches // steps,
               clocks=clk.summary(), coef_points=info["coef_points"], n_dof=info["n_dof_total"],
               kernel=wq.KERNEL_NAMES[info["kernel"][matrix]] if not sgq else "sgq",
               uniform_rules=info["uniform_rules"], ncomp=6 if matrix == wq.WQ_STIFFNESS else 1)
    # end to end through the public host-buffer call (rank-local block)
    if want_e2e:
        n_rows, nnz_l = info["n_rows_local"], info["nnz_local"]
        del rp, col, val
        torch.cuda.empty_cache()
        hrp = torch.empty(n_rows + 1, dtype=torch.int64).pin_memory()
        hcol = torch.empty(nnz_l, dtype=torch.int32).pin_memory()
        hval = torch.empty(nnz_l, dtype=torch.float64).pin_memory()
        hctrl = torch.from_numpy(ctrl).pin_memory()
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
            tt = torch.tensor([te], dtype=torch.float64, device=xdev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        res["e2e"] = dict(t=te / e2e_steps, steps=e2e_steps, h2d=int(hctrl.numel() * 8),
                          d2h=int(nnz_l * 12 + (n_rows + 1) * 8))
    plan.close()
    return res


def roofline(res, hbm_peak, peak_src, sm_max_mhz):
    """Roofline of the dominant launch (wq_assemble): algorithmic bytes = 12 B/nnz written
    (the 8 B/row of row_ptr belong to wq_pattern's launch and are in the step line);
    the coefficient-field reads are reported beside it, not counted."""
    import paper_1605_01238_b200 as wq  # noqa: F401
    alg_bytes = 12 * res["nnz_local"]
    coef_bytes = 8 * res["ncomp"] * res["coef_points"]
    achieved = alg_bytes / res["t_asm"] / 1e9
    fp_peak = fp64_peak_tflops(sm_max_mhz or 1965.0)
    t_hbm, t_fp = alg_bytes / (hbm_peak * 1e9), res["flops"] / (fp_peak * 1e12)
    fp_ach = res["flops"] / res["t_asm"] / 1e12
    hbm_bound = t_hbm >= t_fp
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(res.get("traffic_key", ""))
    r = {"bound": "hbm" if hbm_bound else "alu",
         "achieved": achieved if hbm_bound else fp_ach,
         "peak": hbm_peak if hbm_bound else fp_peak,
         "unit": "GB/s" if hbm_bound else "TFLOP/s",
         "frac": achieved / hbm_peak if hbm_bound else fp_ach / fp_peak,
         "traffic": traffic,
         "peak_source": peak_src if hbm_bound else
         "148 SM x 64 DFMA/clk x 2 at max SM clock (guide unit counts; DMMA microbenchmark 37.1 TF)",
         "kernel": f"wq_assemble ({res['kernel']})", "kernel_ms": res["t_asm"] * 1e3,
         "kernel_share_of_step": res["t_asm"] / res["t_step"],
         "algorithmic_bytes_per_launch": alg_bytes, "algorithmic_bytes": "12 B/nnz (8 value + 4 column)",
         "coef_read_bytes_per_launch": coef_bytes,
         "hbm": {"achieved_gbs": achieved, "frac": achieved / hbm_peak},
         "fp64": {"algorithmic_flops_per_launch": res["flops"], "achieved_tflops": fp_ach, "peak_tflops": fp_peak,
                  "frac": fp_ach / fp_peak},
         "roofline_time_ms": max(t_hbm, t_fp) * 1e3, "frac_of_roofline": max(t_hbm, t_fp) / res["t_asm"],
         "step": {"bytes": 12 * res["nnz_local"] + 8 * (res["rows_local"] + 1) + coef_bytes,
                  "gbs": (12 * res["nnz_local"] + 8 * (res["rows_local"] + 1) + coef_bytes) / res["t_step"] / 1e9}}
    return r


def sweep_entry(cfg, matrix, rr, hbm_peak, label=None):
    roof = roofline(rr, hbm_peak, "", 1965.0)
    return {"config": label or cfg.name, "matrix": "mass" if matrix == 0 else "stiffness", "p": cfg.p,
            "n_el": cfg.n_el, "nnz": rr["nnz"], "value": rr["nnz"] / rr["t_step"],
            "ms_per_step": rr["t_step"] * 1e3, "asm_ms": rr["t_asm"] * 1e3, "kernel": rr["kernel"],
            "hbm_frac": roof["hbm"]["frac"], "fp64_frac": roof["fp64"]["frac"], "bound": roof["bound"],
            "frac_of_roofline": roof["frac_of_roofline"], "sm_mhz": rr["clocks"]["sm_mhz"]}


# ------------------------------------------------------------------- oracle
def run_oracle_sample(cfg, matrix, budget_s=20.0, seed=0):
    """Time the CPU oracle (as it stands) on a bounded, seeded uniform row sample of the workload."""
    from oracle import Oracle
    t0 = time.perf_counter()
    o = Oracle(cfg.p, cfg.knots(), cfg.ctrl())
    t_setup = time.perf_counter() - t0
    rng = np.random.default_rng(seed)
    n = cfg.n_el + cfg.p
    N = n ** cfg.d
    done_nnz, t_rows, nrows = 0, 0.0, 0
    batch = 8
    while t_rows < budget_s:
        rows = rng.integers(0, N, size=batch)
        t1 = time.perf_counter()
        ptr, *_ = o.rows(matrix, rows)
        dt = time.perf_counter() - t1
        t_rows += dt
        done_nnz += int(ptr[-1])
        nrows += rows.size
        if dt < 0.25 * budget_s / 4:
            batch *= 2
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return dict(value=done_nnz / t_rows, rows=nrows, nnz=done_nnz, t_rows=t_rows, t_setup=t_setup, cores=cores)


def oracle_one_core(cfg_name, p, matrix, budget_s):
    """The same oracle sample on one core (OMP_NUM_THREADS=1, a subprocess): the paper's
    single-core setting."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    code = (f"import sys,json; sys.path.insert(0,{ROOT!r}); import bench; from wqinputs import baseline_config; "
            f"print(json.dumps(bench.run_oracle_sample(baseline_config({cfg_name!r}, {p}), {matrix}, {budget_s})))")
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        return json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}


def config_of(name, p):
    if name == "C4":
        return baseline_config("C4", p)
    return baseline_config(name)


def workload_name(cfg, matrix):
    mat = "mass" if matrix == 0 else "stiffness"
    geo = "quarter annulus + 0.05 h noise" if cfg.geometry == "annulus" else "Greville grid + 0.1 h noise"
    return f"{cfg.name}: {cfg.d}D Poisson {mat}, p={cfg.p}, C^{cfg.p - 1}, {cfg.n_el}^{cfg.d} elements, {geo}"


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--p", type=int, default=4, help="C4 degree")
    ap.add_argument("--matrix", default="stiffness", choices=["stiffness", "mass"])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--oracle-seconds", type=float, default=20.0)
    ap.add_argument("--n-el", type=int, default=0, help="override the config's elements per direction (tests)")
    ap.add_argument("--dump-csr", default=None, help="directory: each rank saves its CSR block (tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = config_of(args.config, args.p)
    if args.n_el:
        cfg = Config(f"{cfg.name}e{args.n_el}", cfg.d, cfg.p, args.n_el, cfg.geometry, cfg.amp, cfg.matrices)
    matrix = 0 if args.matrix == "mass" else 1
    workload = workload_name(cfg, matrix)
    config = {"workload": workload, "nnz": cfg.exact_nnz(), "n_dof": cfg.n_dof,
              "matrix": args.matrix, "csr": "int64 row_ptr, int32 col, f64 val"}

    if args.impl == "reference":
        if rank != 0:
            return
        # each step: a bounded sample of the workload, sized so the whole run takes a few minutes
        per = max(2.0, min(args.oracle_seconds, 150.0 / (args.steps + args.warmup)))
        for _ in range(args.warmup):
            run_oracle_sample(cfg, matrix, per / 4, seed=99)
        nnz_done, t_done, rows_done, cores = 0, 0.0, 0, 1
        for k in range(args.steps):
            r = run_oracle_sample(cfg, matrix, per, seed=k)
            nnz_done += r["nnz"]
            t_done += r["t_rows"]
            rows_done += r["rows"]
            cores = r["cores"]
        value = nnz_done / t_done
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": cfg.exact_nnz() / value * 1e3,
                "ms_per_step_note": "extrapolated time of one full matrix (nnz_total / sampled nnz/s)",
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64 (long-double accumulation)", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": cores, "kind": "oracle",
                                 "cpu_model": cpu_model(),
                                 "sample": f"{args.steps} steps x {per:.1f} s of seeded uniformly random rows "
                                           f"({rows_done} rows, {nnz_done} nnz) of {workload}; oracle setup excluded"},
                "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import paper_1605_01238_b200 as wq
    dist = None
    device = local_rank % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(device)
        backend = os.environ.get("WQ_DIST_BACKEND", "nccl")  # gloo: CPU tests of the rank path
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)

    res = run_ours(cfg, matrix, args.steps, args.warmup, rank, world, device, dist, want_e2e=not args.no_e2e,
                   dump=args.dump_csr)
    res["traffic_key"] = cfg.name + ("" if matrix == 1 else "_mass")
    hbm_peak, peak_src, peaks_doc = peaks()
    nnz = res["nnz"]
    value = nnz * args.steps / res["t_total"]
    roof = roofline(res, hbm_peak, peak_src, res["clocks"]["sm_max_mhz"])
    config["parallelism"] = f"x{cfg.d}-slabs over {world} GPUs (rows independent, P:256-260)" if world > 1 else "1 GPU"
    config["l2"] = "256 MB buffer zeroed between timed steps (outside the timed interval); CSR output >> 126 MB L2"
    config["kernel"] = res["kernel"]
    config["uniform_rules"] = bool(res["uniform_rules"])
    line = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["t_total"] / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config, "roofline": roof, "gpu_launches": res["launches"], "clocks": res["clocks"]}
    if "e2e" in res:
        e = res["e2e"]
        line["e2e"] = {"value": nnz / e["t"], "unit": "nnz/s", "h2d_bytes_per_step": e["h2d"],
                       "d2h_bytes_per_step": e["d2h"], "steps": e["steps"],
                       "api": "wq_form_host (pinned host buffers, chunked D2H overlapped with assembly)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        r = run_oracle_sample(cfg, matrix, args.oracle_seconds)
        r1 = oracle_one_core(args.config, args.p, matrix, min(10.0, args.oracle_seconds))
        line["cpu_baseline"] = {"value": r["value"], "unit": "nnz/s", "cores": r["cores"], "kind": "oracle",
                                "cpu_model": cpu_model(),
                                "value_1core": r1.get("value"),
                                "sample": f"{r['rows']} seeded uniformly random rows ({r['nnz']} nnz) of the same "
                                          f"workload, {r['t_rows']:.1f} s on {r['cores']} threads (and "
                                          f"{r1.get('rows')} rows on 1 core); oracle setup {r['t_setup']:.1f} s excluded"}
    if not args.no_sweep and world == 1:
        sweep = []

        def add(c, mat, label=None, sgq=False, steps=3):
            try:
                rr = run_ours(c, mat, steps, 3, rank, world, device, dist, want_e2e=False, sgq=sgq)
                sweep.append(sweep_entry(c, mat, rr, hbm_peak, label))
            except Exception as ex:  # record, never hide
                sweep.append({"config": label or c.name, "matrix": "mass" if mat == 0 else "stiffness", "p": c.p,
                              "error": str(ex)[:200]})
            torch.cuda.empty_cache()
        for p in C4_DEGREES:
            add(baseline_config("C4", p), 1)
        add(baseline_config("C1"), 1)
        add(baseline_config("C1"), 0)
        # d = 2 at a size that fills the GPU (the sum-factorised d <= 2 kernel, WQ_KERNEL_SF2)
        for p in (2, 4, 6):
            c2d = Config(f"D2p{p}", 2, p, 1000, "grid", 0.1)
            add(c2d, 1, label=f"2D 1000^2 p={p} stiffness")
            add(c2d, 0, label=f"2D 1000^2 p={p} mass")
        add(baseline_config("C2"), 1)
        add(baseline_config("C2"), 0)
        add(baseline_config("C3"), 1)
        add(baseline_config("C5"), 1, steps=2)
        # the paper's timing shapes (Sect. 5.2, Fig. 2/3: 3D mass, 20^3 and 40^3 elements, p = 1..10)
        for ne in (20, 40):
            for p in range(1, 11):
                add(Config(f"M{ne}p{p}", 3, p, ne, "grid", 0.1, ("mass",)), 0, label=f"mass {ne}^3 p={p}")
        # WQ vs the standard element-loop Gauss quadrature (the paper's headline comparison)
        for p in (2, 3, 4):
            c = Config(f"M20p{p}", 3, p, 20, "grid", 0.1, ("mass",))
            add(c, 0, label=f"SGQ mass 20^3 p={p}", sgq=True)
            add(c, 1, label=f"SGQ stiffness 20^3 p={p}", sgq=True)
            add(c, 1, label=f"WQ stiffness 20^3 p={p}")
        line["sweep"] = sweep
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
