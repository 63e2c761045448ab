"""Summarize an ncu report (debug helper): headline metrics, stall reasons, hot source lines."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
for k in ["gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum", "dram__bytes_read.sum",
          "dram__bytes_write.sum", "launch__registers_per_thread", "lts__t_bytes.sum"]:
    print(k, d.get(k))
ss = []
for k in h:
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            ss.append((float(d[k].replace(",", "")), k))
        except ValueError:
            pass
ss.sort(reverse=True)
print("stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={int(x)}" for x, k in ss[:10]))
mix = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(mix.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
by = collections.Counter()
reason = collections.defaultdict(collections.Counter)
stall_cols = [(i, k) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
src = {}
cur = None
fname = None
for r in rows[hi + 1:]:
    if len(r) < 5:
        continue
    if r[0] and not r[0].isdigit():
        continue
    if r[0]:
        cur = int(r[0])
        src[cur] = r[1]
    try:
        val = float(r[4] or 0)
    except ValueError:
        continue
    by[cur] += val
    for i, k in stall_cols:
        try:
            reason[cur][k] += float(r[i] or 0)
        except ValueError:
            pass
tot = sum(by.values())
for ln, val in by.most_common(ntop):
    top = reason[ln].most_common(3)
    print(f"{ln:4d} {val / tot * 100:5.1f}% {src.get(ln, '').strip()[:62]:62s} {[(k[6:], int(x)) for k, x in top]}")

# per-region totals: instructions executed and stall samples by source line ranges (argv[3:] as "name:lo-hi")
if len(sys.argv) > 3:
    ie_col = h.index("Instructions Executed")
    inst = collections.Counter()
    cur = None
    for r in rows[hi + 1:]:
        if len(r) < 5 or (r[0] and not r[0].isdigit()):
            continue
        if r[0]:
            cur = int(r[0])
        try:
            inst[cur] += float(r[ie_col] or 0)
        except ValueError:
            pass
    for spec in sys.argv[3:]:
        name, rng = spec.split(":")
        lo, hi_ = map(int, rng.split("-"))
        ii = sum(v for k, v in inst.items() if k and lo <= k <= hi_)
        ss_ = sum(v for k, v in by.items() if k and lo <= k <= hi_)
        print(f"region {name}: instr {ii:.3g}  stall-samples {ss_ / tot * 100:.1f}%")
