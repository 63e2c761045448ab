"""Per-kernel headline metrics of an ncu report as JSON (profiles/ summaries)."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else ""
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(keys)], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
ks = []
for r in rows[2:]:
    d = {"kernel": r[h.index("Kernel Name")]}
    for k in keys:
        if k in h:
            d[k] = r[h.index(k)] + (" " + units[h.index(k)] if units[h.index(k)] else "")
    ks.append(d)
json.dump({"workload": workload, "report": rep, "kernels": ks}, open(out, "w"), indent=1)
print(json.dumps(ks, indent=1)[:3000])
