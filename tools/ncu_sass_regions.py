"""Warp-stall samples of an ncu report (--set full, source counters) by SASS region.

Prints, for the first kernel matching --kernel, the samples and executed instructions between
consecutive barrier / EXIT instructions (BAR.SYNC stalls are charged to the instruction after the
barrier, so each region's first instruction carries the wait at the barrier that opens it), the
opcode mix and the top stalled instructions.  Usage:
  python tools/ncu_sass_regions.py report.ncu-rep [--kernel substring] [--top N]
"""
import argparse
import csv
import io
import subprocess
from collections import Counter

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--kernel", default="")
ap.add_argument("--top", type=int, default=12)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
secs, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "ins": []}
        secs.append(cur)
    elif r and r[0] == "Address":
        hdr = r
    elif cur is not None and len(r) > 5:
        cur["ins"].append(r)
sec = next(s for s in secs if a.kernel in s["name"])
si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ins = sec["ins"]
tot = sum(int(r[si]) for r in ins)
print(sec["name"][:120])
print(f"samples {tot}, SASS instructions {len(ins)}")
cuts = [i for i, r in enumerate(ins) if "BAR.SYNC" in r[1] or "EXIT" in r[1]] + [len(ins) - 1]
prev = 0
for c in cuts:
    seg = ins[prev:c + 2]
    sm = sum(int(r[si]) for r in seg)
    if sm:
        print(f"  [{prev:5d},{c + 2:5d}) samples {sm:8d} ({100 * sm / tot:5.1f} %)  first: {seg[0][1].strip()[:48]}")
    prev = c + 2
ops = Counter()
for r in ins:
    t = r[1].strip().split()
    ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += int(r[si])
print("  opcodes:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(10)))
for i in sorted(range(len(ins)), key=lambda j: -int(ins[j][si]))[:a.top]:
    print(f"  {i:5d} {ins[i][1].strip()[:60]:60s} {int(ins[i][si]):8d} ({100 * int(ins[i][si]) / tot:4.1f} %)"
          f" exec {ins[i][ie]}")
