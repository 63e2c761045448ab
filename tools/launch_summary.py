"""Mean duration per kernel (name prefix) of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = OrderedDict()
for r in rows[h + 1:]:
    if len(r) > vi:
        agg.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")) / 1e3)
for k, v in agg.items():
    print(f"{k:70s} n={len(v):3d} mean={sum(v) / len(v):9.3f} ms")
