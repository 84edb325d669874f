"""Summarise an ncu --csv launch list: time per kernel name (share of total)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T/1e6:.3f} ms over {sum(cnt.values())} launches")
for name, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{v/1e6:10.3f} ms {100*v/T:6.2f}% n={cnt[name]:6d} avg={v/cnt[name]/1e3:9.2f} us  {name}")
