"""Summarise the last N launches of an ncu --csv launch list by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2])
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
recs = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
recs = recs[-n:]
tot = defaultdict(float)
cnt = defaultdict(int)
for name, v in recs:
    k = name.split("(")[0][:60]
    tot[k] += v
    cnt[k] += 1
T = sum(tot.values())
print(f"last {len(recs)} launches: {T/1e3:.1f} us (serialised, cold-ish)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v/1e3:9.1f} us {100*v/T:5.1f}% n={cnt[k]:4d} avg={v/cnt[k]/1e3:7.2f} us  {k}")
