"""Top SASS lines of an ncu report by warp-stall samples (first kernel).
usage: python tools/ncu_hot.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
body = []
for r in rows[1:]:
    if len(r) <= iss or r[0] == "Address":
        break
    try:
        body.append((int(r[iss]), r[ia], r[isrc]))
    except ValueError:
        break
tot = sum(b[0] for b in body)
print(f"total samples {tot}, {len(body)} instructions")
for s, a, src in sorted(body, reverse=True)[:n]:
    print(f"{s:7d} {100.0 * s / tot:5.1f}%  {a[-5:]}  {src.strip()[:90]}")
