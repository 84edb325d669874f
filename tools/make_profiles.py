"""Summarise gpurun_out/prof/* (tools/profile_round.sh) into profiles/rNN_*.txt
and profiles/traffic.json (read by bench.py for roofline.traffic).

    python tools/make_profiles.py r01
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(DST, exist_ok=True)


def launch_rows(path, metric):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, ii, mi, vi = hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
    out = defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) > vi:
            out[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
            names[r[ii]] = r[ki]
    return [(names[k], out[k]) for k in sorted(out, key=int)]


def summary(recs, metric="gpu__time_duration.sum"):
    tot, cnt = defaultdict(float), defaultdict(int)
    for name, m in recs:
        k = name.split("(")[0][:70]
        tot[k] += m.get(metric, 0.0)
        cnt[k] += 1
    T = sum(tot.values()) or 1.0
    lines = [f"total {T / 1e6:.3f} ms over {sum(cnt.values())} launches (ncu-serialised, cold cache)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
        lines.append(f"{v / 1e6:10.3f} ms {100 * v / T:6.2f}%  n={cnt[k]:6d}  avg={v / cnt[k] / 1e3:9.2f} us  {k}")
    return "\n".join(lines)


# 1. launch list
p = os.path.join(SRC, "launches_card.csv")
if os.path.exists(p):
    recs = launch_rows(p, "gpu__time_duration.sum")
    txt = ("# ncu launch list: tools/profile_steps.py (CARD K=100 k=3 r=7, agreement knob s=1e6, 32 new tokens incl. prefill (CUDA graphs reused from the warm-up request's serving session), then run_vanilla AR; model init and the warm-up request excluded via --profile-from-start off)\n"
           "# ncu --metrics gpu__time_duration.sum --clock-control none  (per-launch times are cold-cache and\n"
           "# serialised: compare SHARES of the step, not absolute times)\n" + summary(recs))
    open(os.path.join(DST, f"{tag}_launches_card.txt"), "w").write(txt + "\n")
    print(txt)

# 2. DRAM traffic per tc_gemm launch of one target verify forward
p = os.path.join(SRC, "traffic_t8.csv")
if os.path.exists(p):
    recs = [r for r in launch_rows(p, "") if "tc_gemm" in r[0]]
    per_fwd = 129   # 4 linears x 32 layers + lm_head
    last = recs[-per_fwd:]
    rd = sum(m["dram__bytes_read.sum"] for _, m in last)
    wr = sum(m["dram__bytes_write.sum"] for _, m in last)
    t = sum(m["gpu__time_duration.sum"] for _, m in last)
    unit_rd = "byte"
    # the 8B verify forward's algorithmic weight bytes (bf16), llama-3.1-8b
    H, F, V, L = 4096, 14336, 128256, 32
    alg = 2 * (L * (H * 6144 + 4096 * H + 2 * F * H + H * F) + V * H)
    info = {"source": f"profiles/{tag}_traffic_t8.txt (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                      f"{len(last)} tc_gemm launches of one llama-3.1-8b verify forward, M=8)",
            "bytes_per_launch": round((rd + wr) / len(last)),
            "algorithmic_bytes_per_launch": round(alg / len(last)),
            "ratio_traffic_over_algorithmic": round((rd + wr) / alg, 4)}
    json.dump(info, open(os.path.join(DST, "traffic.json"), "w"), indent=1)
    lines = [f"# {info['source']}",
             f"launches {len(last)}  dram read {rd / 1e9:.3f} GB  write {wr / 1e9:.4f} GB  "
             f"algorithmic (weights) {alg / 1e9:.3f} GB  traffic/algorithmic {info['ratio_traffic_over_algorithmic']}",
             f"ncu-serialised GEMM time {t / 1e6:.3f} ms -> {(rd + wr) / t:.0f} GB/s (cold, per-launch)"]
    open(os.path.join(DST, f"{tag}_traffic_t8.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

# 3. full captures: key metrics + SASS evidence
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Elapsed Cycles",
        "Registers Per Thread", "Grid Size", "Cluster Size", "Dynamic Shared Memory Per Block", "Achieved Occupancy",
        "L2 Hit Rate", "Max Active Clusters"]
for rep in ("gemm_gu_t8", "gemm_qkv_d116", "pfwd_d116", "attn_tc_d116", "lmhead_topk"):
    p = os.path.join(SRC, rep + ".ncu-rep")
    if not os.path.exists(p):
        continue
    det = subprocess.run(["ncu", "-i", p, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [f"# ncu --set full --clock-control none capture: {rep} (tools/profile_round.sh)"]
    if os.path.exists(os.path.join(SRC, rep + ".log")):
        lines.append("# " + open(os.path.join(SRC, rep + ".log")).read().strip().splitlines()[-1][:200])
    drows = list(csv.reader(det.splitlines()))
    dh = drows[0]
    si, ni, ui, vi = (dh.index(c) for c in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    for r in drows[1:]:
        if len(r) > vi and r[ni] in KEYS:
            lines.append(f"{r[si]} | {r[ni]} | {r[vi]} {r[ui]}")
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        d = dict(zip(rr[0], rr[2]))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_op_tcgen05_mma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_tc.sum", "gpu__time_duration.sum"):
            for kk in d:
                if kk.startswith(k):
                    lines.append(f"raw | {kk} | {d[kk]}")
                    break
    sass = subprocess.run(["ncu", "-i", p, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    mn = defaultdict(int)
    for r in csv.reader(sass.splitlines()):
        if len(r) > 1:
            op = r[1].strip().lstrip("@!P0123456789 ").split(" ")[0]
            for tag_ in ("UTCHMMA", "UTCQMMA", "UTCMMA", "UTMALDG", "UBLKCP", "LDTM", "UTMACCTL"):
                if op.startswith(tag_):
                    mn[op] += 1
    lines.append("SASS evidence (static instruction count in the captured kernel): " +
                 ", ".join(f"{k} x{v}" for k, v in sorted(mn.items())))
    open(os.path.join(DST, f"{tag}_{rep}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
