"""Summarise an ncu report (read here): key raw metrics, the SASS opcode mix and the top stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "inst_executed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]
for r in rows[2:]:
    d = dict(zip(h, r))
    for k in keys:
        if k in d:
            print(f"{k:70s} {d[k]}")
    st = {k: d[k] for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    top = sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:8]
    for k, v in top:
        print(f"  stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {v}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
ix = hh.index("Instructions Executed")
cnt = collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ix:
        continue
    try:
        n = int(r[ix])
    except ValueError:
        continue
    toks = r[1].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    cnt[op.split(".")[0]] += n
    tot += n
print("total warp instructions", tot)
print(" ".join(f"{k}:{v * 100 / tot:.1f}%" for k, v in cnt.most_common(28)))
