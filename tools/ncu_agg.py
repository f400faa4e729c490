"""Aggregate an ncu --csv launch list (per-kernel mean time, DRAM bytes, GB/s, grid, registers,
achieved occupancy).  Usage: python tools/ncu_agg.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    if len(r) < len(h):
        continue
    d.setdefault((r[ii], r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.OrderedDict()
for (i, k), m in d.items():
    agg.setdefault(k[:80], []).append(m)


def mean(ms, key):
    v = [m[key] for m in ms if key in m]
    return sum(v) / len(v) if v else float("nan")


for k, ms in agg.items():
    t = mean(ms, "gpu__time_duration.sum")
    b = mean(ms, "dram__bytes_read.sum") + mean(ms, "dram__bytes_write.sum")
    print(f"{len(ms):3d} {t / 1e3:8.1f} us {b / 1e6:8.1f} MB {b / t:6.0f} GB/s grid {mean(ms, 'launch__grid_size'):7.0f} "
          f"regs {mean(ms, 'launch__registers_per_thread'):4.0f} occ {mean(ms, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%  {k}")
