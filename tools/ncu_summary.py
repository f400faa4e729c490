"""Summarise an ncu report: per kernel time, DRAM, IPC, occupancy, top stalls, pipe use.
Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units = r[0], r[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "us": 1e3, "ns": 1, "ms": 1e6}
UNIT = {h[i]: units[i] for i in range(len(h))}
def g(d, k):
    try: return float(d.get(k, "nan").replace(",", "")) * SCALE.get(UNIT.get(k, ""), 1)
    except ValueError: return float("nan")
for row in r[2:]:
    d = {h[i]: row[i] for i in range(len(h))}
    print("==", d["Kernel Name"][:100], "grid", d.get("launch__grid_size"), "regs", d.get("launch__registers_per_thread"))
    t = g(d, "gpu__time_duration.sum")
    dr = g(d, "dram__bytes_read.sum") + g(d, "dram__bytes_write.sum")
    print(f"   time {t/1e3:.1f} us  dram {dr/1e6:.1f} MB ({dr/t:.0f} GB/s)  ipc {g(d,'sm__inst_executed.avg.per_cycle_active'):.2f}  "
          f"warps_active {g(d,'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%  inst {g(d,'smsp__inst_executed.sum')/1e6:.1f}M")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try: st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError: pass
    print("   stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8]))
    pipes = [(g(d, k), k.split("__")[1]) for k in d if k.startswith("sm__inst_executed_pipe_") and k.endswith("avg.pct_of_peak_sustained_active")]
    print("   pipes:", ", ".join(f"{n.replace('inst_executed_pipe_','').split('.')[0]} {v:.0f}%" for v, n in sorted(pipes, reverse=True)[:7]))
    print(f"   l1 hit {g(d,'l1tex__t_sector_hit_rate.pct'):.0f}%  l2 hit {g(d,'lts__t_sector_hit_rate.pct'):.0f}%  smem bank conflicts {g(d,'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum')/1e6:.1f}M  smem wavefronts {g(d,'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')/1e6:.1f}M")
