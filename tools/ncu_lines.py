"""Per-source-line executed-instruction shares of one kernel in an ncu report (needs -lineinfo and
--import-source on).  Usage: python tools/ncu_lines.py report.ncu-rep [launch_index] [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; cur = None; line = None
byline = collections.Counter(); byop = collections.Counter(); src = {}; stall = collections.Counter()
for r in rows:
    if len(r) == 2 and r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) < 6:
        continue
    if r[0]:
        line = (cur, int(r[0])); src[line] = r[1].strip()[:90]
    if r[2].startswith("0x"):
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        byline[line] += ie
        t = r[3].split(); op = t[1] if t[0].startswith("@") else t[0]
        byop[op.split(".")[0]] += ie
        try: stall[line] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError): pass
tot = sum(byop.values()) or 1
stot = sum(stall.values()) or 1
print("total", tot)
print([(k, round(v / tot * 100, 1)) for k, v in byop.most_common(20)])
for l, v in byline.most_common(top):
    print(f"{v/tot*100:5.1f}% inst {stall[l]/stot*100:5.1f}% stall  {l[0]}:{l[1]} | {src.get(l, '')}")
