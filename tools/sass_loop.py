"""Static SASS profile of a kernel's main loop (largest backward branch span): op counts per iteration.
Usage: python tools/sass_loop.py <lib.so> <mangled-name-substring>"""
import re, subprocess, sys
from collections import Counter
lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs if pat in f.split("\n")[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr_idx:
            span = i - addr_idx[tgt]
            if best is None or span > best[0]:
                best = (span, addr_idx[tgt], i)
span, lo, hi = best
ops = Counter()
for _, t in ins[lo:hi + 1]:
    tok = t.split()
    op = tok[1] if tok[0].startswith("@") else tok[0]
    ops[op.split(".")[0]] += 1
print(f"loop: {hi - lo + 1} instructions (static), {sum(ops.values())}")
fp = sum(ops[k] for k in ("FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL", "MUFU", "FMNMX"))
print("FP", fp, "| LDS", ops["LDS"], "| SHFL", ops["SHFL"], "| other", hi - lo + 1 - fp - ops["LDS"] - ops["SHFL"])
print(ops.most_common(25))
