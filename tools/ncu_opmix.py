"""Instruction mix (by SASS opcode) and stall share from an ncu report's source page."""
import csv, io, subprocess, sys
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Source"); iE = hdr.index("Instructions Executed"); iW = hdr.index("Warp Stall Sampling (All Samples)")
c, w = Counter(), Counter()
for r in data:
    if len(r) <= iE or not r[iE].isdigit():
        continue
    toks = r[iS].strip().split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = ".".join(op.split(".")[:2]) if op.startswith(("F2I", "I2F", "LDS", "STS", "LDG", "STG", "IMAD")) else op.split(".")[0]
    c[op] += int(r[iE]); w[op] += int(r[iW] or 0)
tot = sum(c.values()); totw = sum(w.values()) or 1
print("total warp-instructions", tot)
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:16s} {n/tot*100:5.1f}%  {n:>12d}  stall {w[op]/totw*100:5.1f}%")
