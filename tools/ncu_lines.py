"""Per-CUDA-source-line instruction count and stall samples from an ncu report (source page)."""
import csv, io, subprocess, sys
from collections import Counter, defaultdict
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn = None; line = None; src = {}
ins, stall, ops = Counter(), Counter(), defaultdict(Counter)
reason = defaultdict(Counter)
rcols = {}
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]; continue
    if r[0] == "Function Name" or r[0] == "Line No":
        if r[0] == "Line No":
            hdr = r
            rcols = {i: h[6:] for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h}
        continue
    if r[0]:
        line = (fn, int(r[0])); src[line] = r[1][:70]; continue
    if hdr is None or len(r) < 8 or not r[7].isdigit():
        continue
    toks = r[3].strip().split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    k = int(r[7]); s = int(r[4] or 0)
    ins[line] += k; stall[line] += s; ops[line][op.split(".")[0]] += k
    for i, nm in rcols.items():
        if i < len(r) and r[i].isdigit():
            reason[line][nm] += int(r[i])
tot = sum(ins.values()); tots = sum(stall.values()) or 1
print("total warp-instr", tot)
for key, v in sorted(ins.items(), key=lambda kv: -kv[1])[:n]:
    top = ", ".join(f"{o}:{c*100//v}" for o, c in ops[key].most_common(3))
    print(f"{key[0]}:{key[1]:<4d} {v/tot*100:5.1f}% st {stall[key]/tots*100:5.1f}%  {src.get(key,'')[:60]:60s} [{top}]")
for a in sys.argv:
    if a.startswith("--op="):
        want = a[5:]
        print(f"\ntop lines by {want} count:")
        for key, v in sorted(ops.items(), key=lambda kv: -kv[1][want])[:n]:
            if v[want]:
                print(f"{key[0]}:{key[1]:<4d} {v[want]/tot*100:5.2f}%  {src.get(key,'')[:80]}")
if "--stalls" in sys.argv:
    print("\ntop lines by stall samples (main reasons):")
    for key, v in sorted(stall.items(), key=lambda kv: -kv[1])[:n]:
        rs = ", ".join(f"{nm}:{c*100//max(v,1)}" for nm, c in reason[key].most_common(3))
        print(f"{key[0]}:{key[1]:<4d} st {v/tots*100:5.1f}%  {src.get(key,'')[:60]:60s} [{rs}]")
