"""Per-element instruction budget of the INT8 step kernel from an ncu report (source page, SASS
with CUDA line attribution): executed thread-instructions per element computation, grouped by
what the source line does (SURVEY H1 / VERDICT r1 item 4c).

    python tools/ncu_budget.py REPORT.ncu-rep [elements_computed]

elements_computed defaults to the C2 launch (256³ elements × 1.3186 halo/z-chunk redundancy =
22.12 M).  Categories are assigned from the source text of the line, so they survive line shifts.
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter, OrderedDict

rep = sys.argv[1]
ELEMS = float(sys.argv[2]) if len(sys.argv) > 2 else 256 ** 3 * 1.3186
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout

CATS = OrderedDict([
    ("F2I + scale (Eq. 10-12: DMUL ū·R, F2I.S64)", [r"__double2ll_rz", r"__double2int_rz"]),
    ("G half: cG·u (DMUL)", [r"__dmul_rn\(cG"]),
    ("v + 2^56 offset (high word)", [r"AOFF >> 32", r"\+ \(uint32_t\)AOFF"]),
    ("byte packing (PRMT) into the A words", [r"__byte_perm"]),
    ("A operand to TMEM (tcgen05.st)", [r"tmem_st4", r"tmem_st8", r"tcgen05\.st"]),
    ("gather of u_e from shared planes", [r"ue\[j\] =", r"gather16", r"ue\[3 \* a", r"rb\[a\]"]),
    ("s_e = max|ū| (node maxima, 64-bit max)", [r"ullmax", r"max\(ab", r"ab = ", r"amax", r"fmax\(amax", r"qmax"]),
    ("degenerate / fast-path tests", [r"const bool deg", r"const bool vzero", r"const bool fast", r"__all_sync"]),
    ("reciprocal RN(1/s)", [r"1\.0 / s", r"__drcp_rn", r"__dmul_rn\(r, SCALE\)"]),
    ("MMA issue, commit, M-tile barrier", [r"mma_i8", r"mma_commit", r"bar\.sync", r"elect_one", r"smem_desc"]),
    ("MMA completion waits (mbarrier)", [r"mbar_wait", r"try_wait"]),
    ("accumulators from TMEM (tcgen05.ld)", [r"tmem_ld", r"tcgen05\.ld", r"tcgen05\.wait"]),
    ("exact two-limb recombination", [r"limb", r"p0 = ", r"mad\.wide", r"acc\)", r"I8_LIMB_MAGIC", r"add\.cc", r"p1 >> 16"]),
    ("RN(y) and the Eq. 9 scalar (DFMA, DMUL)", [r"__fma_rn\(dhi", r"__dmul_rn\(alpha", r"const double alpha"]),
    ("node sums: x-pairs (shuffle), y-pairs (smem)", [r"__shfl_up_sync", r"shfl", r"ysum", r"plo\[c\]", r"S\.ys\[",
                                                      r"Pb\[c\]", r"Pt\[c\]", r"fbot\[c\]", r"ftop\[c\]", r"ys_ready"]),
    ("post-phase: face sums, T + B, update, store", [r"tfv", r"ucv", r"face\[", r"__fma_rn\(wn", r"un = ", r"dst\[c\]",
                                                    r"\(DAMP \? p\.un : p\.uo\)", r"p\.src_dof", r"2\.0, uc", r"dm >> c",
                                                    r"uc = ", r"p\.uo\[3 \* un_id", r"__dadd_rn\(T\[c\]", r"T\[c\] = ftop",
                                                    r"p\.rec_node", r"p\.fout"]),
    ("plane / operand prefetch and park (global loads, smem stores)", [r"__ldg", r"load_in", r"pfv", r"S\.up\[",
                                                                     r"nmax", r"upv_n", r"wn_n", r"mfar", r"S\.mid",
                                                                     r"cp_async", r"P\.up\[", r"P\.mid", r"mid_next",
                                                                     r"abs_bits", r"mx = b > mx", r"upv\[", r"p\.uo\[3 \* nd"]),
])


import os
_PTX = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2404_13683_b200", "csrc", "ptx.cuh")
_ptx_fn = {}
try:   # ptx.cuh lines -> the helper they belong to (asm text has no keywords)
    cur_fn = ""
    for i, ln in enumerate(open(_PTX), start=1):
        m = re.search(r"__forceinline__ \S+ (\w+)\(", ln)
        if m:
            cur_fn = m.group(1)
        _ptx_fn[i] = cur_fn
except OSError:
    pass
_PTX_CAT = [("mbar_wait", "MMA completion waits (mbarrier)"), ("tmem_st", "A operand to TMEM (tcgen05.st)"),
            ("tmem_ld", "accumulators from TMEM (tcgen05.ld)"), ("mma", "MMA issue, commit, M-tile barrier"),
            ("tc_fence", "MMA issue, commit, M-tile barrier"), ("fence", "MMA issue, commit, M-tile barrier"),
            ("elect", "MMA issue, commit, M-tile barrier")]


def cat_of(text, key=None):
    if key and key[0] == "ptx.cuh":
        f = _ptx_fn.get(key[1], "")
        for k, name in _PTX_CAT:
            if f.startswith(k):
                return name
    for name, pats in CATS.items():
        for pt in pats:
            if re.search(pt, text):
                return name
    return "loop control, indexing, role selection (other)"


fn = None
line_src = {}
counts = Counter()
cur = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        if r[0] == "Line No":
            hdr = r
        continue
    if r[0]:
        cur = (fn, int(r[0]))
        line_src[cur] = r[1]
        continue
    if hdr is None or len(r) < 8 or not r[7].isdigit():
        continue
    counts[cur] += int(r[7])

by = Counter()
for key, n in counts.items():
    by[cat_of(line_src.get(key, ""), key)] += n
tot = sum(by.values())
# the source page's per-instruction counts overcount the launch's smsp__inst_executed.sum (they
# include predicated-off issue of divergent paths); scale the categories to the launch total
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
try:
    launch_tot = float(rr[2][rr[0].index("smsp__inst_executed.sum")].replace(",", ""))
except (ValueError, IndexError):
    launch_tot = tot
scale = launch_tot / tot
by = Counter({k: v * scale for k, v in by.items()})
tot = launch_tot
print(f"warp-instructions (smsp__inst_executed.sum): {tot:.4g}  ->  thread-instructions per element computation: "
      f"{32 * tot / ELEMS:.0f}")
print(f"{'category':66s} {'/elem':>7s} {'share':>6s}")
for name, n in by.most_common():
    print(f"{name:66s} {32 * n / ELEMS:7.0f} {100 * n / tot:5.1f}%")
# the largest lines left in "other" (transparency for the catch-all category)
oth = sorted(((n, k) for k, n in counts.items()
              if cat_of(line_src.get(k, ""), k) == "loop control, indexing, role selection (other)"), reverse=True)[:12]
print("\nlargest 'other' lines (thread-instructions per element):")
for n, k in oth:
    print(f"  {k[0]}:{k[1]:<5d} {32 * n * scale / ELEMS:6.0f}  {line_src.get(k, '')[:70]}")
