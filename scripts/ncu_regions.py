"""Per-region totals of an ncu source page (`ncu -i rep --page source --csv --print-source
cuda,sass > page.csv`): warp-stall samples, warp instructions and active threads per device
function of orca_kernels.cuh, with k_step split at its `// ---- N.` phase markers.

  python scripts/ncu_regions.py page.csv [paper_1908_10107_b200/csrc/orca_kernels.cuh]
"""
import csv
import re
import sys

page = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "paper_1908_10107_b200/csrc/orca_kernels.cuh"
lines = open(src).read().split("\n")
starts = []
for n, l in enumerate(lines, 1):
    m = re.match(r"(?:template <[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", l)
    if m:
        starts.append((n, m.group(1)))
    m = re.match(r"\s*// ---- (\d[^ ]*)", l)
    if m:
        starts.append((n, f"k_step.{m.group(1)}"))
    if "if (blockQ) {" in l and "LP3 of the block" in (lines[n] if n < len(lines) else ""):
        starts.append((n, "k_step.blockQ"))
starts.sort()


def region(ln):
    r = "?"
    for n, name in starts:
        if n <= ln:
            r = name
        else:
            break
    return r


rows = list(csv.reader(open(page)))
hdr, fname = None, ""
agg = {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        ie = int(d["Instructions Executed"] or 0)
        te = int(d["Thread Instructions Executed"] or 0)
    except ValueError:
        continue
    key = region(int(r[0])) if fname == src.split("/")[-1] else fname
    a = agg.setdefault(key, [0, 0, 0])
    a[0] += s
    a[1] += ie
    a[2] += te
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"samples {ts}  warp-instructions {ti}")
for k, (s, ie, te) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if s == 0 and ie == 0:
        continue
    print(f"{k:28s} samples {100*s/ts:5.1f}%  inst {100*ie/ti:5.1f}%  ({ie:>11d})  threads/inst {te/max(ie,1):5.1f}")
