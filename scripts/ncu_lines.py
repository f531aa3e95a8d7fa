"""Per-source-line hotspots from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
fname = ""
out = []
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
    out.append((fname, int(r[0]), r[1], s, ie, te))
tot = sum(o[3] for o in out) or 1
toti = sum(o[4] for o in out) or 1
print(f"samples {tot} warp-inst {toti}")
for f, ln, src, s, ie, te in sorted(out, key=lambda o: -o[3])[:top]:
    print(f"{f[:14]:14s}{ln:5d} samp {100*s/tot:5.1f}% inst {100*ie/toti:5.1f}% thr {te/max(ie,1):5.1f} | {src.strip()[:80]}")
