"""Hot SASS instructions with their source lines and stall reasons.

    ncu -i R --page source --csv --print-source sass       > sass.csv
    ncu -i R --page source --csv --print-source cuda,sass  > mixed.csv
    python tools/sass_lines.py sass.csv mixed.csv [top]

Inlined helpers (mbarrier waits) map to ptx.cuh; the nearest preceding
instruction that maps to a kernel file names the call site.
"""
import csv
import sys

sass = list(csv.reader(open(sys.argv[1])))
hdr = sass[1]
rows = sass[2:]
ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ridx = {h: hdr.index(h) for h in reasons}

# second pass: map address -> (file, line) using the order of the mixed listing
loc = {}
cur_file, cur_line = None, None
for r in csv.reader(open(sys.argv[2])):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
    elif r[0].isdigit():
        cur_line = int(r[0])
    elif len(r) > 2 and r[2].startswith("0x"):
        loc[r[2]] = f"{cur_file}:{cur_line}"
tot = sum(int(r[iall] or 0) for r in rows)
site = None
out = []
for k, r in enumerate(rows):
    l = loc.get(r[ia], "?")
    if not l.startswith("ptx.cuh") and not l.startswith("cuda_") and not l.startswith("sm_"):
        site = l
    s = int(r[iall] or 0)
    top = sorted(((int(r[ridx[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
    out.append((s, k, l, site, r[isrc].strip(), int(r[iex] or 0), top))
print("total samples", tot)
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
for s, k, l, site, src, ex, top in sorted(out, reverse=True)[:n]:
    print(f"{100*s/tot:5.2f}% #{k:<5d} {l:22s} site={site:20s} ex={ex:>9d} {src[:60]:60s} " +
          " ".join(f"{n}={v}" for v, n in top if v))
