"""Summarise an ncu source-page CSV: stall reasons per code region (by SASS index ranges)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
isrc = hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons}
tot = sum(int(r[iall] or 0) for r in data)


def region(lo, hi, name):
    agg = {h: 0 for h in reasons}
    s = 0
    for r in data[lo:hi]:
        s += int(r[iall] or 0)
        for h in reasons:
            agg[h] += int(r[idx[h]] or 0)
    top = sorted(agg.items(), key=lambda kv: -kv[1])[:6]
    print(f"{name:24s} {s:8d} ({100*s/tot:5.1f}%)  " + "  ".join(f"{k[6:]}={v}" for k, v in top if v))


# markers: find instruction indices by pattern
def find(pat, start=0):
    for i in range(start, len(data)):
        if pat in data[i][isrc]:
            return i
    return None


print("total samples", tot)
if len(sys.argv) > 2:
    cuts = [int(x) for x in sys.argv[2].split(",")]
    for a, b in zip(cuts, cuts[1:]):
        region(a, b, f"[{a},{b})")
