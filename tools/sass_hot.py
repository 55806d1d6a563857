"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
top = sorted(data, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
print(f"total samples {tot}")
for r in top:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    reasons = sorted(((int(r[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    rs = " ".join(f"{n}:{c}" for c, n in [(c, n) for n, c in reasons if n])
    print(f"{100*s/tot:5.2f}% {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} ex={r[idx['Instructions Executed']]:>9s} {rs}")
