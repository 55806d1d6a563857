"""Per-CUDA-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
out = {}
cur_file = None
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    key = (cur_file, int(r[0]))
    s = int(float(r[4] or 0))
    a, src, n = out.get(key, (0, r[1], 0))
    out[key] = (a + s, src, n + int(float(r[7] or 0)))
tot = sum(v[0] for v in out.values())
print(f"total samples {tot}")
for (f, ln), (s, src, n) in sorted(out.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/tot:5.2f}% {f}:{ln:<4d} ex={n:>10d}  {src.strip()[:100]}")
