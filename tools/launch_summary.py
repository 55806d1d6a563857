"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: time share per kernel."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
agg = collections.OrderedDict()
for r in rows:
    name = r[4]
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"<.*", "<...>", short) if "bsfa" not in short else re.sub(r"\(.*", "", name)
    key = short[:90]
    ns = float(r[-1])
    n, t = agg.get(key, (0, 0.0))
    agg[key] = (n + 1, t + ns)
tot = sum(t for _, t in agg.values())
print(f"{'kernel':92s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'ms/launch':>10s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:92s} {n:8d} {t/1e6:10.3f} {100*t/tot:6.1f}% {t/n/1e6:10.4f}")
