"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel
count, mean and total time and share of the captured launches."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
t = defaultdict(list)
for r in rows:
    t[r[4].split("(")[0]].append(float(r[14]) / 1e3)
tot = sum(sum(v) for v in t.values())
print(f"{'kernel':60s} {'n':>4s} {'mean us':>10s} {'total us':>11s} {'share':>6s}")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:60]:60s} {len(v):4d} {sum(v) / len(v):10.1f} {sum(v):11.1f} {sum(v) / tot * 100:5.1f}%")
