"""SASS opcode mix (executed warp instructions) of the profiled kernel."""
import csv
import re
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ei = h.index("Source"), h.index("Instructions Executed")
cnt = Counter()
for r in rows[2:]:
    src = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip())
    op = src.split(" ")[0]
    cnt[op] += int(r[ei] or 0)
tot = sum(cnt.values())
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
for op, c in cnt.most_common(30):
    print(f"{op:28s} {c / tot * 100:5.1f}%  {c / norm:10.1f}")
print("total", tot, tot / norm)
