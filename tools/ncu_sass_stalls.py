"""Top SASS instructions by a given stall reason (e.g. stall_long_sb) from an ncu report."""
import csv
import subprocess
import sys

rep, reason = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ri, ai = h.index("Source"), h.index(reason), h.index("Address")
body = rows[2:]
tot = sum(int(r[ri] or 0) for r in body) or 1
idx = {r[ai]: k for k, r in enumerate(body)}
for r in sorted(body, key=lambda r: -int(r[ri] or 0))[:n]:
    k = idx[r[ai]]
    prev = " | ".join(x[si].strip()[:38] for x in body[max(0, k - 2):k])
    print(f"{int(r[ri]) / tot * 100:5.1f}%  {r[si].strip()[:50]:50s}  <- {prev}")
