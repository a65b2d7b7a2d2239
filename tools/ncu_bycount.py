"""Group executed SASS instructions of an ncu report by their execution count (each code
region of a kernel runs a characteristic number of times) and show the opcode mix of
the largest groups."""
import csv, re, subprocess, sys
from collections import Counter, defaultdict
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ei = h.index("Source"), h.index("Instructions Executed")
wi = h.index("Warp Stall Sampling (All Samples)")
groups = defaultdict(Counter)
samples = Counter()
for r in rows[2:]:
    c = int(r[ei] or 0)
    if c == 0:
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip()).split(" ")[0]
    groups[c][op] += 1
    samples[c] += int(r[wi] or 0)
tot_s = sum(samples.values())
for c, cnt in sorted(groups.items(), key=lambda kv: -kv[0] * sum(kv[1].values()))[:int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    n = sum(cnt.values())
    print(f"exec count {c}: {n} instructions/visit, {c * n / 1e6:.1f}M executed, {samples[c] / tot_s * 100:.1f}% of stall samples")
    print("   ", ", ".join(f"{op} {k}" for op, k in cnt.most_common(14)))
