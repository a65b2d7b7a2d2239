"""Per-source-line stall attribution from an ncu report (needs -lineinfo + --import-source)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No", "Kernel Name"):
        continue
    if len(r) > 8 and r[2] == "-":          # per-source-line aggregate row
        try:
            w = int(r[4]); ex = int(r[7])
        except ValueError:
            continue
        agg.append((w, ex, f"{cur}:{r[0]}", r[1].strip()[:90]))
tot = sum(a[0] for a in agg) or 1
for w, ex, loc, src in sorted(agg, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{w / tot * 100:5.1f}% {ex:>12d} {loc:22s} {src}")
