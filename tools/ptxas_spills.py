"""Per-kernel registers and spills from paper_2310_10430_b200/build/ptxas.txt."""
import re
import sys

txt = open(sys.argv[1] if len(sys.argv) > 1 else "paper_2310_10430_b200/build/ptxas.txt").read()
pat = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur and pat in cur:
        st, ld = m.groups()
        name = re.sub(r"_ZN4biot\w*?_GLOBAL__N__\w+?_\d+(\w+?)EEv.*", r"\1", cur)
        print(f"{st:>5} {ld:>5}  {name[-60:]}")
        cur = None
