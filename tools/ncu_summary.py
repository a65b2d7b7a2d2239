"""Summarise an ncu report: key throughput metrics, stall reasons, top SASS lines."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u = r[0], r[1]
rows = r[2:]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__t_bytes.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
for row in rows:
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"{k:65s} {row[i]:>22s} {u[i]}")
    st = [(h[i], row[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_")
          and not h[i].endswith("not_issued")]
    tot = sum(float(v) for _, v in st if v)
    print("stall samples:", tot)
    for k, v in sorted(st, key=lambda x: -float(x[1] or 0))[:8]:
        print(f"   {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {float(v) / tot * 100:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
s = list(csv.reader(io.StringIO(src)))
hh = s[1]
si, wi, ei = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
body = s[2:]
tot = sum(int(x[wi]) for x in body)
print("top stalled SASS:")
for x in sorted(body, key=lambda x: -int(x[wi]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {int(x[wi]) / tot * 100:5.1f}%  {x[ei]:>10s}  {x[si].strip()[:80]}")
