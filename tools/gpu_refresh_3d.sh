#!/bin/bash
# Refresh of the 3D evidence after the tile3d list schedule (run under gpurun from the repo
# root): the schedule the setup picks (BIOT_DEBUG), a planes-per-tile sweep under the list
# schedule, launch lists and one ncu --set full capture of tile3d on config 4.
set -u
mkdir -p gpurun_out
B="timeout 300 python bench.py --config 4 --steps 20 --no-cpu-baseline --e2e-steps 2"
BIOT_DEBUG=1 $B > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
grep "\[biot\]" gpurun_out/bench_c4.err | sort | uniq -c | head -8 > gpurun_out/t3_debug.txt
for zr in 11 13 17 22; do
  for h in 0.25 1.0; do
    BIOT_DEBUG=1 BIOT_ZROWS=$zr BIOT_T3_H=$h $B --repeats 3 > gpurun_out/zr_${zr}_$h.json 2> gpurun_out/zr_${zr}_$h.err
    echo "zrows=$zr h=$h $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/zr_${zr}_$h.json) $(grep -o 'schedule: [0-9]* tiles[^)]*)' gpurun_out/zr_${zr}_$h.err | head -1)"
  done
done > gpurun_out/t3_zrows_sweep.txt
N="timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv"
$N --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$N --log-file gpurun_out/launches_c4_p1.csv python bench.py --config 4 --precond 1 --omega 0.3 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
F="timeout 900 ncu --set full --import-source on --clock-control none -s 3 -c 1"
$F -k regex:tile3d_kernel -o gpurun_out/r02_tile3d_c4 python bench.py --config 4 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
cat gpurun_out/t3_debug.txt gpurun_out/t3_zrows_sweep.txt
