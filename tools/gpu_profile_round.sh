#!/bin/bash
# Round-2 profile set (run under gpurun from the repo root): bench lines, launch lists,
# one ncu --set full capture per dominant kernel, the multi-GPU projection; outputs in
# gpurun_out/ (copied to profiles/ as r02_* afterwards).
set -u
mkdir -p gpurun_out
B="timeout 600 python bench.py"
$B > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
$B --precond 1 --omega 0.3 --steps 50 --no-cpu-baseline > gpurun_out/bench_c3_p1.json 2> /dev/null
for c in 1 2; do
  $B --config $c --no-cpu-baseline > gpurun_out/bench_c$c.json 2> /dev/null
  $B --config $c --no-cpu-baseline --no-graph > gpurun_out/bench_c${c}_nograph.json 2> /dev/null
done
$B --config 4 --steps 20 --no-cpu-baseline > gpurun_out/bench_c4.json 2> /dev/null
$B --config 4 --precond 1 --omega 0.3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c4_p1.json 2> /dev/null
$B --config 5 --steps 3 --warmup 3 --repeats 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c5.json 2> /dev/null
$B --workload trig > gpurun_out/bench_trig.json 2> /dev/null
$B --workload trig --precond 1 --omega 0.3 --steps 50 --no-cpu-baseline > gpurun_out/bench_trig_p1.json 2> /dev/null
$B --method gs --steps 100 --warmup 3 --repeats 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_gs.json 2> /dev/null
$B --method gmres --gmres-k 10 --steps 3 --warmup 3 --repeats 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_gmres.json 2> /dev/null
$B --method gmres --gmres-k 10 --precond 1 --omega 0.3 --steps 3 --warmup 3 --repeats 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_gmres_p1.json 2> /dev/null
$B --method gs_gmres --gmres-k 10 --steps 16 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_gs_gmres16.json 2> /dev/null
$B --method cheb --cheb-m 2 --steps 20 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c3_cheb2.json 2> /dev/null
$B --config 4 --method gmres --gmres-k 10 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_gmres.json 2> /dev/null
N="timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv"
$N --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$N --log-file gpurun_out/launches_c3_p1.csv python bench.py --precond 1 --omega 0.3 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$N --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$N --log-file gpurun_out/launches_c4_p1.csv python bench.py --config 4 --precond 1 --omega 0.3 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$N --log-file gpurun_out/launches_trig.csv python bench.py --workload trig --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
F="timeout 900 ncu --set full --import-source on --clock-control none -s 3 -c 1"
$F -k regex:tile2d_kernel -o gpurun_out/r02_tile2d_c3 python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$F -k regex:tile2d_p1 -o gpurun_out/r02_tile2d_p1_c3 python bench.py --precond 1 --omega 0.3 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$F -k regex:tile3d_kernel -o gpurun_out/r02_tile3d_c4 python bench.py --config 4 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
$F -k regex:tile2d_kernel -o gpurun_out/r02_tile2d_trig python bench.py --workload trig --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 900 python tools/project_scaling.py --configs 3 4 > gpurun_out/proj.json 2> /dev/null
timeout 900 python tools/project_scaling.py --configs 3 4 --precond 1 > gpurun_out/proj_p1.json 2> /dev/null
for f in gpurun_out/bench_*.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*' $f | tr '\n' ' ')"; done > gpurun_out/summary.txt
