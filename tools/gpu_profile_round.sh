#!/bin/bash
# Round profile set (run under gpurun): bench lines, launch lists and one ncu --set full
# capture per dominant kernel; outputs in gpurun_out/ (copied to profiles/ afterwards).
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --precond 1 --omega 0.3 --steps 50 --no-cpu-baseline > gpurun_out/bench_c3_p1.json 2> gpurun_out/bench_c3_p1.err
timeout 600 python bench.py --method gs --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_gs.json 2> gpurun_out/bench_c3_gs.err
timeout 300 python bench.py --config 4 --steps 20 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config 4 --precond 1 --omega 0.3 --steps 20 --no-cpu-baseline > gpurun_out/bench_c4_p1.json 2> gpurun_out/bench_c4_p1.err
timeout 300 python bench.py --config 2 --steps 100 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config 1 --steps 100 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --method gmres --gmres-k 10 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_gmres.json 2> gpurun_out/bench_c3_gmres.err
timeout 1200 python bench.py --method gs_gmres --gmres-k 10 --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c3_gs_gmres.json 2> gpurun_out/bench_c3_gs_gmres.err
timeout 600 python bench.py --method cheb --cheb-m 2 --steps 20 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c3_cheb2.json 2> gpurun_out/bench_c3_cheb2.err
timeout 900 python bench.py --config 4 --method gmres --gmres-k 10 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c4_gmres.json 2> gpurun_out/bench_c4_gmres.err
timeout 600 python bench.py --workload trig > gpurun_out/bench_trig.json 2> gpurun_out/bench_trig.err
timeout 300 python bench.py --workload trig --precond 1 --omega 0.3 --steps 50 --no-cpu-baseline > gpurun_out/bench_trig_p1.json 2> gpurun_out/bench_trig_p1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_trig.csv python bench.py --workload trig --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_trig.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tile2d -s 3 -c 1 -o gpurun_out/r01_tile2d_trig python bench.py --workload trig --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_trig.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_c4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tile2d -s 3 -c 1 -o gpurun_out/r01_tile2d_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_c3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tile3d -s 3 -c 1 -o gpurun_out/r01_tile3d_c4 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full_c4.log 2>&1
for f in gpurun_out/bench_*.json; do echo $f; grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"kernel_ms": [0-9.]*' $f | tr '\n' ' '; echo; done
