#!/bin/bash
# 3D verification after a tile3d change (run under gpurun from the repo root): the 3D GPU
# tests (config-5 full-K ones last), bench lines of configs 4 / 4 P~1 / 5, the config-4
# launch lists and one ncu --set full capture of tile3d.
set -u
mkdir -p gpurun_out
timeout 500 python -m pytest tests -m gpu -x -q -k "3d or config4" --deselect tests/test_gpu_parity_fullk.py 2>&1 | tail -3 > gpurun_out/verify3d_tests.txt
B="timeout 300 python bench.py --no-cpu-baseline"
$B --config 4 --steps 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
$B --config 4 --precond 1 --omega 0.3 --steps 20 > gpurun_out/bench_c4_p1.json 2> /dev/null
$B --config 5 --steps 3 --warmup 3 --repeats 3 --e2e-steps 1 > gpurun_out/bench_c5.json 2> /dev/null
python tools/ab_variants.py --config 4 paper_2310_10430_b200/build/ab/lib_326d395.so - > gpurun_out/ab_revert.txt 2>&1
N="timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv"
$N --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 700 python -m pytest tests/test_gpu_parity_fullk.py -m gpu -x -q -k "config4 or config5" --durations=6 2>&1 | tail -12 >> gpurun_out/verify3d_tests.txt
for f in gpurun_out/bench_c4.json gpurun_out/bench_c4_p1.json gpurun_out/bench_c5.json; do echo "$f $(grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*' $f | tr '\n' ' ')"; done
cat gpurun_out/ab_revert.txt gpurun_out/verify3d_tests.txt
