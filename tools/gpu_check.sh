# Standard GPU session (run under gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [tests|bench|all]'
# Writes logs under gpurun_out/.
set -u
mkdir -p gpurun_out
what=${1:-all}
if [ "$what" = tests ] || [ "$what" = all ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
fi
if [ "$what" = bench ] || [ "$what" = all ]; then
  timeout 300 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 2000 gpurun_out/bench_c3.json
  for c in 2 4; do
    timeout 300 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
    grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*' gpurun_out/bench_c$c.json | tr '\n' ' '; echo " config $c"
  done
fi
