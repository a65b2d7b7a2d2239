set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_invariants.py -k "tile3d" -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py -k "3d or ragged or config4" -x -q 2>&1 | tail -15
timeout 300 python bench.py --config 4 --steps 20 --no-cpu-baseline 2>&1 | tail -2
timeout 300 python bench.py --steps 30 --no-cpu-baseline 2>&1 | tail -1
