mkdir -p gpurun_out
export BIOT_DEBUG=1
timeout 600 python -m pytest tests/test_gpu_invariants.py -k "tile3d" -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -k "3d or config4" -x -q 2>&1 | tail -2
for d in 0 2 1; do BIOT_TILE_DRY=$d timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '\[biot\].*\|"ms_per_step": [0-9.]*' ; done
for z in 22 16; do BIOT_ZROWS=$z timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '\[biot\].*\|"ms_per_step": [0-9.]*' ; done
timeout 300 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '\[biot\].*\|"ms_per_step": [0-9.]*'
