mkdir -p gpurun_out
export BIOT_DEBUG=1
for d in 0 1 2; do BIOT_TILE_DRY=$d timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | grep -o '\[biot\].*\|"ms_per_step": [0-9.]*' ; done
timeout 600 ncu --set full --import-source on -k regex:tile3d -s 2 -c 1 -o gpurun_out/tile3d_c4 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
