mkdir -p gpurun_out
export BIOT_DEBUG=1
BIOT_TILE_DRY=2 timeout 600 ncu --set full --import-source on -k regex:tile3d -s 2 -c 1 -o gpurun_out/tile3d_c4_int python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c4_int.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:tile3d -s 2 -c 1 -o gpurun_out/tile3d_c4_full python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c4_full.log 2>&1
tail -2 gpurun_out/ncu_c4_int.log gpurun_out/ncu_c4_full.log
