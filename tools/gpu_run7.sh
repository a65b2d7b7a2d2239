mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_invariants.py -k "tile3d" -x -q 2>&1 | tail -3
timeout 600 ncu --set full --import-source on -k regex:tile3d -s 2 -c 1 -o gpurun_out/tile3d_c4_v2 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_c4_v2.log 2>&1
tail -n 2 gpurun_out/ncu_c4_v2.log
