#!/bin/bash
# A/B of the tile3d work schedule (BIOT_T3_H: -1 = round robin of uncut tiles, else the
# list schedule with per-tile cost planes + h); the iterate hash must agree across rows.
set -u
mkdir -p gpurun_out
for cfg in "4 2" "4 1"; do
  set -- $cfg
  for h in -1 0.25 0.5 1.0; do
    echo -n "h=$h "; BIOT_T3_H=$h timeout 300 python tools/ab_variants.py --config $1 --precond $2 --steps 10 -
  done
done
for h in -1 0.5; do
  echo -n "h=$h "; BIOT_T3_H=$h timeout 600 python tools/ab_variants.py --config 5 --precond 2 --K 2 --steps 3 --repeats 3 -
done
