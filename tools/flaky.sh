#!/bin/bash
# repeat the GPU test subset to expose intermittent failures
for i in $(seq 1 ${1:-5}); do
  timeout 300 python -m pytest tests -m gpu -q -k "variants_bitwise or config1 or config2 or ragged or slabs" 2>&1 | tail -1
done
