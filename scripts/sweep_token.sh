#!/bin/bash
# token-exact vs block-layout forward for every variants/*/libradial_cuda.so
for d in variants/*/; do
  v=$(basename $d)
  echo "$v $(RADIAL_CUDA_LIB=$PWD/$d/libradial_cuda.so timeout 200 python scripts/token_mode_time.py 2>&1 | tail -1)"
done
