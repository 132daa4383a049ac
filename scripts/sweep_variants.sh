#!/bin/bash
# Runs the H33 bench (no dense/e2e/cpu legs) for every variants/*/libradial_cuda.so; extra
# arguments go to bench.py (e.g. --bwd).
for d in variants/*/; do
  v=$(basename $d)
  RADIAL_CUDA_LIB=$PWD/$d/libradial_cuda.so timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
b=d.get('backward') or {}
print('$v', round(d['value'],1), 'TF/s', round(d['ms_per_step'],2), 'ms', 'bwd', round(b.get('ms_per_step',0),2), 'ms', d['clocks'])"
done
