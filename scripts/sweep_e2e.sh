#!/bin/bash
# e2e (host-buffer) leg of the H33 bench for every variants/*/libradial_cuda.so
for d in variants/*/; do
  v=$(basename $d)
  RADIAL_CUDA_LIB=$PWD/$d/libradial_cuda.so timeout 300 python bench.py --steps 10 --warmup 3 --no-dense --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', round(d['value'],1), 'TF/s', round(d['ms_per_step'],2), 'ms', 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'])"
done
