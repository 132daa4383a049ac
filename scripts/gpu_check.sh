#!/bin/bash
# One gpurun call: GPU test suite, bench line, compute-sanitizer on the small cases.
#   bash scripts/gpu_check.sh <tag> [pytest args...]
tag=${1:-check}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider "$@" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py \
    > gpurun_out/${tag}_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_san_${tool}.log
done
