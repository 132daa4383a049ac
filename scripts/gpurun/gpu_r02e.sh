# Round-2 verification: GPU tests (incl. native CLI), bench line, the four compute-sanitizer
# tools over every kernel family (+ the opt-in pair forward under racecheck / memcheck)
tag=r02e
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py \
    > gpurun_out/${tag}_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_san_${tool}.log
done
for tool in memcheck racecheck; do
  RADIAL_FWD_PAIR=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py \
    > gpurun_out/${tag}_san_pair_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_san_pair_${tool}.log
done
