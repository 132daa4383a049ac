# token-exact over paired lists + early S (variant) vs current; dK/dV per-lane release under
# racecheck; backward tests
tag=r02j
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_new.txt 2>&1
  RADIAL_CUDA_LIB=variants/tok_paired/libradial_cuda.so timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_paired.txt 2>&1
done
RADIAL_CUDA_LIB=variants/tok_paired/libradial_cuda.so timeout 900 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider -k "token or pattern or power" > gpurun_out/${tag}_pytest_paired.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_paired.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/${tag}_san_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_san_racecheck.log
timeout 900 python -m pytest tests/test_gpu_backward.py -q -p no:cacheprovider > gpurun_out/${tag}_pytest_bwd.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_bwd.log
