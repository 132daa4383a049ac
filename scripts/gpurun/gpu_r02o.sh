# token-exact: reciprocal key-frame division (any list order); ascending (product) vs paired
# lists + early S (variant) vs previous commit; token parity with both
tag=r02o
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_new.txt 2>&1
  RADIAL_CUDA_LIB=variants/tok_paired/libradial_cuda.so timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_paired.txt 2>&1
  RADIAL_CUDA_LIB=variants/head/libradial_cuda.so timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_head.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider -k "token or pattern or power" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
RADIAL_CUDA_LIB=variants/tok_paired/libradial_cuda.so timeout 900 python -m pytest tests/test_gpu_attention.py -q -p no:cacheprovider -k "token or pattern or power" > gpurun_out/${tag}_pytest_paired.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_paired.log
