# token-exact: spill-free mask update + 32-bit radial band test, A/B vs previous commit; K1 and
# token parity tests
tag=r02m
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_new.txt 2>&1
  RADIAL_CUDA_LIB=variants/head/libradial_cuda.so timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_head.txt 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_mask.py tests/test_gpu_attention.py tests/test_cpp_dropin.py tests/test_cli.py -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
