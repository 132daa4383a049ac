# token-exact: mask built before the S wait + R2P select; A/B vs the committed HEAD library
# (variants/head) on the same box; token parity tests
tag=r02i
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_cpp_dropin.py -q -p no:cacheprovider -k "token or pattern or dropin or power" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for i in 1 2; do
  timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_new.txt 2>&1
  RADIAL_CUDA_LIB=variants/head/libradial_cuda.so timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_head.txt 2>&1
done
for c in hunyuan33 mochi28; do
  timeout 300 python scripts/fwd_ab.py --config $c --no-dense >> gpurun_out/${tag}_ab_new.txt 2>&1
  RADIAL_CUDA_LIB=variants/head/libradial_cuda.so timeout 300 python scripts/fwd_ab.py --config $c --no-dense >> gpurun_out/${tag}_ab_head.txt 2>&1
done
