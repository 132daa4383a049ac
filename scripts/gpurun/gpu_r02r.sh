# forward register split 40/232 (product) vs 72/216 (previous commit): forward tests, A/B at
# H33 / M28 / W21 and token-exact
tag=r02r
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_mask.py -q -x -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for i in 1 2 3; do
  for c in hunyuan33 mochi28 wan21; do
    timeout 300 python scripts/fwd_ab.py --config $c >> gpurun_out/${tag}_ab_new.txt 2>&1
    RADIAL_CUDA_LIB=variants/head/libradial_cuda.so timeout 300 python scripts/fwd_ab.py --config $c >> gpurun_out/${tag}_ab_head.txt 2>&1
  done
done
for i in 1 2; do
  timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_new.txt 2>&1
  RADIAL_CUDA_LIB=variants/head/libradial_cuda.so timeout 300 python scripts/token_mode_time.py >> gpurun_out/${tag}_token_head.txt 2>&1
done
