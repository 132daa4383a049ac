# stale-max softmax: parity (forward tests, full coverage, peaked) and same-box A/B against the
# previous commit and the same code with the stale-max path compiled out
tag=r02p
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_attention.py tests/test_gpu_fullcov.py tests/test_gpu_backward.py -q -x -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for i in 1 2; do
  for c in hunyuan33 mochi28; do
    timeout 300 python scripts/fwd_ab.py --config $c >> gpurun_out/${tag}_ab_new.txt 2>&1
    RADIAL_CUDA_LIB=variants/head/libradial_cuda.so timeout 300 python scripts/fwd_ab.py --config $c >> gpurun_out/${tag}_ab_head.txt 2>&1
    RADIAL_CUDA_LIB=variants/nostale/libradial_cuda.so timeout 300 python scripts/fwd_ab.py --config $c >> gpurun_out/${tag}_ab_nostale.txt 2>&1
  done
done
timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token.txt 2>&1
