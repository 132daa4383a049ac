# backward L2 eviction hints vs none (same box), backward parity
tag=r02y
mkdir -p gpurun_out
for i in 1 2; do
  for c in hunyuan33 mochi28 hunyuan132; do
    timeout 300 python scripts/fwd_bwd_time.py --config $c --fwd-iters 3 --bwd-iters 3 >> gpurun_out/${tag}_ab.txt 2>&1
    RADIAL_CUDA_LIB=variants/nobwdhint/libradial_cuda.so timeout 300 python scripts/fwd_bwd_time.py --config $c --fwd-iters 3 --bwd-iters 3 >> gpurun_out/${tag}_ab.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_backward.py -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
