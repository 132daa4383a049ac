# dK/dV: dP^T loaded under the last exponentials (kedp32/48) vs after; dQ early-dP now default
tag=r03j
mkdir -p gpurun_out
for i in 1 2 3; do
  for c in hunyuan33 mochi28; do
    for v in base kedp48 kedp32; do
      lib=""; [ "$v" != base ] && lib="RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so"
      env $lib timeout 300 python scripts/fwd_bwd_time.py --config $c --fwd-iters 2 --bwd-iters 3 | sed "s/^/$v /" >> gpurun_out/${tag}_ab.txt 2>&1
    done
  done
done
timeout 1500 python -m pytest tests/test_gpu_backward.py tests/test_gpu_fullcov.py -q -p no:cacheprovider -k "backward" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
