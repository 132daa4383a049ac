# dQ kernel chain: S loaded in halves (split), dP loaded under the last exponentials (edp32/48)
tag=r03i
mkdir -p gpurun_out
for i in 1 2 3; do
  for c in hunyuan33 mochi28; do
    for v in base dqsplit edp48 edp32 split_edp48; do
      lib=""; [ "$v" != base ] && lib="RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so"
      env $lib timeout 300 python scripts/fwd_bwd_time.py --config $c --fwd-iters 2 --bwd-iters 3 | sed "s/^/$v /" >> gpurun_out/${tag}_ab.txt 2>&1
    done
  done
done
for v in dqsplit edp48 split_edp48; do
  RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so timeout 900 python -m pytest tests/test_gpu_backward.py -q -x -p no:cacheprovider -k "oracle or floor" > gpurun_out/${tag}_pytest_$v.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_$v.log
done
