# dQ kernel: share of exp2 on the FMA pipe (RADIAL_BWD_DQ_POLY 0..3), dQ alone and full backward
tag=r03a
mkdir -p gpurun_out
for i in 1 2; do
  for v in base dqpoly1 dqpoly2 dqpoly3; do
    lib=""; [ "$v" != base ] && lib="RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so"
    env $lib RADIAL_BWD_DQ_ONLY=1 timeout 300 python scripts/fwd_bwd_time.py --config hunyuan33 --fwd-iters 2 --bwd-iters 4 | sed "s/^/$v dqonly /" >> gpurun_out/${tag}_ab.txt 2>&1
    env $lib timeout 300 python scripts/fwd_bwd_time.py --config hunyuan33 --fwd-iters 2 --bwd-iters 3 | sed "s/^/$v full /" >> gpurun_out/${tag}_ab.txt 2>&1
  done
done
