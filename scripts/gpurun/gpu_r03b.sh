# backward: exp2 share on the FMA pipe in the dQ (1/8 steps) and dK/dV (1/4 steps) kernels
tag=r03b
mkdir -p gpurun_out
for i in 1 2 3; do
  for c in hunyuan33 mochi28; do
    for v in base dqpoly1 dq2kv0 dq1kv1 dq1kv2; do
      lib=""; [ "$v" != base ] && lib="RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so"
      env $lib timeout 300 python scripts/fwd_bwd_time.py --config $c --fwd-iters 2 --bwd-iters 3 | sed "s/^/$v /" >> gpurun_out/${tag}_ab.txt 2>&1
    done
  done
done
