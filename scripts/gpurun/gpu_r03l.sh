# dK/dV: 1/8 and 2/8 of the exponentials on the FMA pipe (quads per 8)
tag=r03l
mkdir -p gpurun_out
for i in 1 2 3; do
  for c in hunyuan33 mochi28; do
    for v in base kvpoly8_1 kvpoly8_2; do
      lib=""; [ "$v" != base ] && lib="RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so"
      env $lib timeout 300 python scripts/fwd_bwd_time.py --config $c --fwd-iters 2 --bwd-iters 3 | sed "s/^/$v /" >> gpurun_out/${tag}_ab.txt 2>&1
    done
  done
done
