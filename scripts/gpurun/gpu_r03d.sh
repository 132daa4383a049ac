# forward: share of the softmax exponentials on the FMA pipe (RADIAL_POLY_PAIRS 0/1/2 of 8) with
# the 40/232 register split
tag=r03d
mkdir -p gpurun_out
for i in 1 2 3; do
  for c in hunyuan33 mochi28; do
    for v in base fpoly1 fpoly2; do
      lib=""; [ "$v" != base ] && lib="RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so"
      env $lib timeout 300 python scripts/fwd_ab.py --config $c | sed "s/^/$v /" >> gpurun_out/${tag}_ab.txt 2>&1
    done
  done
done
