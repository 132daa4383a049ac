# register split 40/232 (spill-free) with and without the stale-max path vs the previous commit
tag=r02q
mkdir -p gpurun_out
for i in 1 2; do
  for c in hunyuan33 mochi28; do
    for v in stale_r40 nostale_r40 head; do
      RADIAL_CUDA_LIB=variants/$v/libradial_cuda.so timeout 300 python scripts/fwd_ab.py --config $c >> gpurun_out/${tag}_ab_$v.txt 2>&1
    done
  done
done
