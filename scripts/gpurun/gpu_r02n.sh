# LPT window size (1 / 2 / 4 x SM count): forward + backward at H33 and H132, same box
tag=r02n
mkdir -p gpurun_out
for c in hunyuan132 hunyuan33; do
  for i in 1 2; do
    timeout 300 python scripts/fwd_bwd_time.py --config $c >> gpurun_out/${tag}_win.txt 2>&1
    RADIAL_CUDA_LIB=variants/win1/libradial_cuda.so timeout 300 python scripts/fwd_bwd_time.py --config $c >> gpurun_out/${tag}_win.txt 2>&1
    RADIAL_CUDA_LIB=variants/win4/libradial_cuda.so timeout 300 python scripts/fwd_bwd_time.py --config $c >> gpurun_out/${tag}_win.txt 2>&1
  done
done
