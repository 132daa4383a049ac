# L2 eviction hints (Q evict-first, K/V evict-last, O streaming stores) vs none, same box
tag=r02x
mkdir -p gpurun_out
for i in 1 2; do
  for c in hunyuan132 hunyuan33 mochi28; do
    timeout 300 python scripts/fwd_bwd_time.py --config $c --bwd-iters 1 >> gpurun_out/${tag}_ab.txt 2>&1
    RADIAL_CUDA_LIB=variants/l2hints/libradial_cuda.so timeout 300 python scripts/fwd_bwd_time.py --config $c --bwd-iters 1 >> gpurun_out/${tag}_ab.txt 2>&1
  done
done
RADIAL_CUDA_LIB=variants/l2hints/libradial_cuda.so timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:radial_attn_fwd -c 1 --csv python scripts/profile_step.py --config hunyuan33 > gpurun_out/${tag}_ncu_l2.csv 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:radial_attn_fwd -c 1 --csv python scripts/profile_step.py --config hunyuan33 > gpurun_out/${tag}_ncu_base.csv 2>&1
