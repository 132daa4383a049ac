tag=r02k
mkdir -p gpurun_out
timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token_base.txt 2>&1
RADIAL_CUDA_LIB=variants/tok_nomask/libradial_cuda.so timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token_nomask.txt 2>&1
RADIAL_CUDA_LIB=variants/tok_noselect/libradial_cuda.so timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token_noselect.txt 2>&1
