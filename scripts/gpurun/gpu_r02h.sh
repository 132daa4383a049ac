# racecheck probe (both release modes); token-exact timing hooks (variant builds)
tag=r02h
mkdir -p gpurun_out
for m in 0 1; do
  timeout 300 compute-sanitizer --tool racecheck python scripts/racecheck_probe.py $m > gpurun_out/${tag}_probe_$m.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_probe_$m.log
done
timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token_base.txt 2>&1
RADIAL_CUDA_LIB=variants/tok_nomask/libradial_cuda.so timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token_nomask.txt 2>&1
RADIAL_CUDA_LIB=variants/tok_noselect/libradial_cuda.so timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token_noselect.txt 2>&1
