# N > 1 bench code path end to end on a one-GPU box (ranks share cuda:0, gloo collectives)
tag=r02s
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --shared-gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench2.json 2> gpurun_out/${tag}_bench2.err
echo "rc=$?" >> gpurun_out/${tag}_bench2.err
timeout 900 python bench.py --gpus 4 --shared-gpu --steps 3 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/${tag}_bench4.json 2> gpurun_out/${tag}_bench4.err
echo "rc=$?" >> gpurun_out/${tag}_bench4.err
timeout 600 python bench.py --gpus 2 > gpurun_out/${tag}_bench_mismatch.json 2> gpurun_out/${tag}_bench_mismatch.err
echo "rc=$?" >> gpurun_out/${tag}_bench_mismatch.err
