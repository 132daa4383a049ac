tag=r02c
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 120 python scripts/fwd_ab.py --config hunyuan33 > gpurun_out/${tag}_ab_pair.txt 2>&1
RADIAL_FWD_PAIR=0 timeout 120 python scripts/fwd_ab.py --config hunyuan33 > gpurun_out/${tag}_ab_one.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
