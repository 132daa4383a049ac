# FlashAttention-4 comparator refresh on the final code (same box, same inputs)
tag=r03n
mkdir -p gpurun_out
timeout 1200 python scripts/fa4_compare.py --config hunyuan33 --bwd > gpurun_out/${tag}_fa4_h33.json 2> gpurun_out/${tag}_fa4_h33.err
echo "rc=$?" >> gpurun_out/${tag}_fa4_h33.err
timeout 900 python scripts/fa4_compare.py --config mochi28 --bwd > gpurun_out/${tag}_fa4_m28.json 2> gpurun_out/${tag}_fa4_m28.err
echo "rc=$?" >> gpurun_out/${tag}_fa4_m28.err
