# final-code sanitizer pass (all four tools) and determinism stress
tag=r03e
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/${tag}_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_san_${tool}.log
done
timeout 900 python scripts/stress_determinism.py --config hunyuan33 --iters 12 > gpurun_out/${tag}_stress_h33.json 2>&1
timeout 900 python scripts/stress_determinism.py --config mochi28 --iters 30 > gpurun_out/${tag}_stress_m28.json 2>&1
timeout 900 python scripts/stress_determinism.py --config hunyuan132 --iters 3 > gpurun_out/${tag}_stress_h132.json 2>&1
