# dK/dV split stage release under racecheck; backward tests at the tightened tolerance; forward
# timing after the per-role work-item change (spill-free MMA warp); bench line
tag=r02g
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/${tag}_san_racecheck.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_san_racecheck.log
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_attention.py -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
for c in hunyuan33 mochi28; do timeout 300 python scripts/fwd_ab.py --config $c --no-dense >> gpurun_out/${tag}_ab.txt 2>&1; done
timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token.txt 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
