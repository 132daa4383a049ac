# final code: full GPU suite, default bench line, other configs' lines, ncu of the dQ kernel
tag=r03k
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
for c in wan21 mochi28 hunyuan132; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-extra > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_bwd_dq -c 1 -o gpurun_out/${tag}_bwd_dq_h33 \
    python scripts/profile_bwd.py --config hunyuan33 > gpurun_out/${tag}_ncu_dq.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_bwd.csv \
    python scripts/profile_bwd.py --config hunyuan33 > /dev/null 2>&1
