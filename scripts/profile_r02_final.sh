#!/bin/bash
# Round-2 evidence in one gpurun call (repo root): full GPU suite, the default bench line, the
# other BASELINE configs' lines, per-rank head-share scaling, token-exact timing, the ncu launch
# list of the bench command and ncu --set full captures (forward, token-exact forward, dQ, dK/dV
# at H33).  bash scripts/profile_r02_final.sh <tag>
tag=${1:-r02l}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> $out/${tag}_pytest.log
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
for c in wan21 mochi28 hunyuan132; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-extra > $out/${tag}_bench_$c.json 2> $out/${tag}_bench_$c.err
done
timeout 300 python scripts/head_scaling.py > $out/${tag}_scaling.txt 2>&1
timeout 300 python scripts/token_mode_time.py >> $out/${tag}_scaling.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/${tag}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-extra > $out/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_fwd -c 1 -o $out/${tag}_fwd_h33 \
    python scripts/profile_step.py --config hunyuan33 > $out/${tag}_ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_fwd -c 1 -o $out/${tag}_tok_h33 \
    python scripts/profile_step.py --config hunyuan33 --token > $out/${tag}_ncu_tok.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_bwd_dq -c 1 -o $out/${tag}_bwd_dq_h33 \
    python scripts/profile_bwd.py --config hunyuan33 > $out/${tag}_ncu_dq.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_bwd_dkdv -c 1 -o $out/${tag}_bwd_dkdv_h33 \
    python scripts/profile_bwd.py --config hunyuan33 > $out/${tag}_ncu_dkdv.log 2>&1
