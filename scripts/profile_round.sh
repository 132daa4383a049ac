#!/bin/bash
# One GPU call's worth of evidence for profiles/ (run under gpurun from the repo root):
#   bench line, ncu launch list of the bench command, ncu --set full of the forward and
#   of both backward kernels at H33.  Usage: bash scripts/profile_round.sh <tag>
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
timeout 600 python bench.py --bwd > $out/bench_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_fwd_$tag.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $out/ncu_launch_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:radial_attn_fwd -c 1 -o $out/fwd_h33_$tag \
    python scripts/profile_step.py --config hunyuan33 > $out/ncu_fwd_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:radial_attn_bwd_dq -c 1 -o $out/bwd_dq_h33_$tag \
    python scripts/profile_bwd.py --config hunyuan33 > $out/ncu_dq_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:radial_attn_bwd_dkdv -c 1 -o $out/bwd_dkdv_h33_$tag \
    python scripts/profile_bwd.py --config hunyuan33 > $out/ncu_dkdv_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_bwd_$tag.csv \
    python scripts/profile_bwd.py --config hunyuan33 > /dev/null 2>&1
