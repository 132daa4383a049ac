#!/bin/bash
# Round-2 evidence in one gpurun call (repo root): GPU tests, the bench line, token-exact
# timing, racecheck, the ncu launch list of the bench command and ncu --set full captures of
# the forward (block + token-exact) and both backward kernels at H33.
#   bash scripts/profile_r02.sh <tag> [skip-tests]
tag=${1:-r02}
out=gpurun_out
mkdir -p $out
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/${tag}_pytest.log 2>&1
  echo "pytest rc=$?" >> $out/${tag}_pytest.log
  timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_cases.py \
    > $out/${tag}_san_racecheck.log 2>&1; echo "rc=$?" >> $out/${tag}_san_racecheck.log
  timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python scripts/sanitize_cases.py \
    > $out/${tag}_san_initcheck.log 2>&1; echo "rc=$?" >> $out/${tag}_san_initcheck.log
fi
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 300 python scripts/token_mode_time.py > $out/${tag}_token.txt 2>&1
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
