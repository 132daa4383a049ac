# racecheck probe (tool vs mbarrier-ordered bulk copies), backward bf16-floor test, token-exact
# timing and one ncu --set full capture of the token-exact forward with source
tag=r02f
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool racecheck python scripts/racecheck_probe.py > gpurun_out/${tag}_racecheck_probe.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_racecheck_probe.log
timeout 600 python -m pytest tests/test_gpu_backward.py -q -s -k floor -p no:cacheprovider > gpurun_out/${tag}_floor.log 2>&1
timeout 300 python scripts/token_mode_time.py > gpurun_out/${tag}_token.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_fwd -c 1 -o gpurun_out/${tag}_tok_h33 \
    python scripts/profile_step.py --config hunyuan33 --token > gpurun_out/${tag}_ncu_tok.log 2>&1
