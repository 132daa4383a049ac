# CTA-pair forward: ncu full captures (sparse + dense, H33) and A/B timings at M28/H132
tag=r02d
mkdir -p gpurun_out
RADIAL_FWD_PAIR=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_fwd_pair -c 2 -o gpurun_out/${tag}_pair_h33 \
    python scripts/profile_step.py --config hunyuan33 --dense > gpurun_out/${tag}_ncu_pair.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radial_attn_fwd -s 1 -c 1 -o gpurun_out/${tag}_one_dense_h33 \
    python scripts/profile_step.py --config hunyuan33 --dense > gpurun_out/${tag}_ncu_one.log 2>&1
for c in mochi28 hunyuan132; do
  timeout 300 python scripts/fwd_ab.py --config $c --no-dense >> gpurun_out/${tag}_ab.txt 2>&1
  RADIAL_FWD_PAIR=1 timeout 300 python scripts/fwd_ab.py --config $c --no-dense >> gpurun_out/${tag}_ab.txt 2>&1
done
