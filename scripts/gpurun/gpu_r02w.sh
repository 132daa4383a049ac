tag=r02w
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullcov.py tests/test_gpu_mask.py -q -s -p no:cacheprovider -k "other_configs or paper_scale" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
