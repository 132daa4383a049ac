tag=r02v
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullcov.py -q -s -p no:cacheprovider -k "token" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 600 python -m pytest tests/test_heads_parallel.py -q -p no:cacheprovider -m gpu > gpurun_out/${tag}_pytest_hp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_hp.log
