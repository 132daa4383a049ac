# full coverage of the other K2 tile instantiations (B 64 / d 64) at M28
tag=r03f
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullcov.py -q -s -p no:cacheprovider -k "tile_shapes" > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
