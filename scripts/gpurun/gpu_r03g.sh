# smoke() (now also the d128/B128 forward and K3) and the final default bench line
tag=r03g
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "rc=$?" >> gpurun_out/${tag}_bench.err
