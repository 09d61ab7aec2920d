cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r4l_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r4l_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r4l_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r4l_bench.json 2>gpurun_out/r4l_bench.err
echo done
